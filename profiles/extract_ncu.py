"""Summarise an `ncu --set full` capture of the bench's hot kernels into profiles/.

    python profiles/extract_ncu.py gpurun_out/prof_rNN_full.ncu-rep rNN

Writes profiles/<tag>_ncu_full_summary.txt (key counters per kernel) and updates
profiles/ncu_traffic.json: dram read+write bytes per CALL, keyed the way bench.py looks them up
("zc_encode_f32": the kernels of one zc_encode_batches_f32 call — profile / range / scan / emit;
"zc_decode": one zc_decode_batches_f32 call — fl_decode / decode / fixup).  Capture exactly one
encode + decode call (e.g. --launch-skip / --launch-count over tools/codec_probe.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic",
]
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}


def main(rep, tag):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full --clock-control none ({os.path.basename(rep)}); one launch per kernel, cold L2 (ncu replay)"]
    traffic_path = os.path.join(HERE, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    sums = {}
    for v in data:
        name = v[hdr.index("Kernel Name")]
        lines.append(name)
        vals = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                vals[k] = v[i]
                lines.append(f"  {k:60s} {v[i]:>14s} {units[i]}")
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(k)
            b += float(v[i].replace(",", "")) * UNIT.get(units[i], 1.0)
        enc = any(k in name for k in ("profile_kernel", "range_kernel", "scan_kernel", "emit_kernel"))
        dec = any(k in name for k in ("decode_kernel", "fixup_kernel"))
        key = "zc_encode_f32" if enc else ("zc_decode" if dec else None)
        if key:
            sums[key] = sums.get(key, 0) + int(b)
    for key, b in sums.items():
        traffic[key] = b
        traffic[key + "_source"] = f"{tag}: {os.path.basename(rep)} (sum over the call's kernels)"
        lines.append(f"{key}: dram read+write per call = {b} bytes")
    with open(os.path.join(HERE, f"{tag}_ncu_full_summary.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(traffic_path, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
