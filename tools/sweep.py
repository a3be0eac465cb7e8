"""Message-size sweep of the compressed AllReduce (BASELINE config 4 / SURVEY §8(d) C5) on the GPUs
this process sees, written in the reference's report formats (report.emit_csv / emit_markdown,
bench.cpp:551-671).

With one GPU the ranks form a loopback group on cuda:0 (their ring kernels share the device; frames
move through HBM, not NVLink).  Per (ranks, size, codec pin): allreduce_eb on Laplacian data (the C2
generator, b = 1e-2, abs eb 1e-4), device time from CUDA events, WireStats of the timed calls, and
speed-up against the RAW-pinned run of the same size.

    python tools/sweep.py --ranks 2 4 --sizes-mb 1 4 16 64 256 --out profiles/r01_sweep
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_12396_b200 import abi, report, zcomm  # noqa: E402

PINS = [("raw", abi.PIN_RAW), ("auto", abi.PIN_AUTO), ("fixedlen", abi.PIN_FIXEDLEN), ("huffman", abi.PIN_HUFFMAN)]
CODEC_INDEX = {"auto": 0, "raw": 1, "fixedlen": 2, "huffman": 3}


def laplacian(count, rank):
    g = torch.Generator(device="cuda")
    g.manual_seed(100 + rank)
    u = torch.rand(count, generator=g, device="cuda", dtype=torch.float64) - 0.5
    return (-1e-2 * torch.sign(u) * torch.log1p(-2 * u.abs())).float()


def run(n, count, pin, reps, warmup, shared=True):
    xs = [laplacian(count, r) for r in range(n)]
    gmax = max(float(x.abs().max().item()) for x in xs)
    rel = 1e-4 / gmax
    grp = zcomm.Group(n, cfg=zcomm.collective_config(pin))
    if pin == abi.PIN_HUFFMAN or (pin == abi.PIN_AUTO and shared):
        scale = 2 * rel * gmax
        grp.set_shared_huffman_from_bytes(zcomm.eb_quantize_with_scale(xs[0][: 1 << 20], scale).cpu().numpy().view("uint8"))
    outs = [torch.empty_like(x) for x in xs]
    for _ in range(warmup):
        grp.allreduce_eb(xs, rel, outs=outs)
    torch.cuda.synchronize()
    grp.reset_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    a.record()
    for _ in range(reps):
        grp.allreduce_eb(xs, rel, outs=outs)
    b.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - w0) / reps
    dt = a.elapsed_time(b) / 1e3 / reps
    w = grp.wire_stats()
    grp.close()
    return dt, wall, w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, nargs="+", default=[2, 4])
    ap.add_argument("--sizes-mb", type=int, nargs="+", default=[1, 4, 16, 64, 256])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--out", default="profiles/sweep")
    ap.add_argument("--no-shared", action="store_true",
                    help="Auto without a shared Huffman context (FixedLen / RAW only: the fused ring kernel runs)")
    args = ap.parse_args()
    rows = []
    for n in args.ranks:
        for mb in args.sizes_mb:
            count = mb * (1 << 20) // 4
            t_raw = None
            for name, pin in PINS:
                dt, wall, w = run(n, count, pin, args.reps, args.warmup, shared=not args.no_shared)
                if name == "raw":
                    t_raw = dt
                r = report.ReportRow(collective=0, ranks=n, msg_bytes=4 * count, codec=CODEC_INDEX[name], quant=1,
                                     dist=0, seed=100, overlap=0, regime=0)
                r.sim_time_sec, r.wall_time_sec = dt, wall
                r.fill_wire(w)
                r.fill_bandwidths(4 * count)
                r.speedup_vs_raw = t_raw / dt if t_raw else 1.0
                rows.append(r)
                print(f"n={n} {mb:5d} MB {name:9s} {dt * 1e3:8.3f} ms  algbw {r.alg_bw_bytes_per_sec / 1e9:7.1f} GB/s  "
                      f"CR {r.cr_final:.3f}  x{r.speedup_vs_raw:.2f} vs raw", flush=True)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".csv", "w") as f:
        f.write(report.emit_csv(rows))
    with open(args.out + ".md", "w") as f:
        f.write(f"Loopback compressed AllReduce on {torch.cuda.get_device_name(0)} "
                f"({torch.cuda.device_count()} GPU(s) visible; ranks share a GPU when there are fewer GPUs than ranks). "
                "`sim time` = device time from CUDA events.\n\n")
        f.write(report.emit_markdown(rows))


if __name__ == "__main__":
    main()
