"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list: per-kernel launches,
mean device time and share of the total (ncu times are cold-cache and serialised: compare shares)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
ik, im, iu, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
agg = {}
for r in data:
    if len(r) > iv and r[im] == "gpu__time_duration.sum":
        agg.setdefault(r[ik][:70], []).append(float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:72s} launches={len(v):3d} mean_us={sum(v) / len(v):10.2f} share={sum(v) / tot * 100:5.1f}%")
