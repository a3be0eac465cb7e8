"""Measured send/decode timeline of the compressed ring AllReduce (BASELINE config 1 shape: 2-rank
loopback group, 64 Mi Laplacian fp32 per rank, abs eb 1e-4) written in the reference's timeline CSV
format (pipeline.cpp:160-170) plus an overlap summary — the ablation SPEC shows with a modelled
schedule, here from CUDA events.  Usage: python tools/timeline.py OUT.csv [count]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_12396_b200 import report, zcomm  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/timeline.csv"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 64 << 20
g = zcomm.Group(2)
gen = torch.Generator(device="cuda").manual_seed(100)
xs = []
for r in range(2):
    u = torch.rand(count, device="cuda", generator=gen, dtype=torch.float64) - 0.5
    xs.append((-1e-2 * torch.sign(u) * torch.log1p(-2 * u.abs())).float())
gmax = max(float(x.abs().max()) for x in xs)
rel = 1e-4 / gmax
g.allreduce_eb(xs, rel)  # warm-up
torch.cuda.synchronize()
g.timeline_enable(4096)
g.allreduce_eb(xs, rel)
rows = g.timeline()
with open(out, "w") as f:
    f.write(report.emit_timeline_csv(rows))
summ = report.overlap_summary(rows)
summ["rows"] = len(rows)
summ["workload"] = "2-rank loopback allreduce_eb, %d Laplacian fp32 per rank, abs eb 1e-4 (ranks share one GPU)" % count
print(json.dumps(summ))
