"""Developer probe: loopback ring AllReduce (one process, N ranks on cuda:0) through the group API."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_12396_b200 import zcomm  # noqa: E402

n = int(os.environ.get("NR", 2))
count = int(os.environ.get("COUNT", 64 << 20))
xs = []
for r in range(n):
    g = torch.Generator(device="cuda").manual_seed(100 + r)
    u = torch.rand(count, generator=g, device="cuda", dtype=torch.float64) - 0.5
    xs.append((-1e-2 * torch.sign(u) * torch.log1p(-2 * u.abs())).float())
grp = zcomm.Group(n)
rel = 1e-4 / max(float(x.abs().max()) for x in xs)
for _ in range(2):
    outs = grp.allreduce_eb(xs, rel)
torch.cuda.synchronize()
reps = int(os.environ.get("REPS", 5))
t0 = time.perf_counter()
for _ in range(reps):
    outs = grp.allreduce_eb(xs, rel)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / reps
exact = sum(x.double() for x in xs)
err = float((outs[0].double() - exact).abs().max())
print(f"group allreduce_eb n={n} count={count}: {dt * 1e3:.2f} ms/step, algbw {4 * count / dt / 1e9:.1f} GB/s, "
      f"max err {err:.3e} (bound {n * 1e-4:.1e}), wire {grp.wire_stats().payload_bytes}")
