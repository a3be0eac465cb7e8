"""Developer probe: loopback ring AllReduce (one process, N ranks on cuda:0) through the group API.
Env: NR ranks, COUNT per rank, REPS, PIN (auto|fixedlen|raw|huffman), SHARED=1 primes a shared
Huffman context (bench.cpp:169-204)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_12396_b200 import abi, zcomm  # noqa: E402

n = int(os.environ.get("NR", 2))
count = int(os.environ.get("COUNT", 64 << 20))
pin = {"auto": abi.PIN_AUTO, "fixedlen": abi.PIN_FIXEDLEN, "raw": abi.PIN_RAW,
       "huffman": abi.PIN_HUFFMAN}[os.environ.get("PIN", "auto")]
xs = []
for r in range(n):
    g = torch.Generator(device="cuda").manual_seed(100 + r)
    u = torch.rand(count, generator=g, device="cuda", dtype=torch.float64) - 0.5
    xs.append((-1e-2 * torch.sign(u) * torch.log1p(-2 * u.abs())).float())
grp = zcomm.Group(n, cfg=zcomm.collective_config(pin))
rel = 1e-4 / max(float(x.abs().max()) for x in xs)
if os.environ.get("SHARED"):
    grp.set_shared_huffman(zcomm.HuffmanContext.from_bytes(
        zcomm.eb_quantize_with_scale(xs[0][: 1 << 20], 2 * rel * max(float(x.abs().max()) for x in xs))))
outs = [torch.empty_like(x) for x in xs]
for _ in range(int(os.environ.get("WARM", 2))):
    grp.allreduce_eb(xs, rel, outs=outs)
torch.cuda.synchronize()
reps = int(os.environ.get("REPS", 5))
t0 = time.perf_counter()
for _ in range(reps):
    grp.allreduce_eb(xs, rel, outs=outs)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / reps
exact = sum(x.double() for x in xs)
err = float((outs[0].double() - exact).abs().max())
print(f"group allreduce_eb n={n} count={count} pin={os.environ.get('PIN', 'auto')}: {dt * 1e3:.3f} ms/step, "
      f"algbw {4 * count / dt / 1e9:.1f} GB/s, max err {err:.3e} (bound {n * 1e-4:.1e}), "
      f"wire {grp.wire_stats().payload_bytes}")
