"""compute-sanitizer target: a small 2-rank loopback allreduce_eb, allgather and broadcast (the flag
protocol, the fused sinks, the relay lane) plus one codec round trip, exactness asserted."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_12396_b200 import zcomm  # noqa: E402

n = int(os.environ.get("NR", 3))
count = 3 * ((3 << 20) // 4)  # chunk bases 16-byte aligned: the fused ring kernel runs
g = torch.Generator(device="cuda").manual_seed(5)
xs = [torch.randn(count, generator=g, device="cuda") for _ in range(n)]
grp = zcomm.Group(n)
rel = 1e-3
outs = grp.allreduce_eb(xs, rel, torch.float64)
exact = sum(x.double() for x in xs)
assert float((outs[0] - exact).abs().max()) <= n * rel * max(float(x.abs().max()) for x in xs) * 1.0001
blocks = [torch.randint(-1000, 1000, (count,), generator=g, device="cuda", dtype=torch.int32) for _ in range(n)]
alls = grp.allgather(blocks)
assert all(torch.equal(a, torch.cat(blocks)) for a in alls)
data = [blocks[0].clone() if r == 0 else torch.zeros_like(blocks[0]) for r in range(n)]
grp.broadcast(data, 0)
assert all(torch.equal(d, blocks[0]) for d in data)
fr = zcomm.encode_batches(xs[0], 0, scale=2e-4)
y = zcomm.decode_batches(fr, None, scale=2e-4)
assert float((y.double() - xs[0].double()).abs().max()) <= 1e-4 * 1.0001 + 1e-6
print("sanitize probe ok")
