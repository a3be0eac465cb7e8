"""Developer probe: small-message latency of the loopback group AllReduce (one process, N ranks on
cuda:0).  Per pin: wall time per group allreduce_eb call (the call is synchronous: enqueue, run,
drain), the same call on symbols (allreduce_sym), and an empty barrier (allreduce_max).
Env: NR ranks (2), COUNT elements per rank (262144 = 1 MiB), REPS (50), PINS (raw,fixedlen,auto),
EB_ONLY=1 (allreduce_eb only); ZC_HOST_TIMING=1 makes the
library print its enqueue / drain split per call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_12396_b200 import abi, zcomm  # noqa: E402

n = int(os.environ.get("NR", 2))
count = int(os.environ.get("COUNT", 1 << 18))
reps = int(os.environ.get("REPS", 50))
xs = []
for r in range(n):
    g = torch.Generator(device="cuda").manual_seed(100 + r)
    u = torch.rand(count, generator=g, device="cuda", dtype=torch.float64) - 0.5
    xs.append((-1e-2 * torch.sign(u) * torch.log1p(-2 * u.abs())).float())
rel = 1e-4 / max(float(x.abs().max()) for x in xs)
outs = [torch.empty_like(x) for x in xs]
syms0 = [torch.randint(-100, 100, (count,), dtype=torch.int32, device="cuda") for _ in range(n)]
syms = [s.clone() for s in syms0]


def sym_call(grp):
    for s, s0 in zip(syms, syms0):  # in place: restart from the same symbols
        s.copy_(s0)
    grp.allreduce(syms, [1.0] * n)


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2] * 1e6, ts[0] * 1e6


PINS = {"raw": abi.PIN_RAW, "fixedlen": abi.PIN_FIXEDLEN, "auto": abi.PIN_AUTO}
for name in os.environ.get("PINS", "raw,fixedlen,auto").split(","):
    pin = PINS[name]
    grp = zcomm.Group(n, cfg=zcomm.collective_config(pin))
    med, lo = timeit(lambda: grp.allreduce_eb(xs, rel, outs=outs))
    if os.environ.get("EB_ONLY"):
        print(f"n={n} count={count} {name:8s}: allreduce_eb median {med:7.1f} us (min {lo:7.1f})", flush=True)
        grp.close()
        continue
    med_s, lo_s = timeit(lambda: sym_call(grp))
    med_m, lo_m = timeit(lambda: grp.allreduce_max([1.0] * n))
    print(f"n={n} count={count} {name:8s}: allreduce_eb median {med:7.1f} us (min {lo:7.1f}); "
          f"allreduce_sym {med_s:7.1f} us (min {lo_s:7.1f}); allreduce_max {med_m:7.1f} us (min {lo_m:7.1f})",
          flush=True)
    grp.close()
