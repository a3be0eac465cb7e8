"""Developer probe: device QSGD timings — mt19937_64 draws (jump-ahead + twist), qsgd_quantize_chunk
(caller norm, parallel), the sequential norm, and a 2-rank loopback allreduce_qsgd."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_12396_b200 import zcomm  # noqa: E402

L = zcomm.lib()
res = {}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for n in (1 << 20, 64 << 20):
    x = torch.randn(n, device="cuda")
    d = torch.empty(n, dtype=torch.int64, device="cuda")
    res[f"mt19937_64_draws_ms_n{n}"] = timed(lambda: zcomm.check(L.zc_mt19937_64(1, 0, n, zcomm._ptr(d), zcomm._stream())))
    res[f"qsgd_chunk_ms_n{n}"] = timed(lambda: zcomm.qsgd_quantize_chunk(x, 16, 100.0, 7))
    nd = torch.zeros(1, dtype=torch.float64, device="cuda")
    res[f"seq_norm_ms_n{n}"] = timed(lambda: zcomm.check(L.zc_qsgd_norm_f32(zcomm._ptr(x), n, zcomm._ptr(nd), None,
                                                                          zcomm._stream())), reps=1)
g = zcomm.Group(2)
xs = [torch.randn(16 << 20, device="cuda") for _ in range(2)]
res["allreduce_qsgd_2rank_16Mi_ms"] = timed(lambda: g.allreduce_qsgd(xs, 16, [1, 2]), reps=1)
print(json.dumps({k: round(v, 3) for k, v in res.items()}))
