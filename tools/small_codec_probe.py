"""Developer probe: device time of the codec kernels on SMALL inputs (the latency regime of small
collectives): encode_batches / decode_batches on fp32 and int32 inputs of 64 KiB .. 4 MiB, CUDA
events around R back-to-back calls (eager launches; launch overhead included)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_12396_b200 import abi, zcomm  # noqa: E402

R = int(os.environ.get("REPS", 50))
for kb in (64, 256, 512, 1024, 4096):
    n = kb * 256
    x = torch.randn(n, device="cuda") * 0.01
    scale = 2e-4
    fr = zcomm.encode_batches(x, abi.PIN_FIXEDLEN, scale=scale)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    for name, fn in (("encode f32", lambda: zcomm.encode_batches(x, abi.PIN_FIXEDLEN, scale=scale, frames=fr)),
                     ("decode f32", lambda: zcomm.decode_batches(fr, scale=scale, out=out))):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(R):
            fn()
        b.record()
        torch.cuda.synchronize()
        print(f"{kb:5d} KiB {name}: {a.elapsed_time(b) / R * 1e3:7.1f} us/call", flush=True)
