"""Developer probe: zc_codec_roundtrip_host_f32 (pinned host in/out) per pipeline group size, beside
the box's raw pinned H2D / D2H / bidirectional copy bandwidth (the PCIe ceiling of e2e)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_12396_b200 import abi, zcomm  # noqa: E402

count = 64 << 20
L = zcomm.lib()
x = torch.randn(count, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
hx = torch.empty(count, dtype=torch.float32, pin_memory=True)
hx.copy_(x.cpu())
hy = torch.empty(count, dtype=torch.float32, pin_memory=True)
work = torch.empty_like(x)
fr = zcomm.alloc_frames(count * 4, x.device)
err = torch.zeros(1, dtype=torch.int32, device="cuda")
hint, cfg = abi.make_hint(), zcomm.default_arb_config()
prime = zcomm.eb_quantize_with_scale(x[: 1 << 20], 2e-4)
ctx = zcomm.HuffmanContext.from_bytes(prime)
s = torch.cuda.current_stream()
P = zcomm._ptr


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


dx = torch.empty_like(x)
print(f"H2D 256 MiB: {count * 4 / timed(lambda: dx.copy_(hx, non_blocking=True)) / 1e6:.1f} GB/s")
print(f"D2H 256 MiB: {count * 4 / timed(lambda: hy.copy_(dx, non_blocking=True)) / 1e6:.1f} GB/s")
s2 = torch.cuda.Stream()


def both():
    dx.copy_(hx, non_blocking=True)
    with torch.cuda.stream(s2):
        hy.copy_(work, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


print(f"H2D || D2H 256 MiB each: {count * 4 / timed(both) / 1e6:.1f} GB/s per direction")
for gb in (1, 2, 4, 8, 16):
    def step():
        zcomm.check(L.zc_codec_roundtrip_host_f32(hx.data_ptr(), count, 2e-4, P(work), P(fr.stages), zcomm.STAGE_STRIDE,
                                                  abi.STAGE_BANK_BYTES, abi.PIN_AUTO, C.byref(hint), ctx.handle,
                                                  C.byref(cfg), P(fr.results), P(fr.index), P(err), hy.data_ptr(), gb,
                                                  C.c_void_p(s.cuda_stream)))
    ms = timed(step)
    print(f"e2e group_batches={gb:2d}: {ms:.3f} ms  {count * 4 / ms / 1e6:.1f} GB/s")
