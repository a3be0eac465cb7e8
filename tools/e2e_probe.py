"""Developer probe: PCIe copy rates and the host-buffer round trip at several group sizes."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_12396_b200 import abi, zcomm  # noqa: E402

count = 64 << 20
L = zcomm.lib()
x = torch.randn(count, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
hx = torch.empty(count, pin_memory=True)
hx.copy_(x.cpu())
hy = torch.empty(count, pin_memory=True)
d = torch.empty_like(x)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


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


def both():
    ev = torch.cuda.Event()
    ev.record()
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d.copy_(hx, non_blocking=True)
    with torch.cuda.stream(s2):
        hy.copy_(x, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


gb = count * 4 / 1e9
t = timed(lambda: d.copy_(hx, non_blocking=True))
print(f"H2D {gb / t * 1e3:.1f} GB/s")
t = timed(lambda: hy.copy_(x, non_blocking=True))
print(f"D2H {gb / t * 1e3:.1f} GB/s")
t = timed(both)
print(f"H2D+D2H concurrent: {2 * gb / t * 1e3:.1f} GB/s total ({t:.2f} ms)")
for cb in [1, 4, 16]:
    n = cb << 20
    def chunked():
        ev0 = torch.cuda.Event()
        ev0.record()
        s1.wait_event(ev0)
        s2.wait_event(ev0)
        for i in range(0, count, n):
            with torch.cuda.stream(s1):
                d[i:i + n].copy_(hx[i:i + n], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s1)
            s2.wait_event(e)
            with torch.cuda.stream(s2):
                hy[i:i + n].copy_(d[i:i + n], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    t = timed(chunked)
    print(f"chunked H2D->D2H copies, {cb * 4} MiB chunks: {t:.3f} ms ({gb / t * 1e3:.1f} GB/s per direction)")
prime = zcomm.eb_quantize_with_scale(x[: 1 << 20], 2e-4)
ctx = zcomm.HuffmanContext.from_bytes(prime)
fr = zcomm.alloc_frames(count * 4, x.device)
err = torch.zeros(1, dtype=torch.int32, device="cuda")
hint, cfg = abi.make_hint(), zcomm.default_arb_config()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
P = zcomm._ptr
for g in [1, 2, 4, 8, 16]:
    t = timed(lambda: zcomm.check(L.zc_codec_roundtrip_host_f32(hx.data_ptr(), count, 2e-4, P(d), P(fr.stages),
                                                                zcomm.STAGE_STRIDE, abi.STAGE_BANK_BYTES, abi.PIN_AUTO,
                                                                C.byref(hint), ctx.handle, C.byref(cfg), P(fr.results),
                                                                P(fr.index), P(err), hy.data_ptr(), g, s)))
    import time
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    zcomm.check(L.zc_codec_roundtrip_host_f32(hx.data_ptr(), count, 2e-4, P(d), P(fr.stages), zcomm.STAGE_STRIDE,
                                              abi.STAGE_BANK_BYTES, abi.PIN_AUTO, C.byref(hint), ctx.handle,
                                              C.byref(cfg), P(fr.results), P(fr.index), P(err), hy.data_ptr(), g, s))
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"roundtrip group={g:2d} batches: {t:.3f} ms  e2e {gb / t * 1e3:.1f} GB/s  host submit {1e3 * (h1 - h0):.3f} ms")
