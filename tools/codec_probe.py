"""Developer probe: one Auto-pinned encode + decode of the C1 workload (64 Mi Gaussian fp32,
scale 2e-4) through the C-ABI, for ncu captures and quick timings.  Not the bench."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_12396_b200 import abi, zcomm  # noqa: E402

count = int(os.environ.get("COUNT", 64 << 20))
reps = int(os.environ.get("REPS", 10))
pins = os.environ.get("PINS", "auto,huffman").split(",")
L = zcomm.lib()
x = torch.randn(count, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
prime = zcomm.eb_quantize_with_scale(x[: 1 << 20], 2e-4)
ctx = zcomm.HuffmanContext.from_bytes(prime)
fr = zcomm.alloc_frames(count * 4, x.device)
out = torch.empty_like(x)
err = torch.zeros(1, dtype=torch.int32, device="cuda")
codecs = torch.zeros(fr.nbatches, dtype=torch.int32, device="cuda")
hint, cfg = abi.make_hint(), zcomm.default_arb_config()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
P = zcomm._ptr
PIN = {"auto": abi.PIN_AUTO, "fixedlen": abi.PIN_FIXEDLEN, "raw": abi.PIN_RAW, "huffman": abi.PIN_HUFFMAN}


def enc(pin):
    zcomm.check(L.zc_encode_batches_f32(P(x), count, 2e-4, P(fr.stages), zcomm.STAGE_STRIDE, abi.STAGE_BANK_BYTES,
                                        pin, C.byref(hint), ctx.handle, C.byref(cfg), P(fr.results), P(fr.index),
                                        P(err), s))


def dec():
    zcomm.check(L.zc_decode_batches_f32(P(fr.stages), zcomm.STAGE_STRIDE, abi.STAGE_BANK_BYTES, P(fr.results), count,
                                        2e-4, ctx.handle, P(fr.index), P(out), P(codecs), s))


for name in pins:
    pin = PIN[name]
    for _ in range(2):
        enc(pin)
        dec()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    te = td = 0.0
    for _ in range(reps):
        ev[0].record()
        enc(pin)
        ev[1].record()
        dec()
        ev[2].record()
        torch.cuda.synchronize()
        te += ev[0].elapsed_time(ev[1])
        td += ev[1].elapsed_time(ev[2])
    res = fr.encode_results()
    pay = sum(r.payload_bytes for r in res)
    e = int(err.item())
    ok = bool(((out.double() - x.double()).abs().max() <= 1e-4 * (1 + 1e-9) + x.abs().max().double() * 2**-24).item())
    print(f"{name:9s} encode {te / reps * 1e3:8.1f} us  decode {td / reps * 1e3:8.1f} us  CR {count * 4 / pay:.4f}  "
          f"err=0x{e:x} bound_ok={ok}")
