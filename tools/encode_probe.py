"""Quick timing probe of the batched encoder/decoder (developer tool; not the bench)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_12396_b200 import abi, zcomm  # noqa: E402

count = int(os.environ.get("COUNT", 64 << 20))
L = zcomm.lib()
x = torch.randn(count, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
fr = zcomm.alloc_frames(count * 4, x.device)
err = torch.zeros(1, dtype=torch.int32, device="cuda")
hint, cfg = abi.make_hint(), zcomm.default_arb_config()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
P = zcomm._ptr
for name, pin in [("auto", abi.PIN_AUTO), ("fixedlen", abi.PIN_FIXEDLEN), ("raw", abi.PIN_RAW)]:
    def run():
        zcomm.check(L.zc_encode_batches_f32(P(x), count, 2e-4, P(fr.stages), zcomm.STAGE_STRIDE, abi.STAGE_BANK_BYTES,
                                            pin, C.byref(hint), None, C.byref(cfg), P(fr.results), P(fr.index), P(err), s))
    for _ in range(3):
        run()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        run()
    b.record()
    torch.cuda.synchronize()
    print(f"clusters={os.environ.get('ZC_ENCODE_CLUSTERS', 'default')} {name:9s} encode {a.elapsed_time(b) / 10 * 1e3:8.1f} us")
