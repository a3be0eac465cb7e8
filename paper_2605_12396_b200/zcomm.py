"""Python face of libzcomm_b200.so — the zcomm API (/root/reference/proj/core/include/zcomm/)
over the C-ABI in include/zcomm_b200.h, with torch CUDA tensors as device memory.

Names, argument meaning and error behaviour follow the reference:

* ``std::invalid_argument`` -> :class:`ValueError`, ``std::overflow_error`` -> :class:`OverflowError`,
  ``std::runtime_error`` -> :class:`RuntimeError`, ``std::logic_error`` -> :class:`AssertionError`,
  ``LinkPoisoned`` -> :class:`LinkPoisoned` (a :class:`RuntimeError`).
* codec "failure sentinels" stay values: encoders return payload size 0, decoders return False.

Every compute call runs sm_100a kernels; there is no CPU fallback.  The library is loaded on first
use and a missing library or GPU raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Sequence

import torch

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libzcomm_b200.so")
P = C.POINTER
vp = C.c_void_p


class LinkPoisoned(RuntimeError):
    """A peer aborted the collective (transport.hpp:50-52)."""


class CudaError(RuntimeError):
    """CUDA launch/runtime failure (no device, bad pointer, ...)."""


_EXC = {abi.ERR_INVALID_ARGUMENT: ValueError, abi.ERR_OVERFLOW: OverflowError, abi.ERR_RUNTIME: RuntimeError,
        abi.ERR_LOGIC: AssertionError, abi.ERR_CUDA: CudaError, abi.ERR_PEER: LinkPoisoned}

_lib = None


def build(verbose: bool = False) -> str:
    """Compile the CUDA library in-tree (nvcc, sm_100a)."""
    out = subprocess.run(["make", "-s", "-j8", "-C", os.path.join(HERE, "csrc")], capture_output=not verbose, text=True)
    if out.returncode != 0:
        raise RuntimeError("libzcomm_b200 build failed:\n" + (out.stdout or "") + (out.stderr or ""))
    return LIB_PATH


def _sig(L, name, restype, *args):
    f = getattr(L, name)
    f.restype = restype
    f.argtypes = list(args)


def lib():
    """The loaded C library (raises if it was never built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run paper_2605_12396_b200.zcomm.build() (no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    u64, i32, u32, dbl = C.c_uint64, C.c_int32, C.c_uint32, C.c_double
    _sig(L, "zc_last_error", C.c_char_p)
    _sig(L, "zc_version", C.c_char_p)
    _sig(L, "zc_launch_count", C.c_uint64)
    _sig(L, "zc_device_count", C.c_int, P(C.c_int))
    _sig(L, "zc_device_malloc", C.c_int, u64, P(vp))
    _sig(L, "zc_device_free", None, vp)
    _sig(L, "zc_memcpy", C.c_int, vp, vp, u64)
    _sig(L, "zc_memset", C.c_int, vp, C.c_int, u64)
    _sig(L, "zc_stream_synchronize", C.c_int, vp)
    _sig(L, "zc_flush_deferred", None)
    _sig(L, "zc_default_arb_config", None, P(abi.ArbConfig))
    _sig(L, "zc_default_transport_hint", None, P(abi.TransportHint))
    _sig(L, "zc_default_collective_config", None, P(abi.CollectiveConfig))
    _sig(L, "zc_load_arbitration_config", C.c_int, C.c_char_p, P(abi.ArbConfig))
    _sig(L, "zc_apply_env_overrides", C.c_int, P(abi.ArbConfig))
    _sig(L, "zc_write_header", C.c_int, P(abi.FrameHeader), vp, u64)
    _sig(L, "zc_parse_header", C.c_int, vp, u64, P(abi.FrameHeader))
    _sig(L, "zc_validate_header", C.c_int, P(abi.FrameHeader), u64)
    _sig(L, "zc_frame_commit_raw", C.c_int, vp, u64, vp, u64, vp, vp)
    _sig(L, "zc_absmax_f32", C.c_int, vp, u64, vp, vp, vp)
    _sig(L, "zc_absmax_f64", C.c_int, vp, u64, vp, vp, vp)
    _sig(L, "zc_eb_quantize_f32", C.c_int, vp, u64, dbl, vp, vp, vp)
    _sig(L, "zc_eb_quantize_f64", C.c_int, vp, u64, dbl, vp, vp, vp)
    _sig(L, "zc_eb_quantize_rel_f32", C.c_int, vp, u64, dbl, vp, P(dbl), vp)
    _sig(L, "zc_dequantize_f64", C.c_int, vp, u64, i32, dbl, u32, vp, vp)
    _sig(L, "zc_dequantize_f32", C.c_int, vp, u64, i32, dbl, u32, vp, vp)
    _sig(L, "zc_mt19937_64", C.c_int, u64, u64, u64, vp, vp)
    _sig(L, "zc_qsgd_quantize_chunk_f32", C.c_int, vp, u64, u32, dbl, u64, u64, vp, vp)
    _sig(L, "zc_qsgd_norm_f32", C.c_int, vp, u64, vp, vp, vp)
    _sig(L, "zc_qsgd_quantize_f32", C.c_int, vp, u64, u32, u64, vp, P(dbl), vp)
    _sig(L, "zc_comm_allreduce_qsgd_f32", C.c_int, vp, vp, vp, i32, u64, u32, u64, vp)
    _sig(L, "zc_fixedlen_encode", C.c_int, vp, u64, vp, u64, vp, vp, vp)
    _sig(L, "zc_fixedlen_decode", C.c_int, P(abi.FrameHeader), vp, u64, vp, u64, vp, vp)
    _sig(L, "zc_huff_ctx_create", C.c_int, vp, P(vp))
    _sig(L, "zc_huff_ctx_create_from_bytes", C.c_int, vp, u64, P(vp))
    _sig(L, "zc_huff_ctx_create_from_device_bytes", C.c_int, vp, u64, P(vp), vp)
    _sig(L, "zc_huff_ctx_from_lengths", C.c_int, vp, P(vp))
    _sig(L, "zc_huff_ctx_valid", C.c_int, vp)
    _sig(L, "zc_huff_ctx_code_lengths", C.c_int, vp, vp)
    _sig(L, "zc_huff_ctx_codes", C.c_int, vp, vp, vp)
    _sig(L, "zc_huff_ctx_destroy", None, vp)
    _sig(L, "zc_huffman_expected_code_len", C.c_int, vp, vp, P(dbl), P(i32))
    _sig(L, "zc_huffman_self_code_len", C.c_int, vp, P(dbl), P(i32))
    _sig(L, "zc_huffman_encode", C.c_int, vp, u64, vp, vp, u64, i32, vp, vp, vp)
    _sig(L, "zc_huffman_decode", C.c_int, P(abi.FrameHeader), vp, u64, vp, vp, vp, u64, vp, vp)
    _sig(L, "zc_profile_sample", C.c_int, vp, u64, vp, vp, vp)
    _sig(L, "zc_predict_payload", u64, i32, u64, P(abi.SampleStats), P(abi.ArbConfig))
    _sig(L, "zc_arbitrate_plan", C.c_int, u64, u64, P(abi.SampleStats), P(abi.TransportHint), vp, P(abi.ArbConfig),
         P(abi.ArbitrationPlan))
    _sig(L, "zc_encode_best", C.c_int, vp, u64, vp, u64, P(abi.TransportHint), vp, P(abi.ArbConfig), vp, vp)
    _sig(L, "zc_encode_batches_sym", C.c_int, vp, u64, vp, u64, u64, i32, P(abi.TransportHint), vp, P(abi.ArbConfig),
         vp, vp, vp, vp)
    _sig(L, "zc_encode_batches_f32", C.c_int, vp, u64, dbl, vp, u64, u64, i32, P(abi.TransportHint), vp,
         P(abi.ArbConfig), vp, vp, vp, vp)
    _sig(L, "zc_decode_batches_sym", C.c_int, vp, u64, u64, vp, u64, vp, vp, vp, vp, vp)
    _sig(L, "zc_decode_batches_f32", C.c_int, vp, u64, u64, vp, u64, dbl, vp, vp, vp, vp, vp)
    _sig(L, "zc_decode_batches_add_sym", C.c_int, vp, u64, u64, vp, u64, vp, vp, vp, vp, vp)
    _sig(L, "zc_codec_roundtrip_host_f32", C.c_int, vp, u64, dbl, vp, vp, u64, u64, i32, P(abi.TransportHint), vp,
         P(abi.ArbConfig), vp, vp, vp, vp, u32, vp)
    _sig(L, "zc_comm_create", C.c_int, C.c_int, C.c_int, C.c_int, P(abi.CollectiveConfig), P(vp))
    _sig(L, "zc_comm_export_size", C.c_int)
    _sig(L, "zc_comm_export", C.c_int, vp, vp)
    _sig(L, "zc_comm_connect", C.c_int, vp, vp)
    _sig(L, "zc_comm_create_group", C.c_int, C.c_int, P(C.c_int), P(abi.CollectiveConfig), P(vp))
    _sig(L, "zc_comm_destroy", None, vp)
    _sig(L, "zc_comm_rank", C.c_int, vp)
    _sig(L, "zc_comm_nranks", C.c_int, vp)
    _sig(L, "zc_comm_set_shared_huffman", C.c_int, vp, vp)
    _sig(L, "zc_comm_allreduce_sym", C.c_int, vp, vp, u64, i32, P(dbl), u32, vp)
    _sig(L, "zc_comm_allreduce_eb_f32", C.c_int, vp, vp, vp, i32, u64, dbl, vp)
    _sig(L, "zc_comm_reduce_scatter_sym", C.c_int, vp, vp, u64, vp)
    _sig(L, "zc_comm_allgather_sym", C.c_int, vp, vp, u64, vp)
    _sig(L, "zc_comm_allreduce_max", C.c_int, vp, dbl, P(dbl), vp)
    _sig(L, "zc_comm_sync", C.c_int, vp)
    _sig(L, "zc_comm_reset", C.c_int, vp)
    _sig(L, "zc_comm_send_encoded", C.c_int, vp, i32, vp, u64, vp)
    _sig(L, "zc_comm_recv_decoded", C.c_int, vp, i32, vp, u64, vp)
    _sig(L, "zc_comm_abort", C.c_int, vp)
    _sig(L, "zc_comm_wire_stats", C.c_int, vp, P(abi.WireStats))
    _sig(L, "zc_comm_reset_stats", C.c_int, vp)
    _sig(L, "zc_group_allreduce_sym", C.c_int, P(vp), C.c_int, P(vp), u64, i32, P(dbl), u32)
    _sig(L, "zc_group_allreduce_eb_f32", C.c_int, P(vp), C.c_int, P(vp), P(vp), i32, u64, dbl)
    _sig(L, "zc_group_reduce_scatter_sym", C.c_int, P(vp), C.c_int, P(vp), u64)
    _sig(L, "zc_group_allgather_sym", C.c_int, P(vp), C.c_int, P(vp), u64)
    _sig(L, "zc_group_allreduce_max", C.c_int, P(vp), C.c_int, P(dbl), P(dbl))
    _sig(L, "zc_comm_alltoall_sym", C.c_int, vp, vp, vp, u64, vp)
    _sig(L, "zc_comm_broadcast_sym", C.c_int, vp, vp, u64, i32, vp)
    _sig(L, "zc_comm_group_execute", C.c_int, vp, P(abi.CollRequest), i32, vp)
    _sig(L, "zc_group_alltoall_sym", C.c_int, P(vp), C.c_int, P(vp), P(vp), u64)
    _sig(L, "zc_group_broadcast_sym", C.c_int, P(vp), C.c_int, P(vp), u64, i32)
    _sig(L, "zc_group_execute", C.c_int, P(vp), C.c_int, P(P(abi.CollRequest)), i32)
    _sig(L, "zc_comm_timeline_enable", C.c_int, vp, i32)
    _sig(L, "zc_comm_timeline_rows", C.c_int, vp, P(abi.TimelineRow), i32, P(i32))
    _sig(L, "zc_comm_timeline_origin_delta", C.c_int, vp, vp, P(dbl))
    _lib = L
    return L


def launch_count() -> int:
    """Kernels this library has launched so far in this process."""
    return int(lib().zc_launch_count())


def check(rc: int) -> None:
    if rc != abi.OK:
        msg = lib().zc_last_error().decode(errors="replace")
        raise _EXC.get(rc, RuntimeError)(msg)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t: torch.Tensor) -> None:
    if not t.is_cuda:
        raise ValueError("device tensor expected (the compute path is CUDA only)")


def _bytes(t: torch.Tensor) -> torch.Tensor:
    return t.contiguous().view(torch.uint8).reshape(-1)


# ------------------------------------------------------------------ config
def default_arb_config() -> abi.ArbConfig:
    c = abi.ArbConfig()
    lib().zc_default_arb_config(C.byref(c))
    return c


def load_arbitration_config(text: str, cfg: Optional[abi.ArbConfig] = None) -> abi.ArbConfig:
    """load_arbitration_config (rea.cpp:240-263)."""
    cfg = cfg or default_arb_config()
    check(lib().zc_load_arbitration_config(text.encode(), C.byref(cfg)))
    return cfg


def apply_env_overrides(cfg: abi.ArbConfig) -> abi.ArbConfig:
    """apply_env_overrides (rea.cpp:270-279)."""
    check(lib().zc_apply_env_overrides(C.byref(cfg)))
    return cfg


# ------------------------------------------------------------------ frame (frame.hpp:38-50)
def write_header(h: abi.FrameHeader, size: int = abi.HEADER_BYTES) -> bytes:
    buf = (C.c_uint8 * size)()
    check(lib().zc_write_header(C.byref(h), C.cast(buf, vp), size))
    return bytes(buf)


def parse_header(src: bytes) -> Optional[abi.FrameHeader]:
    if len(src) < abi.HEADER_BYTES:
        return None
    buf = (C.c_uint8 * len(src)).from_buffer_copy(src)
    h = abi.FrameHeader()
    check(lib().zc_parse_header(C.cast(buf, vp), len(src), C.byref(h)))
    return h


def validate_header(h: abi.FrameHeader, region: int) -> bool:
    return lib().zc_validate_header(C.byref(h), region) == 1


def frame_commit_raw(raw: torch.Tensor, region: torch.Tensor) -> int:
    raw, region = _bytes(raw), _bytes(region)
    tot = torch.zeros(1, dtype=torch.int64, device=raw.device)
    check(lib().zc_frame_commit_raw(_ptr(raw), raw.numel(), _ptr(region), region.numel(), _ptr(tot), _stream()))
    return int(tot.item())


# ------------------------------------------------------------------ quant (quant.hpp:29-53)
def _err_word(device) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device)


def _raise_derr(e: int, where: str) -> None:
    if e & abi.DERR_NONFINITE:
        raise ValueError(f"{where}: non-finite input")
    if e & abi.DERR_RANGE:
        raise ValueError("quantize: bin index exceeds int32 range")
    if e:
        raise RuntimeError(f"{where}: device error 0x{e:x}")


def eb_quantize_with_scale(x: torch.Tensor, scale: float) -> torch.Tensor:
    """eb_quantize_with_scale (quant.cpp:43-52): symbols = llround(x / scale)."""
    _dev(x)
    x = x.contiguous()
    sym = torch.empty(x.numel(), dtype=torch.int32, device=x.device)
    err = _err_word(x.device)
    fn = lib().zc_eb_quantize_f64 if x.dtype == torch.float64 else lib().zc_eb_quantize_f32
    if x.dtype not in (torch.float32, torch.float64):
        raise ValueError("eb_quantize: float32 or float64 input")
    check(fn(_ptr(x), x.numel(), float(scale), _ptr(sym), _ptr(err), _stream()))
    _raise_derr(int(err.item()), "eb_quantize_with_scale")
    return sym


def eb_quantize(x: torch.Tensor, rel: float):
    """eb_quantize (quant.cpp:30-41): returns (symbols, scale)."""
    _dev(x)
    x = x.contiguous().float()
    sym = torch.empty(x.numel(), dtype=torch.int32, device=x.device)
    scale = C.c_double()
    check(lib().zc_eb_quantize_rel_f32(_ptr(x), x.numel(), float(rel), _ptr(sym), C.byref(scale), _stream()))
    return sym, scale.value


def mt19937_64(seed: int, n: int, skip: int = 0, device=None) -> torch.Tensor:
    """std::mt19937_64(seed) draws skip .. skip+n-1, generated on the device (uint64 as int64)."""
    out = torch.empty(max(n, 1), dtype=torch.int64, device=device or "cuda")
    check(lib().zc_mt19937_64(seed, skip, n, _ptr(out), _stream()))
    return out[:n]


def qsgd_quantize(x: torch.Tensor, levels: int, seed: int):
    """qsgd_quantize (quant.cpp:84-98): returns (symbols, scale = norm or 1)."""
    _dev(x)
    x = x.contiguous().float()
    sym = torch.empty(max(x.numel(), 1), dtype=torch.int32, device=x.device)
    sc = C.c_double()
    check(lib().zc_qsgd_quantize_f32(_ptr(x), x.numel(), levels, seed, _ptr(sym), C.byref(sc), _stream()))
    return sym[:x.numel()], sc.value


def qsgd_quantize_chunk(x: torch.Tensor, levels: int, norm: float, seed: int, skip: int = 0) -> torch.Tensor:
    """qsgd_quantize_chunk (quant.cpp:64-82) with rng = mt19937_64(seed) after `skip` draws."""
    _dev(x)
    x = x.contiguous().float()
    sym = torch.empty(max(x.numel(), 1), dtype=torch.int32, device=x.device)
    check(lib().zc_qsgd_quantize_chunk_f32(_ptr(x), x.numel(), levels, float(norm), seed, skip, _ptr(sym), _stream()))
    return sym[:x.numel()]


def absmax(x: torch.Tensor) -> float:
    _dev(x)
    x = x.contiguous()
    out = torch.zeros(1, dtype=torch.float64, device=x.device)
    err = _err_word(x.device)
    fn = lib().zc_absmax_f64 if x.dtype == torch.float64 else lib().zc_absmax_f32
    check(fn(_ptr(x), x.numel(), _ptr(out), _ptr(err), _stream()))
    _raise_derr(int(err.item()), "absmax")
    return float(out.item())


def dequantize(sym: torch.Tensor, mode: int = abi.QUANT_ERROR_BOUNDED, scale: float = 1.0, levels: int = 0,
               dtype=torch.float64) -> torch.Tensor:
    """dequantize_into (quant.cpp:107-127); float64 output is bit-exact with the reference."""
    _dev(sym)
    sym = sym.contiguous()
    out = torch.empty(sym.numel(), dtype=dtype, device=sym.device)
    fn = lib().zc_dequantize_f64 if dtype == torch.float64 else lib().zc_dequantize_f32
    check(fn(_ptr(sym), sym.numel(), mode, float(scale), levels, _ptr(out), _stream()))
    return out


# ------------------------------------------------------------------ fixedlen (fixedlen.hpp:22-42)
def fixedlen_encode(sym: torch.Tensor, out_cap: int):
    """fixedlen_encode (fixedlen.cpp:15-37): returns (payload bytes tensor, width); size 0 = failure."""
    _dev(sym)
    sym = sym.contiguous()
    out = torch.zeros(max(out_cap, 16), dtype=torch.uint8, device=sym.device)
    pay = torch.zeros(1, dtype=torch.int64, device=sym.device)
    w = torch.zeros(1, dtype=torch.int32, device=sym.device)
    check(lib().zc_fixedlen_encode(_ptr(sym), sym.numel(), _ptr(out), out_cap, _ptr(pay), _ptr(w), _stream()))
    n = int(pay.item())
    return out[:n], int(w.item())


def fixedlen_decode(h: abi.FrameHeader, payload: torch.Tensor, dst_len: int):
    """fixedlen_decode_into (fixedlen.cpp:39-65): returns (ok, dst bytes)."""
    payload = _aligned_copy(payload)
    dst = torch.zeros(max(dst_len, 16), dtype=torch.uint8, device=payload.device)
    ok = torch.zeros(1, dtype=torch.int32, device=payload.device)
    check(lib().zc_fixedlen_decode(C.byref(h), _ptr(payload), payload.numel(), _ptr(dst), dst_len, _ptr(ok), _stream()))
    return bool(ok.item()), dst[:dst_len]


def _aligned_copy(t: torch.Tensor) -> torch.Tensor:
    t = _bytes(t)
    if t.data_ptr() % 16 == 0:
        return t
    return t.clone()


# ------------------------------------------------------------------ huffman (huffman.hpp:38-70)
class HuffmanContext:
    """HuffmanContext (huffman.hpp:20-33): immutable canonical code; tables live in HBM."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def from_hist(cls, hist256) -> "HuffmanContext":
        """huffman_build_context (huffman.cpp:165-173)."""
        arr = (C.c_uint64 * 256)(*[int(v) for v in hist256])
        h = vp()
        check(lib().zc_huff_ctx_create(C.cast(arr, vp), C.byref(h)))
        return cls(h)

    @classmethod
    def from_bytes(cls, sample) -> "HuffmanContext":
        """set_shared_huffman_from_bytes' +1-smoothed context (collectives.cpp:99-106)."""
        if isinstance(sample, torch.Tensor) and sample.is_cuda:
            s = _bytes(sample)
            h = vp()
            check(lib().zc_huff_ctx_create_from_device_bytes(_ptr(s), s.numel(), C.byref(h), _stream()))
            return cls(h)
        b = bytes(sample.cpu().numpy().tobytes() if isinstance(sample, torch.Tensor) else sample)
        buf = (C.c_uint8 * max(len(b), 1)).from_buffer_copy(b or b"\0")
        h = vp()
        check(lib().zc_huff_ctx_create_from_bytes(C.cast(buf, vp), len(b), C.byref(h)))
        return cls(h)

    @classmethod
    def from_lengths(cls, lens256) -> Optional["HuffmanContext"]:
        """huffman_context_from_lengths (huffman.cpp:175-180); None for an invalid length set."""
        arr = (C.c_uint8 * 256)(*[int(v) for v in lens256])
        h = vp()
        rc = lib().zc_huff_ctx_from_lengths(C.cast(arr, vp), C.byref(h))
        if rc == abi.ERR_INVALID_ARGUMENT:
            return None
        check(rc)
        return cls(h)

    @property
    def valid(self) -> bool:
        return lib().zc_huff_ctx_valid(self._h) == 1

    @property
    def code_lengths(self) -> list:
        arr = (C.c_uint8 * 256)()
        check(lib().zc_huff_ctx_code_lengths(self._h, C.cast(arr, vp)))
        return list(arr)

    def codes(self):
        code = (C.c_uint32 * 256)()
        rev = (C.c_uint32 * 256)()
        check(lib().zc_huff_ctx_codes(self._h, C.cast(code, vp), C.cast(rev, vp)))
        return list(code), list(rev)

    def expected_code_len(self, hist256) -> Optional[float]:
        arr = (C.c_uint64 * 256)(*[int(v) for v in hist256])
        bits, valid = C.c_double(), C.c_int32()
        check(lib().zc_huffman_expected_code_len(self._h, C.cast(arr, vp), C.byref(bits), C.byref(valid)))
        return bits.value if valid.value else None

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if self._h and _lib is not None:
                _lib.zc_huff_ctx_destroy(self._h)
        except Exception:
            pass


def huffman_self_code_len(hist256) -> Optional[float]:
    arr = (C.c_uint64 * 256)(*[int(v) for v in hist256])
    bits, valid = C.c_double(), C.c_int32()
    check(lib().zc_huffman_self_code_len(C.cast(arr, vp), C.byref(bits), C.byref(valid)))
    return bits.value if valid.value else None


def huffman_encode(raw: torch.Tensor, ctx: HuffmanContext, out_cap: int, embed: bool = False, with_index=False):
    """huffman_encode (huffman.cpp:216-246): returns payload (size 0 = failure) [, companion index]."""
    raw = _bytes(raw)
    out = torch.zeros(max(out_cap, 16), dtype=torch.uint8, device=raw.device)
    pay = torch.zeros(1, dtype=torch.int64, device=raw.device)
    nidx = max(1, (raw.numel() + abi.HUFF_INDEX_GRAIN - 1) // abi.HUFF_INDEX_GRAIN)
    idx = torch.zeros(nidx, dtype=torch.int32, device=raw.device) if with_index else None
    check(lib().zc_huffman_encode(_ptr(raw), raw.numel(), ctx.handle, _ptr(out), out_cap, int(embed), _ptr(pay),
                                  _ptr(idx), _stream()))
    n = int(pay.item())
    return (out[:n], idx) if with_index else out[:n]


def huffman_decode(h: abi.FrameHeader, payload: torch.Tensor, ctx: Optional[HuffmanContext], dst_len: int,
                   index: Optional[torch.Tensor] = None):
    """huffman_decode_into (huffman.cpp:248-316): returns (ok, dst bytes)."""
    payload = _aligned_copy(payload)
    dst = torch.zeros(max(dst_len, 16), dtype=torch.uint8, device=payload.device)
    ok = torch.zeros(1, dtype=torch.int32, device=payload.device)
    check(lib().zc_huffman_decode(C.byref(h), _ptr(payload), payload.numel(), ctx.handle if ctx else None,
                                  _ptr(index), _ptr(dst), dst_len, _ptr(ok), _stream()))
    return bool(ok.item()), dst[:dst_len]


# ------------------------------------------------------------------ rea (rea.hpp:114-133)
def profile_sample(raw: torch.Tensor, ctx: Optional[HuffmanContext] = None) -> abi.SampleStats:
    """profile_sample (rea.cpp:93-118), computed on device."""
    raw = _bytes(raw)
    d = torch.zeros(C.sizeof(abi.SampleStats), dtype=torch.uint8, device=raw.device)
    check(lib().zc_profile_sample(_ptr(raw), raw.numel(), ctx.handle if ctx else None, _ptr(d), _stream()))
    return abi.SampleStats.from_buffer_copy(d.cpu().numpy().tobytes())


def predict_payload(codec: int, raw_bytes: int, stats: abi.SampleStats, cfg: Optional[abi.ArbConfig] = None) -> int:
    return lib().zc_predict_payload(codec, raw_bytes, C.byref(stats), C.byref(cfg or default_arb_config()))


def arbitrate_plan(raw_bytes: int, payload_cap: int, stats: abi.SampleStats, hint: Optional[abi.TransportHint] = None,
                   ctx: Optional[HuffmanContext] = None, cfg: Optional[abi.ArbConfig] = None) -> abi.ArbitrationPlan:
    plan = abi.ArbitrationPlan()
    check(lib().zc_arbitrate_plan(raw_bytes, payload_cap, C.byref(stats), C.byref(hint or abi.make_hint()),
                                  ctx.handle if ctx else None, C.byref(cfg or default_arb_config()), C.byref(plan)))
    return plan


def _result(d: torch.Tensor, n: int = 1):
    raw = d.cpu().numpy().tobytes()
    sz = C.sizeof(abi.EncodeResult)
    return [abi.EncodeResult.from_buffer_copy(raw[i * sz:(i + 1) * sz]) for i in range(n)]


def encode_best(raw: torch.Tensor, stage_len: int = abi.STAGE_BANK_BYTES, hint: Optional[abi.TransportHint] = None,
                ctx: Optional[HuffmanContext] = None, cfg: Optional[abi.ArbConfig] = None):
    """encode_best (rea.cpp:178-238): returns (EncodeResult, frame bytes tensor)."""
    raw = _bytes(raw)
    stage = torch.zeros(max(stage_len, 16), dtype=torch.uint8, device=raw.device)
    res = torch.zeros(C.sizeof(abi.EncodeResult), dtype=torch.uint8, device=raw.device)
    check(lib().zc_encode_best(_ptr(raw), raw.numel(), _ptr(stage), stage_len, C.byref(hint or abi.make_hint()),
                               ctx.handle if ctx else None, C.byref(cfg or default_arb_config()), _ptr(res), _stream()))
    r = _result(res)[0]
    return r, stage[: r.total_bytes]


# ------------------------------------------------------------------ batched hot path
STAGE_STRIDE = (abi.STAGE_BANK_BYTES + 255) // 256 * 256


@dataclass
class Frames:
    """Encoded 4 MiB batches of one message: stages (one frame each), results, companion index."""
    stages: torch.Tensor      # uint8 [nbatches * STAGE_STRIDE]
    results: torch.Tensor     # raw zc_encode_result array (uint8)
    index: torch.Tensor       # int32 [nbatches * HUFF_INDEX_ENTRIES]
    raw_bytes: int
    nbatches: int

    def encode_results(self):
        return _result(self.results, self.nbatches)

    def frame(self, b: int) -> torch.Tensor:
        r = self.encode_results()[b]
        return self.stages[b * STAGE_STRIDE: b * STAGE_STRIDE + r.total_bytes]

    def payload_bytes(self) -> int:
        return sum(r.payload_bytes for r in self.encode_results())


def alloc_frames(raw_bytes: int, device) -> Frames:
    nb = (raw_bytes + abi.BATCH_RAW_BYTES - 1) // abi.BATCH_RAW_BYTES
    return Frames(stages=torch.empty(max(nb, 1) * STAGE_STRIDE, dtype=torch.uint8, device=device),
                  results=torch.zeros(max(nb, 1) * C.sizeof(abi.EncodeResult), dtype=torch.uint8, device=device),
                  index=torch.zeros(max(nb, 1) * abi.HUFF_INDEX_ENTRIES, dtype=torch.int32, device=device),
                  raw_bytes=raw_bytes, nbatches=nb)


def encode_batches(src: torch.Tensor, pin: int = abi.PIN_AUTO, scale: Optional[float] = None,
                   hint: Optional[abi.TransportHint] = None, ctx: Optional[HuffmanContext] = None,
                   cfg: Optional[abi.ArbConfig] = None, frames: Optional[Frames] = None,
                   err: Optional[torch.Tensor] = None) -> Frames:
    """send_encoded over a message (collectives.cpp:350-356, 201-302), all batches in one launch.

    ``src`` is either int32 symbols (raw bytes of any tensor) or float32 data with ``scale`` given,
    in which case quantization is fused into the encoder (symbols never reach HBM)."""
    _dev(src)
    src = src.contiguous()
    own_err = err is None
    err = _err_word(src.device) if own_err else err
    L = lib()
    if scale is not None:
        if src.dtype != torch.float32:
            raise ValueError("fused quantize+encode takes float32 input")
        frames = frames or alloc_frames(src.numel() * 4, src.device)
        check(L.zc_encode_batches_f32(_ptr(src), src.numel(), float(scale), _ptr(frames.stages), STAGE_STRIDE,
                                      abi.STAGE_BANK_BYTES, pin, C.byref(hint or abi.make_hint()),
                                      ctx.handle if ctx else None, C.byref(cfg or default_arb_config()),
                                      _ptr(frames.results), _ptr(frames.index), _ptr(err), _stream()))
    else:
        raw = _bytes(src)
        frames = frames or alloc_frames(raw.numel(), src.device)
        check(L.zc_encode_batches_sym(_ptr(raw), raw.numel(), _ptr(frames.stages), STAGE_STRIDE, abi.STAGE_BANK_BYTES,
                                      pin, C.byref(hint or abi.make_hint()), ctx.handle if ctx else None,
                                      C.byref(cfg or default_arb_config()), _ptr(frames.results),
                                      _ptr(frames.index), _ptr(err), _stream()))
    if own_err:
        e = int(err.item())
        _raise_derr(e & (abi.DERR_NONFINITE | abi.DERR_RANGE), "encode")
        if e & abi.DERR_CAPACITY:
            raise RuntimeError("staging capacity exhausted; batch cannot ship even raw")
    return frames


def decode_batches(frames: Frames, ctx: Optional[HuffmanContext] = None, scale: Optional[float] = None,
                   out: Optional[torch.Tensor] = None, use_index: bool = True, codecs: Optional[torch.Tensor] = None):
    """recv_decoded over a message (collectives.cpp:304-348): int32 symbols, or fp32 with ``scale``."""
    L = lib()
    dev = frames.stages.device
    idx = frames.index if use_index else None
    if scale is None:
        out = out if out is not None else torch.empty((frames.raw_bytes + 3) // 4, dtype=torch.int32, device=dev)
        check(L.zc_decode_batches_sym(_ptr(frames.stages), STAGE_STRIDE, abi.STAGE_BANK_BYTES, _ptr(frames.results),
                                      frames.raw_bytes, ctx.handle if ctx else None, _ptr(idx), _ptr(out),
                                      _ptr(codecs), _stream()))
    else:
        n = frames.raw_bytes // 4
        out = out if out is not None else torch.empty(n, dtype=torch.float32, device=dev)
        check(L.zc_decode_batches_f32(_ptr(frames.stages), STAGE_STRIDE, abi.STAGE_BANK_BYTES, _ptr(frames.results),
                                      n, float(scale), ctx.handle if ctx else None, _ptr(idx), _ptr(out),
                                      _ptr(codecs), _stream()))
    return out


# ------------------------------------------------------------------ collectives (collectives.hpp:48-153)
def _wire(handle) -> abi.WireStats:
    w = abi.WireStats()
    check(lib().zc_comm_wire_stats(handle, C.byref(w)))
    return w


def collective_config(pin: int = abi.PIN_AUTO, **kw) -> abi.CollectiveConfig:
    c = abi.CollectiveConfig()
    lib().zc_default_collective_config(C.byref(c))
    c.pin = pin
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def _timeline_rows(h):
    n = C.c_int32(0)
    check(lib().zc_comm_timeline_rows(h, None, 0, C.byref(n)))
    arr = (abi.TimelineRow * max(n.value, 1))()
    check(lib().zc_comm_timeline_rows(h, arr, n.value, C.byref(n)))
    return list(arr[:n.value])


def _request(q: dict) -> abi.CollRequest:
    """A CollectiveRequest (collectives.hpp:94-101) from a dict: op, sym (int32 tensor), and per op
    recv (AllGather: nranks*block, AllToAll: like sym), root (Broadcast), scale/mode/levels
    (AllReduce).  count: the block (AllGather/AllToAll per-rank block) or the symbol count."""
    op = q["op"]
    sym = q.get("sym")
    recv = q.get("recv")
    count = q.get("count")
    if count is None:
        count = 0 if sym is None else (sym.numel() if op != abi.COLL_ALLTOALL else sym.numel() // q["nranks"])
    return abi.CollRequest(op, q.get("root", 0), q.get("mode", abi.QUANT_ERROR_BOUNDED), q.get("levels", 0),
                           None if sym is None else sym.data_ptr(), None if recv is None else recv.data_ptr(),
                           count, float(q.get("scale", 1.0)))


class Group:
    """A single-process Communicator (collectives.cpp:66-190): nranks ranks on local devices
    (several ranks may share one GPU), every collective runs all ranks concurrently, like the
    reference's thread-per-rank ``Communicator::run``."""

    def __init__(self, nranks: int, devices: Optional[Sequence[int]] = None,
                 cfg: Optional[abi.CollectiveConfig] = None):
        self.nranks = nranks
        self.devices = list(devices) if devices is not None else [torch.cuda.current_device()] * nranks
        self.cfg = cfg or collective_config()
        arr = (vp * nranks)()
        devs = (C.c_int * nranks)(*self.devices)
        check(lib().zc_comm_create_group(nranks, devs, C.byref(self.cfg), arr))
        self._h = arr

    def set_shared_huffman(self, ctx: HuffmanContext) -> None:
        for r in range(self.nranks):
            check(lib().zc_comm_set_shared_huffman(self._h[r], ctx.handle))

    def run(self, fn):
        """Communicator::run (collectives.cpp:137-173): fn(RankCtx) on one thread per rank.  A rank
        whose body raises poisons every link (zc_comm_abort; peers blocked on it fail with
        LinkPoisoned), the communicator is reset, and the root cause is re-raised.  Returns the
        per-rank results."""
        import threading
        n = self.nranks
        res, errs = [None] * n, [None] * n

        def body(r):
            torch.cuda.set_device(self.devices[r])
            try:
                res[r] = fn(RankCtx(self, r))
            except BaseException as e:  # noqa: BLE001 - every rank's failure is collected
                errs[r] = e
                lib().zc_comm_abort(self._h[r])

        th = [threading.Thread(target=body, args=(r,)) for r in range(n)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        lib().zc_flush_deferred()  # frees queued while the rank threads were in collectives
        failed = [e for e in errs if e is not None]
        if failed:
            for r in range(n):
                lib().zc_comm_reset(self._h[r])
            root = next((e for e in failed if not isinstance(e, LinkPoisoned)), failed[0])
            raise root
        return res

    def set_shared_huffman_from_bytes(self, sample) -> None:
        self.set_shared_huffman(HuffmanContext.from_bytes(sample))

    def _ptrs(self, ts):
        return (vp * self.nranks)(*[t.data_ptr() for t in ts])

    def allreduce(self, syms: Sequence[torch.Tensor], scales: Sequence[float], mode: int = abi.QUANT_ERROR_BOUNDED,
                  levels: int = 0):
        """RankCtx::allreduce on every rank (in place); returns the reconciled scales."""
        sc = (C.c_double * self.nranks)(*scales)
        check(lib().zc_group_allreduce_sym(self._h, self.nranks, self._ptrs(syms), syms[0].numel(), mode, sc, levels))
        return list(sc)

    def allreduce_eb(self, xs: Sequence[torch.Tensor], rel: float, out_dtype=torch.float32,
                     outs: Optional[Sequence[torch.Tensor]] = None):
        outs = outs if outs is not None else [torch.empty(x.numel(), dtype=out_dtype, device=x.device) for x in xs]
        out_dtype = outs[0].dtype
        check(lib().zc_group_allreduce_eb_f32(self._h, self.nranks, self._ptrs(xs), self._ptrs(outs),
                                              1 if out_dtype == torch.float64 else 0, xs[0].numel(), float(rel)))
        return outs

    def reduce_scatter(self, syms: Sequence[torch.Tensor]):
        check(lib().zc_group_reduce_scatter_sym(self._h, self.nranks, self._ptrs(syms), syms[0].numel()))

    def allgather(self, blocks: Sequence[torch.Tensor]):
        n = self.nranks
        outs = []
        for r, b in enumerate(blocks):
            o = torch.zeros(n * b.numel(), dtype=torch.int32, device=b.device)
            o[r * b.numel():(r + 1) * b.numel()] = b
            outs.append(o)
        check(lib().zc_group_allgather_sym(self._h, n, self._ptrs(outs), blocks[0].numel()))
        return outs

    def alltoall(self, sends: Sequence[torch.Tensor]):
        """RankCtx::alltoall (collectives.cpp:546-567) on every rank: block j of rank r's send goes
        to rank j; returns each rank's received buffer."""
        n = self.nranks
        block = sends[0].numel() // n
        for t in sends:
            if t.numel() != block * n:
                raise ValueError("alltoall buffer must split evenly across ranks")
        outs = [torch.empty_like(t) for t in sends]
        check(lib().zc_group_alltoall_sym(self._h, n, self._ptrs(sends), self._ptrs(outs), block))
        return outs

    def broadcast(self, datas: Sequence[torch.Tensor], root: int):
        """RankCtx::broadcast (collectives.cpp:569-591) on every rank, in place."""
        check(lib().zc_group_broadcast_sym(self._h, self.nranks, self._ptrs(datas), datas[0].numel(), root))

    def group_execute(self, requests: Sequence[Sequence[dict]]):
        """group_execute (collectives.cpp:593-616): requests[r] is rank r's list; see
        make_requests.  Returns the requests with outputs (recv tensors, reconciled scales)."""
        n = self.nranks
        k = len(requests[0])
        arrs = [(abi.CollRequest * k)(*[_request(q) for q in requests[r]]) for r in range(n)]
        ptrs = (C.POINTER(abi.CollRequest) * n)(*[C.cast(a, C.POINTER(abi.CollRequest)) for a in arrs])
        check(lib().zc_group_execute(self._h, n, ptrs, k))
        for r in range(n):
            for i, q in enumerate(requests[r]):
                if q["op"] == abi.COLL_ALLREDUCE:
                    q["scale"] = arrs[r][i].scale
        return requests

    def allreduce_qsgd(self, xs: Sequence[torch.Tensor], levels: int, seeds: Sequence[int], out_dtype=torch.float64):
        """RankCtx::allreduce_qsgd (collectives.cpp:518-523) on every rank: qsgd_quantize per rank on
        the device, the group's compressed allreduce in QSGD mode, dequantize."""
        qs = [qsgd_quantize(x, levels, sd) for x, sd in zip(xs, seeds)]
        syms = [q[0] for q in qs]
        scales = self.allreduce(syms, [q[1] for q in qs], abi.QUANT_QSGD, levels)
        return [dequantize(s, abi.QUANT_QSGD, sc, levels, out_dtype) for s, sc in zip(syms, scales)]

    def timeline_enable(self, max_pieces: int = 4096) -> None:
        """Start recording the measured piece timeline on every rank (0 stops)."""
        for r in range(self.nranks):
            check(lib().zc_comm_timeline_enable(self._h[r], max_pieces))

    def timeline(self):
        """Measured BatchTimelineRows (pipeline.hpp:32-46) of everything sent since
        timeline_enable, one per 4 MiB batch: the sender's encode (its stores are the transfer over
        peer memory) joined with the receiver's wait / decode of the same piece (matched by the
        receiver's piece sequence number), all on rank 0's clock."""
        per = []
        for r in range(self.nranks):
            rows = _timeline_rows(self._h[r])
            d = C.c_double(0.0)
            if r:
                check(lib().zc_comm_timeline_origin_delta(self._h[0], self._h[r], C.byref(d)))
            per.append((rows, d.value))
        recv = {}
        for r, (rows, off) in enumerate(per):
            for x in rows:
                if x.kind == 1:
                    recv[(r, x.seq)] = (x.ready_sec + off, x.end_sec + off)
        out = []
        for r, (rows, off) in enumerate(per):
            for x in rows:
                if x.kind != 0:
                    continue
                dec = recv.get((x.peer, x.seq), (float("nan"), float("nan")))
                out.append(dict(rank=r, seq=x.seq, batch=x.batch, codec=x.codec, raw_bytes=x.raw_bytes,
                                total_bytes=x.total_bytes, enc_start_sec=x.start_sec + off,
                                enc_end_sec=x.end_sec + off, xfer_start_sec=x.start_sec + off,
                                xfer_end_sec=x.end_sec + off, dec_start_sec=dec[0], dec_end_sec=dec[1]))
        out.sort(key=lambda d: (d["enc_start_sec"], d["rank"], d["batch"]))
        return out

    def allreduce_max(self, vs: Sequence[float]):
        a = (C.c_double * self.nranks)(*vs)
        o = (C.c_double * self.nranks)()
        check(lib().zc_group_allreduce_max(self._h, self.nranks, a, o))
        return list(o)

    def wire_stats(self) -> abi.WireStats:
        """Communicator::wire_stats (collectives.cpp:175-186): summed over ranks."""
        agg = abi.WireStats()
        for r in range(self.nranks):
            w = _wire(self._h[r])
            for i in range(3):
                agg.frames_by_codec[i] += w.frames_by_codec[i]
            agg.raw_bytes += w.raw_bytes
            agg.payload_bytes += w.payload_bytes
            agg.total_bytes += w.total_bytes
            agg.index_bytes += w.index_bytes
        return agg

    def reset_stats(self):
        for r in range(self.nranks):
            check(lib().zc_comm_reset_stats(self._h[r]))

    def close(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            for r in range(self.nranks):
                _lib.zc_comm_destroy(self._h[r])
            self._h = None

    def __del__(self):
        self.close()


class RankCtx:
    """The per-rank face of a single-process Group inside Group.run (collectives.hpp:48-110): the
    rank's collectives and point-to-point calls, each on the rank's own communicator (the calls of
    different ranks run concurrently on their own threads, like the reference's rank threads)."""

    def __init__(self, group: "Group", rank: int):
        self._g, self._h, self._rank = group, group._h[rank], rank

    def rank(self) -> int:
        return self._rank

    def nranks(self) -> int:
        return self._g.nranks

    def send_encoded(self, peer: int, raw: torch.Tensor):
        check(lib().zc_comm_send_encoded(self._h, peer, _ptr(raw), raw.numel() * raw.element_size(), None))

    def recv_decoded(self, peer: int, dst: torch.Tensor):
        check(lib().zc_comm_recv_decoded(self._h, peer, _ptr(dst), dst.numel() * dst.element_size(), None))

    def allreduce(self, sym: torch.Tensor, scale: float, mode: int = abi.QUANT_ERROR_BOUNDED, levels: int = 0) -> float:
        s = C.c_double(scale)
        check(lib().zc_comm_allreduce_sym(self._h, _ptr(sym), sym.numel(), mode, C.byref(s), levels, None))
        return s.value

    def allreduce_eb(self, x: torch.Tensor, rel: float, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        out = out if out is not None else torch.empty(x.numel(), dtype=torch.float32, device=x.device)
        check(lib().zc_comm_allreduce_eb_f32(self._h, _ptr(x), _ptr(out), 1 if out.dtype == torch.float64 else 0,
                                             x.numel(), float(rel), None))
        return out

    def allgather(self, all_blocks: torch.Tensor, block: int):
        check(lib().zc_comm_allgather_sym(self._h, _ptr(all_blocks), block, None))

    def broadcast(self, data: torch.Tensor, root: int):
        check(lib().zc_comm_broadcast_sym(self._h, _ptr(data), data.numel(), root, None))

    def allreduce_max(self, v: float) -> float:
        o = C.c_double(0.0)
        check(lib().zc_comm_allreduce_max(self._h, float(v), C.byref(o), None))
        return o.value


class Communicator:
    """One rank of a multi-process communicator (one process per GPU).  The peers' IPC blobs are
    exchanged with torch.distributed (any backend; the data path never uses it)."""

    def __init__(self, rank: int, nranks: int, device: int, cfg: Optional[abi.CollectiveConfig] = None,
                 exchange=None):
        self.rank, self.nranks, self.device = rank, nranks, device
        self.cfg = cfg or collective_config()
        exchange = exchange or _dist_allgather_bytes
        check_consistent_config(self.cfg, rank, exchange)
        h = vp()
        check(lib().zc_comm_create(rank, nranks, device, C.byref(self.cfg), C.byref(h)))
        self._h = h
        n = lib().zc_comm_export_size()
        blob = (C.c_uint8 * n)()
        check(lib().zc_comm_export(h, C.cast(blob, vp)))
        blobs = exchange(bytes(blob))
        allb = (C.c_uint8 * (n * nranks)).from_buffer_copy(b"".join(blobs))
        check(lib().zc_comm_connect(h, C.cast(allb, vp)))

    def set_shared_huffman(self, ctx: HuffmanContext):
        check(lib().zc_comm_set_shared_huffman(self._h, ctx.handle))

    def set_shared_huffman_from_bytes(self, sample) -> None:
        """Communicator::set_shared_huffman_from_bytes (collectives.cpp:99-106)."""
        self.set_shared_huffman(HuffmanContext.from_bytes(sample))

    def allreduce(self, sym: torch.Tensor, scale: float, mode: int = abi.QUANT_ERROR_BOUNDED, levels: int = 0) -> float:
        s = C.c_double(scale)
        check(lib().zc_comm_allreduce_sym(self._h, _ptr(sym), sym.numel(), mode, C.byref(s), levels, _stream()))
        return s.value

    def allreduce_eb(self, x: torch.Tensor, rel: float, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        out = out if out is not None else torch.empty(x.numel(), dtype=torch.float32, device=x.device)
        check(lib().zc_comm_allreduce_eb_f32(self._h, _ptr(x), _ptr(out), 1 if out.dtype == torch.float64 else 0,
                                             x.numel(), float(rel), _stream()))
        return out

    def reduce_scatter(self, sym: torch.Tensor):
        check(lib().zc_comm_reduce_scatter_sym(self._h, _ptr(sym), sym.numel(), _stream()))

    def allgather(self, all_blocks: torch.Tensor, block: int):
        check(lib().zc_comm_allgather_sym(self._h, _ptr(all_blocks), block, _stream()))

    def allreduce_qsgd(self, x: torch.Tensor, levels: int, seed: int, out: Optional[torch.Tensor] = None):
        out = out if out is not None else torch.empty(x.numel(), dtype=torch.float64, device=x.device)
        check(lib().zc_comm_allreduce_qsgd_f32(self._h, _ptr(x), _ptr(out), 1 if out.dtype == torch.float64 else 0,
                                               x.numel(), levels, seed, _stream()))
        return out

    def alltoall(self, send: torch.Tensor) -> torch.Tensor:
        if send.numel() % self.nranks:
            raise ValueError("alltoall buffer must split evenly across ranks")
        out = torch.empty_like(send)
        check(lib().zc_comm_alltoall_sym(self._h, _ptr(send), _ptr(out), send.numel() // self.nranks, _stream()))
        return out

    def broadcast(self, data: torch.Tensor, root: int):
        check(lib().zc_comm_broadcast_sym(self._h, _ptr(data), data.numel(), root, _stream()))

    def send_encoded(self, peer: int, raw: torch.Tensor):
        """RankCtx::send_encoded (collectives.cpp:350-356): the tensor's bytes, framed per batch."""
        check(lib().zc_comm_send_encoded(self._h, peer, _ptr(raw), raw.numel() * raw.element_size(), _stream()))

    def recv_decoded(self, peer: int, dst: torch.Tensor):
        """RankCtx::recv_decoded (collectives.cpp:358-364): fills dst's bytes from peer's frames."""
        check(lib().zc_comm_recv_decoded(self._h, peer, _ptr(dst), dst.numel() * dst.element_size(), _stream()))

    def group_execute(self, requests: Sequence[dict]):
        k = len(requests)
        arr = (abi.CollRequest * k)(*[_request(q) for q in requests])
        check(lib().zc_comm_group_execute(self._h, arr, k, _stream()))
        for i, q in enumerate(requests):
            if q["op"] == abi.COLL_ALLREDUCE:
                q["scale"] = arr[i].scale
        return requests

    def allreduce_max(self, v: float) -> float:
        o = C.c_double()
        check(lib().zc_comm_allreduce_max(self._h, float(v), C.byref(o), None))
        return o.value

    def reset(self):
        check(lib().zc_comm_reset(self._h))

    def wire_stats(self) -> abi.WireStats:
        return _wire(self._h)

    def close(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.zc_comm_destroy(self._h)
            self._h = None


def check_consistent_config(cfg: abi.CollectiveConfig, rank: int, exchange) -> None:
    """Every rank must run the same CollectiveConfig.  Frames are self-describing, so a hint or
    cost-model mismatch would still decode, but ranks would pick different codecs than the
    reference's single config does; a pin or fused_codec_min_msg_bytes mismatch would make ranks
    run different step schedules over the same banks (a hang until the timeout).  The reference
    gets this for free (one Communicator object, collectives.cpp:137-152); across processes it is
    checked once at rendezvous, like the stream-meta check (collectives.cpp:428-452), and raises
    ValueError (std::invalid_argument) on every rank."""
    mine = bytes(cfg)
    allc = exchange(mine)
    bad = [r for r, b in enumerate(allc) if bytes(b) != mine]
    if bad:
        raise ValueError(f"rank {rank}: CollectiveConfig differs on rank(s) {bad}")


def _dist_allgather_bytes(b: bytes):
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, b)
    return out
