"""TEST INFRASTRUCTURE ONLY — the parity checker.

Two CPU implementations of the reference's hot path, loaded with ctypes:

* ``port`` — ``_build/libzc_oracle.so``, the plain-C restatement in zc_oracle.c;
* ``ref``  — ``_ref/libzcomm_ref.so``, the UNMODIFIED reference sources compiled in
  place (oracle/Makefile) behind the shim ref_shim.cpp.  Present whenever
  /root/reference was available at build time (the .so travels to the GPU box).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline / reference
arm may import this package, and only as the checker or the timed baseline.
The product library (paper_2605_12396_b200) never imports it.
"""
import ctypes as C
import os
import subprocess

import numpy as np

from paper_2605_12396_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libzc_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libzcomm_ref.so")
REF_SRC = "/root/reference/proj/core"

u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
P = C.POINTER


def build(ref: bool = True) -> None:
    """Compile the C restatement, and the reference (when its sources are present)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


class HuffStruct(C.Structure):  # zo_huff (zc_oracle.h)
    _fields_ = [("valid", C.c_int32), ("len", C.c_uint8 * 256), ("code", C.c_uint32 * 256),
                ("rev", C.c_uint32 * 256), ("sym_order", C.c_uint8 * 256), ("count_at_len", C.c_uint32 * 33),
                ("first_code", C.c_uint64 * 33), ("first_index", C.c_uint32 * 33), ("lut", C.c_uint16 * 4096),
                ("min_len", C.c_uint32), ("max_len", C.c_uint32)]


def _sig(lib, name, restype, *args):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(args)
    return f


class Port:
    """The C restatement (zc_oracle.c)."""

    def __init__(self, path=PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        H = P(HuffStruct)
        _sig(L, "zo_write_header", None, P(abi.FrameHeader), u8p)
        _sig(L, "zo_parse_header", C.c_int, u8p, C.c_uint64, P(abi.FrameHeader))
        _sig(L, "zo_validate_header", C.c_int, P(abi.FrameHeader), C.c_uint64)
        _sig(L, "zo_frame_commit_raw", C.c_uint64, u8p, C.c_uint64, u8p, C.c_uint64)
        _sig(L, "zo_eb_quantize_f64", C.c_int, f64p, C.c_uint64, C.c_double, i32p)
        _sig(L, "zo_eb_quantize_f32", C.c_int, f32p, C.c_uint64, C.c_double, i32p)
        _sig(L, "zo_qsgd_quantize_f32", C.c_int, f32p, C.c_uint64, C.c_uint32, C.c_uint64, i32p, P(C.c_double))
        _sig(L, "zo_qsgd_quantize_chunk_f32", C.c_int, f32p, C.c_uint64, C.c_uint32, C.c_double, C.c_uint64,
             C.c_uint64, i32p)
        _sig(L, "zo_absmax_f32", C.c_int, f32p, C.c_uint64, P(C.c_double))
        _sig(L, "zo_dequantize_f64", None, i32p, C.c_uint64, C.c_int, C.c_double, C.c_uint32, f64p)
        _sig(L, "zo_dequantize_f32", None, i32p, C.c_uint64, C.c_int, C.c_double, C.c_uint32, f32p)
        _sig(L, "zo_fixedlen_width", C.c_uint32, i32p, C.c_uint64)
        _sig(L, "zo_fixedlen_encode", C.c_uint64, i32p, C.c_uint64, u8p, C.c_uint64, P(C.c_uint32))
        _sig(L, "zo_fixedlen_decode", C.c_int, P(abi.FrameHeader), u8p, C.c_uint64, u8p, C.c_uint64)
        _sig(L, "zo_huff_lengths", None, u64p, u8p)
        _sig(L, "zo_huff_build", C.c_int, u64p, H)
        _sig(L, "zo_huff_from_lengths", C.c_int, u8p, H)
        _sig(L, "zo_huff_from_bytes", C.c_int, u8p, C.c_uint64, H)
        _sig(L, "zo_huff_expected_len", C.c_int, H, u64p, P(C.c_double))
        _sig(L, "zo_huff_self_len", C.c_int, u64p, P(C.c_double))
        _sig(L, "zo_huffman_encode", C.c_uint64, u8p, C.c_uint64, H, u8p, C.c_uint64, C.c_int)
        _sig(L, "zo_huffman_decode", C.c_int, P(abi.FrameHeader), u8p, C.c_uint64, H, u8p, C.c_uint64)
        _sig(L, "zo_profile_sample", None, u8p, C.c_uint64, H, P(abi.SampleStats))
        _sig(L, "zo_predict_payload", C.c_uint64, C.c_int, C.c_uint64, P(abi.SampleStats), P(abi.ArbConfig))
        _sig(L, "zo_arbitrate_plan", None, C.c_uint64, C.c_uint64, P(abi.SampleStats), P(abi.TransportHint), H,
             P(abi.ArbConfig), P(abi.ArbitrationPlan))
        _sig(L, "zo_encode_best", None, u8p, C.c_uint64, u8p, C.c_uint64, P(abi.TransportHint), H,
             P(abi.ArbConfig), P(abi.EncodeResult))
        _sig(L, "zo_send_batch", None, u8p, C.c_uint64, u8p, C.c_uint64, C.c_int, P(abi.TransportHint), H,
             P(abi.ArbConfig), P(abi.EncodeResult))
        _sig(L, "zo_recv_batch", C.c_int, u8p, C.c_uint64, H, u8p, C.c_uint64)
        _sig(L, "zo_ring_allreduce", C.c_int, C.c_int, i32p, C.c_uint64, f64p, C.c_int, P(abi.TransportHint), H,
             P(abi.ArbConfig), C.c_uint64, P(abi.WireStats))
        _sig(L, "zo_ring_allgather", C.c_int, C.c_int, i32p, C.c_uint64, C.c_int, P(abi.TransportHint), H,
             P(abi.ArbConfig), i32p, P(abi.WireStats))
        _sig(L, "zo_set_per_slot_framing", None, C.c_int)
        _sig(L, "zo_gen_data", C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, f64p)

    # --- convenience wrappers (numpy in, numpy out) ---
    def huff_from_hist(self, hist):
        h = HuffStruct()
        self.lib.zo_huff_build(np.ascontiguousarray(hist, np.uint64), C.byref(h))
        return h

    def huff_from_bytes(self, sample):
        h = HuffStruct()
        self.lib.zo_huff_from_bytes(np.ascontiguousarray(sample, np.uint8), len(sample), C.byref(h))
        return h

    def eb_quantize_f32(self, x, scale):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros(len(x), np.int32)
        rc = self.lib.zo_eb_quantize_f32(x, len(x), scale, out)
        return rc, out

    def qsgd_quantize_f32(self, x, levels, seed):
        """qsgd_quantize (quant.cpp:84-98): (rc, symbols, scale)."""
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros(max(len(x), 1), np.int32)
        sc = C.c_double(0.0)
        rc = self.lib.zo_qsgd_quantize_f32(x, len(x), levels, seed, out, C.byref(sc))
        return rc, out[:len(x)], sc.value

    def qsgd_quantize_chunk_f32(self, x, levels, norm, seed, skip=0):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros(max(len(x), 1), np.int32)
        rc = self.lib.zo_qsgd_quantize_chunk_f32(x, len(x), levels, norm, seed, skip, out)
        return rc, out[:len(x)]

    def send_batch(self, raw, pin=abi.PIN_AUTO, hint=None, ctx=None, cfg=None, cap=abi.STAGE_BANK_BYTES):
        raw = np.ascontiguousarray(raw).view(np.uint8).ravel()
        stage = np.zeros(max(cap, 1), np.uint8)
        r = abi.EncodeResult()
        self.lib.zo_send_batch(raw, len(raw), stage, cap, pin, C.byref(hint or abi.make_hint()),
                               C.byref(ctx) if ctx is not None else None, C.byref(cfg or abi.default_arb_config()),
                               C.byref(r))
        return r, stage[: r.total_bytes].copy()

    def encode_best(self, raw, hint=None, ctx=None, cfg=None, cap=abi.STAGE_BANK_BYTES):
        raw = np.ascontiguousarray(raw).view(np.uint8).ravel()
        stage = np.zeros(max(cap, 1), np.uint8)
        r = abi.EncodeResult()
        self.lib.zo_encode_best(raw, len(raw), stage, cap, C.byref(hint or abi.make_hint()),
                                C.byref(ctx) if ctx is not None else None, C.byref(cfg or abi.default_arb_config()),
                                C.byref(r))
        return r, stage[: r.total_bytes].copy()

    def fixedlen_encode(self, sym, cap=None):
        sym = np.ascontiguousarray(sym, np.int32)
        out = np.zeros(cap if cap is not None else len(sym) * 4 + 8, np.uint8)
        w = C.c_uint32()
        p = self.lib.zo_fixedlen_encode(sym, len(sym), out, len(out), C.byref(w))
        return out[:p].copy(), w.value

    def huffman_encode(self, raw, ctx, embed=False, cap=None):
        raw = np.ascontiguousarray(raw, np.uint8)
        out = np.zeros(cap if cap is not None else len(raw) * 4 + 512, np.uint8)
        p = self.lib.zo_huffman_encode(raw, len(raw), C.byref(ctx), out, len(out), 1 if embed else 0)
        return out[:p].copy()

    def ring_allgather(self, blocks, pin=abi.PIN_AUTO, hint=None, ctx=None, cfg=None, per_slot=False):
        blocks = np.ascontiguousarray(blocks, np.int32)
        n, block = blocks.shape
        out = np.zeros((n, n * block), np.int32)  # every rank's gathered copy
        w = abi.WireStats()
        self.lib.zo_set_per_slot_framing(1 if per_slot else 0)
        try:
            rc = self.lib.zo_ring_allgather(n, blocks.ravel(), block, pin, C.byref(hint or abi.make_hint()),
                                            C.byref(ctx) if ctx is not None else None,
                                            C.byref(cfg or abi.default_arb_config()), out.ravel(), C.byref(w))
        finally:
            self.lib.zo_set_per_slot_framing(0)
        return rc, out, w

    def encode_batches(self, raw, pin=abi.PIN_AUTO, hint=None, ctx=None, cfg=None, stage_len=abi.STAGE_BANK_BYTES):
        """Frame every 4 MiB batch of a message exactly as send_encoded does (collectives.cpp:350-356)."""
        raw = np.ascontiguousarray(raw).view(np.uint8).ravel()
        out = []
        for off in range(0, len(raw), abi.BATCH_RAW_BYTES):
            out.append(self.send_batch(raw[off:off + abi.BATCH_RAW_BYTES], pin, hint, ctx, cfg, cap=stage_len))
        return out

    def recv_batch(self, frame, dlen, ctx=None):
        frame = np.ascontiguousarray(frame, np.uint8)
        dst = np.zeros(max(dlen, 1), np.uint8)
        codec = self.lib.zo_recv_batch(frame, len(frame), C.byref(ctx) if ctx is not None else None, dst, dlen)
        return codec, dst[:dlen]

    def gen_data(self, dist, seed, rank, count, offset=0, geom_p=0.7):
        out = np.zeros(count, np.float64)
        rc = self.lib.zo_gen_data(dist, geom_p, seed, rank, offset, count, out)
        if rc:
            raise ValueError("gen_data failed")
        return out

    def profile(self, raw, ctx=None):
        raw = np.ascontiguousarray(raw).view(np.uint8).ravel()
        st = abi.SampleStats()
        self.lib.zo_profile_sample(raw, len(raw), C.byref(ctx) if ctx is not None else None, C.byref(st))
        return st

    def ring_allreduce(self, syms, scales, pin=abi.PIN_AUTO, hint=None, ctx=None, cfg=None,
                       fused_min=abi.BATCH_RAW_BYTES, per_slot=False):
        syms = np.ascontiguousarray(syms, np.int32).copy()
        n, count = syms.shape
        sc = np.ascontiguousarray(scales, np.float64).copy()
        w = abi.WireStats()
        self.lib.zo_set_per_slot_framing(1 if per_slot else 0)
        try:
            rc = self.lib.zo_ring_allreduce(n, syms.ravel(), count, sc, pin, C.byref(hint or abi.make_hint()),
                                            C.byref(ctx) if ctx is not None else None,
                                            C.byref(cfg or abi.default_arb_config()), fused_min, C.byref(w))
        finally:
            self.lib.zo_set_per_slot_framing(0)
        return rc, syms, sc, w


class Ref:
    """The reference itself (oracle/_ref/libzcomm_ref.so)."""

    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.lib = C.CDLL(path)
        vp = C.c_void_p
        _sig(L, "zr_last_error", C.c_char_p)
        _sig(L, "zr_default_arb_config", None, P(abi.ArbConfig))
        _sig(L, "zr_write_header", C.c_int, P(abi.FrameHeader), u8p, C.c_uint64)
        _sig(L, "zr_parse_header", C.c_int, u8p, C.c_uint64, P(abi.FrameHeader))
        _sig(L, "zr_validate_header", C.c_int, P(abi.FrameHeader), C.c_uint64)
        _sig(L, "zr_frame_commit_raw", C.c_uint64, u8p, C.c_uint64, u8p, C.c_uint64)
        _sig(L, "zr_eb_quantize_with_scale", C.c_int, f64p, C.c_uint64, C.c_double, i32p)
        _sig(L, "zr_eb_quantize", C.c_int, f64p, C.c_uint64, C.c_double, i32p, P(C.c_double))
        _sig(L, "zr_eb_quantize_chunk", C.c_int, f64p, C.c_uint64, C.c_double, i32p)
        _sig(L, "zr_dequantize", C.c_int, i32p, C.c_uint64, C.c_int, C.c_double, C.c_uint32, f64p)
        _sig(L, "zr_fixedlen_width", C.c_uint32, i32p, C.c_uint64)
        _sig(L, "zr_fixedlen_encode", C.c_uint64, i32p, C.c_uint64, u8p, C.c_uint64, P(C.c_uint32))
        _sig(L, "zr_fixedlen_decode", C.c_int, P(abi.FrameHeader), u8p, C.c_uint64, u8p, C.c_uint64)
        _sig(L, "zr_huff_ctx_new", vp, u64p)
        _sig(L, "zr_huff_ctx_from_bytes", vp, u8p, C.c_uint64)
        _sig(L, "zr_huff_ctx_from_lengths", vp, u8p)
        _sig(L, "zr_huff_ctx_free", None, vp)
        _sig(L, "zr_huff_ctx_valid", C.c_int, vp)
        _sig(L, "zr_huff_ctx_tables", None, vp, u8p, u32p, u32p, np.ctypeslib.ndpointer(np.uint16), u32p)
        _sig(L, "zr_huffman_expected_code_len", C.c_int, vp, u64p, P(C.c_double))
        _sig(L, "zr_huffman_self_code_len", C.c_int, u64p, P(C.c_double))
        _sig(L, "zr_huffman_encode", C.c_uint64, u8p, C.c_uint64, vp, u8p, C.c_uint64, C.c_int)
        _sig(L, "zr_huffman_decode", C.c_int, P(abi.FrameHeader), u8p, C.c_uint64, vp, u8p, C.c_uint64)
        _sig(L, "zr_profile_sample", None, u8p, C.c_uint64, vp, P(abi.SampleStats))
        _sig(L, "zr_predict_payload", C.c_uint64, C.c_int, C.c_uint64, P(abi.SampleStats), P(abi.ArbConfig))
        _sig(L, "zr_arbitrate_plan", None, C.c_uint64, C.c_uint64, P(abi.SampleStats), C.c_int, C.c_double, vp,
             P(abi.ArbConfig), P(abi.ArbitrationPlan))
        _sig(L, "zr_encode_best", None, u8p, C.c_uint64, u8p, C.c_uint64, C.c_int, C.c_double, vp, P(abi.ArbConfig),
             P(abi.EncodeResult))
        _sig(L, "zr_allreduce_eb", C.c_int, C.c_int, P(abi.CollectiveConfig), f64p, C.c_uint64, C.c_double, vp,
             C.c_uint64, f64p, P(abi.WireStats), P(C.c_double))
        _sig(L, "zr_allreduce_sym", C.c_int, C.c_int, P(abi.CollectiveConfig), i32p, C.c_uint64, C.c_int, f64p,
             C.c_uint32, vp, C.c_uint64, P(abi.WireStats), P(C.c_double))
        _sig(L, "zr_allgather_sym", C.c_int, C.c_int, P(abi.CollectiveConfig), i32p, C.c_uint64, vp, C.c_uint64,
             i32p, P(abi.WireStats))
        _sig(L, "zr_gen_data", C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, f64p)
        _sig(L, "zr_qsgd_quantize", C.c_int, f64p, C.c_uint64, C.c_uint32, C.c_uint64, i32p, P(C.c_double))
        _sig(L, "zr_qsgd_quantize_chunk", C.c_int, f64p, C.c_uint64, C.c_uint32, C.c_double, C.c_uint64, C.c_uint64,
             i32p)
        _sig(L, "zr_mt19937_64", C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, u64p)
        _sig(L, "zr_allreduce_qsgd", C.c_int, C.c_int, P(abi.CollectiveConfig), f64p, C.c_uint64, C.c_uint32, u64p,
             f64p)
        _sig(L, "zr_emit_csv", C.c_int, f64p, C.c_int, C.c_char_p, C.c_uint64)
        _sig(L, "zr_emit_markdown", C.c_int, f64p, C.c_int, C.c_char_p, C.c_uint64)
        _sig(L, "zr_codec_roundtrip_mt", C.c_int, f32p, C.c_uint64, C.c_double, C.c_int, vp, P(abi.ArbConfig),
             C.c_int, C.c_double, C.c_int, vp, P(C.c_uint64), u64p, P(C.c_double))

    def _emit(self, fn, rows):
        flat = np.ascontiguousarray([v for r in rows for v in r.flat()], np.float64)
        buf = C.create_string_buffer(1 << 20)
        n = fn(flat, len(rows), buf, len(buf))
        assert n >= 0
        return buf.value.decode()

    def qsgd_quantize(self, x, levels, seed):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(max(len(x), 1), np.int32)
        sc = C.c_double(0.0)
        rc = self.lib.zr_qsgd_quantize(x, len(x), levels, seed, out, C.byref(sc))
        return rc, out[:len(x)], sc.value

    def qsgd_quantize_chunk(self, x, levels, norm, seed, skip=0):
        x = np.ascontiguousarray(x, np.float64)
        out = np.zeros(max(len(x), 1), np.int32)
        rc = self.lib.zr_qsgd_quantize_chunk(x, len(x), levels, norm, seed, skip, out)
        return rc, out[:len(x)]

    def mt19937_64(self, seed, skip, n):
        out = np.zeros(max(n, 1), np.uint64)
        self.lib.zr_mt19937_64(seed, skip, n, out)
        return out[:n]

    def allreduce_qsgd(self, xs, levels, seeds, pin=abi.PIN_AUTO):
        """RankCtx::allreduce_qsgd (collectives.cpp:518-523) on n rank threads: f64 outputs."""
        xs = np.ascontiguousarray(np.stack(xs), np.float64)
        n, count = xs.shape
        out = np.zeros(n * count, np.float64)
        cfg = abi.default_collective_config(pin)
        rc = self.lib.zr_allreduce_qsgd(n, C.byref(cfg), xs.ravel(), count, levels,
                                        np.ascontiguousarray(seeds, np.uint64), out)
        return rc, out.reshape(n, count)

    def emit_csv(self, rows):
        """bench.cpp:551-565 emit_csv over ReportRow records (report.ReportRow)."""
        return self._emit(self.lib.zr_emit_csv, rows)

    def emit_markdown(self, rows):
        """bench.cpp:620-671 emit_markdown."""
        return self._emit(self.lib.zr_emit_markdown, rows)

    def huff_from_hist(self, hist):
        return C.c_void_p(self.lib.zr_huff_ctx_new(np.ascontiguousarray(hist, np.uint64)))

    def huff_from_bytes(self, sample):
        s = np.ascontiguousarray(sample, np.uint8)
        return C.c_void_p(self.lib.zr_huff_ctx_from_bytes(s, len(s)))

    def huff_tables(self, ctx):
        lens = np.zeros(256, np.uint8)
        code = np.zeros(256, np.uint32)
        rev = np.zeros(256, np.uint32)
        lut = np.zeros(4096, np.uint16)
        mm = np.zeros(2, np.uint32)
        self.lib.zr_huff_ctx_tables(ctx, lens, code, rev, lut, mm)
        return lens, code, rev, lut, mm

    def encode_best(self, raw, hint=None, ctx=None, cfg=None, cap=abi.STAGE_BANK_BYTES):
        raw = np.ascontiguousarray(raw).view(np.uint8).ravel()
        hint = hint or abi.make_hint()
        stage = np.zeros(max(cap, 1), np.uint8)
        r = abi.EncodeResult()
        self.lib.zr_encode_best(raw, len(raw), stage, cap, hint.regime, hint.beta_eff_bytes_per_sec, ctx,
                                C.byref(cfg or abi.default_arb_config()), C.byref(r))
        return r, stage[: r.total_bytes].copy()

    def error(self):
        return self.lib.zr_last_error().decode()


_port = None
_ref = None


def port() -> Port:
    global _port
    if _port is None:
        _port = Port()
    return _port


def ref():
    """The compiled reference, or None when it was never built (no /root/reference at build time)."""
    global _ref
    if _ref is None and os.path.exists(REF_SO):
        _ref = Ref()
    return _ref
