"""Generate the golden fixtures from the REFERENCE ITSELF (oracle/_ref/libzcomm_ref.so, compiled from
/root/reference/proj/core/src by oracle/Makefile).  Test infrastructure only.

    python tests/golden/make_golden.py        # needs oracle/_ref built (`make -C oracle ref`)

Writes tests/golden/codec.npz (inputs + frames/payloads) and tests/golden/golden.json (small
known answers, collective outputs as sha256 + a prefix).  Inputs come from deterministic
generators — the reference's own gen_data (bench.cpp:49-68) and numpy's PCG64 with fixed seeds —
and are stored verbatim, so the fixtures do not depend on regenerating them.
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

sys.path.insert(0, os.path.dirname(HERE))
import oracle  # noqa: E402
from golden_data import RING_COUNT, ring_input  # noqa: E402
from paper_2605_12396_b200 import abi  # noqa: E402

GAUSSIAN, UNIFORM, GEOMETRIC = 1, 0, 2  # bench.hpp:13 DataDist
HINTS = {"inter10g": abi.make_hint(), "nvlink900g": abi.make_hint(900e9, abi.REGIME_INTRA),
         "thin1g": abi.make_hint(1e9)}


def sha(b) -> str:
    return hashlib.sha256(np.ascontiguousarray(b).view(np.uint8).tobytes()).hexdigest()


def quantize_scale(R, x, scale):
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(len(x), np.int32)
    rc = R.lib.zr_eb_quantize_with_scale(x, len(x), scale, out)
    assert rc == 0, R.error()
    return out


def quantize_rel(R, x, rel):
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(len(x), np.int32)
    sc = C.c_double()
    rc = R.lib.zr_eb_quantize(x, len(x), rel, out, C.byref(sc))
    assert rc == 0, R.error()
    return out, sc.value


def gen(R, dist, seed, count, geom_p=0.7, rank=0):
    out = np.zeros(count, np.float64)
    assert R.lib.zr_gen_data(dist, geom_p, seed, rank, 0, count, out) == 0
    return out


def codec_inputs(R):
    """name -> raw bytes (uint8).  Sizes straddle the 4096 B small-batch threshold, the 64 KiB
    profile window / Huffman minimum, and include a length that is not a multiple of 4."""
    rng = np.random.default_rng(20260517)
    n = 32768  # 128 KiB of int32 symbols
    cases = {}
    g = gen(R, GAUSSIAN, 1, n).astype(np.float32).astype(np.float64)
    cases["gaussian"] = quantize_scale(R, g, 2e-4)
    u = rng.random(n)
    lap = (-1e-2 * np.sign(u - 0.5) * np.log1p(-2.0 * np.abs(u - 0.5))).astype(np.float32).astype(np.float64)
    cases["laplacian"] = quantize_scale(R, lap, 2e-4)
    cases["geometric"], _ = quantize_rel(R, gen(R, GEOMETRIC, 5, n), 1e-4)
    i = np.arange(n)
    smooth = (np.sin(2 * np.pi * i / 512) * np.cos(4 * np.pi * (i // 512) / 64)).astype(np.float32).astype(np.float64)
    cases["smooth"], _ = quantize_rel(R, smooth, 1e-3)
    cases["uniform"] = quantize_scale(R, gen(R, UNIFORM, 3, n), 1e-3)
    cases["zeros"] = np.zeros(n, np.int32)
    cases["random_i32"] = rng.integers(-2**31, 2**31, n, dtype=np.int64).astype(np.int32)
    cases["lowent_bytes"] = rng.geometric(0.6, n * 4).clip(0, 255).astype(np.uint8)  # Huffman territory
    cases["small_4096"] = cases["gaussian"][:1024].copy()
    cases["small_4100"] = cases["gaussian"][:1025].copy()
    cases["odd_70001"] = cases["gaussian"].view(np.uint8)[:70001].copy()
    cases["tiny_33"] = cases["geometric"].view(np.uint8)[:33].copy()
    cases["w32_extremes"] = np.array([-2**31, 2**31 - 1, 0, -1] * 20000, np.int32)
    return {k: np.ascontiguousarray(v).view(np.uint8).ravel().copy() for k, v in cases.items()}


def ref_fixedlen(R, sym):
    out = np.zeros(len(sym) * 4 + 8, np.uint8)
    w = C.c_uint32()
    p = R.lib.zr_fixedlen_encode(sym, len(sym), out, len(out), C.byref(w))
    return out[:p].copy(), w.value


def ref_huffman(R, raw, ctx, embed):
    out = np.zeros(len(raw) * 4 + 512, np.uint8)
    p = R.lib.zr_huffman_encode(raw, len(raw), ctx, out, len(out), 1 if embed else 0)
    return out[:p].copy()


def main():
    R = oracle.ref()
    if R is None:
        sys.exit("oracle/_ref/libzcomm_ref.so missing: run `make -C oracle ref` (needs /root/reference)")
    arrays, meta = {}, {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (reference sources)",
                        "codec": {}, "known": {}, "collectives": {}}
    cfg = abi.default_arb_config()

    # ---------------- codec cases: encode_best (rea.cpp:178-238) under three hints, with/without ctx
    for name, raw in codec_inputs(R).items():
        arrays[f"raw/{name}"] = raw
        ctx = R.huff_from_bytes(raw[: abi.BATCH_RAW_BYTES])  # set_shared_huffman_from_bytes (+1 smoothing)
        lens = R.huff_tables(ctx)[0]
        arrays[f"ctxlens/{name}"] = lens
        entry = {"raw_bytes": int(len(raw)), "frames": {}}
        for hname, hint in HINTS.items():
            for use_ctx in (False, True):
                r, frame = R.encode_best(raw, hint, ctx if use_ctx else None, cfg)
                key = f"{hname}/{'ctx' if use_ctx else 'noctx'}"
                arrays[f"frame/{sha(frame)}"] = frame  # deduplicated by content
                entry["frames"][key] = {"codec": int(r.codec), "payload_bytes": int(r.payload_bytes),
                                        "total_bytes": int(r.total_bytes), "sha256": sha(frame)}
        if len(raw) % 4 == 0 and len(raw) > 0:
            fl, w = ref_fixedlen(R, raw.view(np.int32))
            arrays[f"fixedlen/{name}"] = fl
            entry["fixedlen_width"] = int(w)
        hf = ref_huffman(R, raw, ctx, False)
        arrays[f"huffman/{name}"] = hf
        entry["huffman_payload"] = int(len(hf))
        st = abi.SampleStats()
        R.lib.zr_profile_sample(raw, len(raw), ctx, C.byref(st))
        entry["profile"] = {"sampled_bytes": int(st.sampled_bytes), "max_zigzag": int(st.max_zigzag),
                            "ctx_code_len_bits": float(st.ctx_code_len_bits),
                            "ctx_code_len_valid": int(st.ctx_code_len_valid), "hist_sha256": sha(np.array(st.hist, np.uint64))}
        R.lib.zr_huff_ctx_free(ctx)
        meta["codec"][name] = entry

    # ---------------- known answers quoted by the reference's own unit tests
    k = meta["known"]
    s, sc = quantize_rel(R, np.array([1.0, 1.05]), 0.1)                       # test_quant.cpp:20-30
    k["eb_hand"] = {"x": [1.0, 1.05], "rel": 0.1, "scale": sc, "symbols": s.tolist()}
    for nm, syms in {"hand": [0, 1, -1, 2], "zeros": [0, 0, 0, 0],              # test_fixedlen.cpp:51-75
                     "full_width": [-2**31, 2**31 - 1, 0, -1]}.items():        # test_fixedlen.cpp:115-125
        p, w = ref_fixedlen(R, np.array(syms, np.int32))
        k[f"fixedlen_{nm}"] = {"symbols": syms, "width": w, "payload": p.tolist()}
    fib = np.zeros(256, np.uint64)                                            # test_huffman.cpp:205-231
    a, b = 1, 1
    for i in range(60):
        fib[i] = a
        a, b = b, a + b
    hists = {"single42": {42: 1000}, "two_equal": {0: 500, 255: 500},
             "geometric8": {i: 1 << (10 - i) for i in range(8)}}
    for nm, hd in hists.items():
        h = np.zeros(256, np.uint64)
        for kk, vv in hd.items():
            h[kk] = vv
        hists[nm] = h
    hists["fibonacci60"] = fib
    rng = np.random.default_rng(31)
    for t in range(6):
        h = np.zeros(256, np.uint64)
        for _ in range(int(rng.integers(2, 200))):
            h[int(rng.integers(0, 256))] += int(rng.integers(1, 100000))
        hists[f"random{t}"] = h
    for nm, h in hists.items():
        ctx = R.huff_from_hist(h)
        lens, code, rev, lut, mm = R.huff_tables(ctx)
        el = C.c_double()
        ok = R.lib.zr_huffman_expected_code_len(ctx, h, C.byref(el))
        k[f"huff_{nm}"] = {"hist": [int(v) for v in h], "valid": int(R.lib.zr_huff_ctx_valid(ctx)),
                           "lens": lens.tolist(), "code": code.tolist(), "rev": rev.tolist(),
                           "lut_sha256": sha(lut), "expected_len": el.value if ok else None}
        R.lib.zr_huff_ctx_free(ctx)
    raw7 = np.full(1000, 7, np.uint8)                                         # test_huffman.cpp:112-123
    h7 = np.bincount(raw7, minlength=256).astype(np.uint64)
    ctx = R.huff_from_hist(h7)
    k["huff_embedded_repeat"] = {"n": 1000, "payload": int(len(ref_huffman(R, raw7, ctx, True)))}
    R.lib.zr_huff_ctx_free(ctx)

    # selector decisions on rigged profiles (rea.cpp:145-176) for a sweep of beta
    sel = []
    for name in ("gaussian", "laplacian", "geometric", "lowent_bytes", "random_i32", "zeros"):
        raw = arrays[f"raw/{name}"]
        ctx = R.huff_from_bytes(raw)
        st = abi.SampleStats()
        R.lib.zr_profile_sample(raw, len(raw), ctx, C.byref(st))
        for beta in (1e8, 1e9, 1e10, 1.0737e10, 1e11, 2.4e11, 9e11, 0.0):
            for raw_bytes in (65536, 1 << 20, abi.BATCH_RAW_BYTES):
                plan = abi.ArbitrationPlan()
                R.lib.zr_arbitrate_plan(raw_bytes, abi.BATCH_RAW_BYTES, C.byref(st), abi.REGIME_INTER, beta, ctx,
                                        C.byref(cfg), C.byref(plan))
                sel.append({"case": name, "beta": beta, "raw_bytes": raw_bytes, "choice": int(plan.choice),
                            "pred": [int(plan.raw.predicted_payload), int(plan.fixedlen.predicted_payload),
                                     int(plan.huffman.predicted_payload)],
                            "sec": [plan.raw.predicted_sec, plan.fixedlen.predicted_sec, plan.huffman.predicted_sec],
                            "admissible": [int(plan.raw.admissible), int(plan.fixedlen.admissible),
                                           int(plan.huffman.admissible)]})
        R.lib.zr_huff_ctx_free(ctx)
    k["selector"] = sel

    # ---------------- collectives (collectives.cpp:426-523) through the reference Communicator
    col = meta["collectives"]
    # symbol sum and scale reconciliation hand vectors (test_collectives.cpp:83-118)
    for nm, (syms, scales) in {"symsum4": ([[r + 1, -(r + 1), 100] for r in range(4)], [1.0] * 4),
                               "reconcile2": ([[10, -6, 3, 7], [1, 2, 3, 4]], [0.5, 1.0])}.items():
        s = np.array(syms, np.int32)
        sc = np.array(scales, np.float64)
        w = abi.WireStats()
        c = abi.default_collective_config()
        rc = R.lib.zr_allreduce_sym(len(s), C.byref(c), s.ravel(), s.shape[1], abi.QUANT_ERROR_BOUNDED, sc, 0,
                                    None, 0, C.byref(w), None)
        assert rc == 0, R.error()
        col[nm] = {"in": syms, "scales_in": scales, "out": s.tolist(), "scales_out": sc.tolist()}
    # multi-batch ring allreduce (fused compressed RS + AG), every pin, n = 2, 3, 4
    count = RING_COUNT
    for n in (2, 3, 4):
        base = ring_input(n, count)  # regenerated by the tests; its hash is pinned below
        col[f"ring{n}_input_sha256"] = sha(base)
        for pin in (abi.PIN_AUTO, abi.PIN_RAW, abi.PIN_FIXEDLEN, abi.PIN_HUFFMAN):
            s = base.copy()
            sc = np.full(n, 2e-4)
            w = abi.WireStats()
            c = abi.default_collective_config(pin)
            sample = np.ascontiguousarray(base[0].view(np.uint8)[: abi.BATCH_RAW_BYTES])
            rc = R.lib.zr_allreduce_sym(n, C.byref(c), s.ravel(), count, abi.QUANT_ERROR_BOUNDED, sc, 0,
                                        sample.ctypes.data_as(C.POINTER(C.c_uint8)), len(sample), C.byref(w), None)
            assert rc == 0, R.error()
            assert all((s[r] == s[0]).all() for r in range(n))
            col[f"ring{n}_{abi.PIN_NAMES[pin]}"] = {
                "n": n, "count": count, "pin": pin, "out_sha256": sha(s[0]), "out_head": s[0][:8].tolist(),
                "wire": {"frames_by_codec": list(w.frames_by_codec), "raw_bytes": int(w.raw_bytes),
                         "payload_bytes": int(w.payload_bytes), "total_bytes": int(w.total_bytes)}}
        # per-slot framing (CollectiveConfig::perSlotFraming, collectives.cpp:197-199): every
        # exchange batches at 512 KiB, so frames, decisions and WireStats all change
        for pin in (abi.PIN_AUTO, abi.PIN_RAW, abi.PIN_FIXEDLEN, abi.PIN_HUFFMAN):
            s = base.copy()
            sc = np.full(n, 2e-4)
            w = abi.WireStats()
            c = abi.default_collective_config(pin)
            c.per_slot_framing = 1
            sample = np.ascontiguousarray(base[0].view(np.uint8)[: abi.BATCH_RAW_BYTES])
            rc = R.lib.zr_allreduce_sym(n, C.byref(c), s.ravel(), count, abi.QUANT_ERROR_BOUNDED, sc, 0,
                                        sample.ctypes.data_as(C.POINTER(C.c_uint8)), len(sample), C.byref(w), None)
            assert rc == 0, R.error()
            col[f"ring{n}_{abi.PIN_NAMES[pin]}_slot"] = {
                "n": n, "count": count, "pin": pin, "per_slot_framing": 1, "out_sha256": sha(s[0]),
                "wire": {"frames_by_codec": list(w.frames_by_codec), "raw_bytes": int(w.raw_bytes),
                         "payload_bytes": int(w.payload_bytes), "total_bytes": int(w.total_bytes)}}
        # allgather (collectives.cpp:525-544) of ragged-free blocks
        blk = base[:, :300_000].copy()
        out = np.zeros(n * n * 300_000, np.int32)  # every rank's gathered copy
        w = abi.WireStats()
        c = abi.default_collective_config(abi.PIN_AUTO)
        rc = R.lib.zr_allgather_sym(n, C.byref(c), blk.ravel(), 300_000, None, 0, out, C.byref(w))
        assert rc == 0, R.error()
        out = out.reshape(n, n * 300_000)
        assert all((out[r] == out[0]).all() for r in range(n)) and (out[0] == blk.ravel()).all()
        col[f"allgather{n}"] = {"n": n, "block": 300_000, "out_sha256": sha(out[0]),
                                "wire": {"frames_by_codec": list(w.frames_by_codec), "raw_bytes": int(w.raw_bytes),
                                         "payload_bytes": int(w.payload_bytes), "total_bytes": int(w.total_bytes)}}

    np.savez_compressed(os.path.join(HERE, "codec.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays;", os.path.getsize(os.path.join(HERE, "codec.npz")) >> 10, "KiB npz")


if __name__ == "__main__":
    main()
