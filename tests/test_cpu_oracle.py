"""CPU: pin the oracle (oracle/zc_oracle.c, the C restatement) to the reference.

Two anchors, both produced by the reference itself:
  * tests/golden/{codec.npz,golden.json} — generated from oracle/_ref (the unmodified reference
    sources compiled by oracle/Makefile) by tests/golden/make_golden.py; they travel with the repo;
  * a live differential against oracle/_ref when it is built (skipped otherwise).
The known-answer cases restate the reference's own unit tests (file:line cited per test).
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from paper_2605_12396_b200 import abi

from golden_data import GOLDEN, arrays, frame_of, ring_input, sha


def _port_ctx(port, raw):
    return port.huff_from_bytes(np.ascontiguousarray(raw[: abi.BATCH_RAW_BYTES]))


HINTS = {"inter10g": abi.make_hint(), "nvlink900g": abi.make_hint(900e9, abi.REGIME_INTRA),
         "thin1g": abi.make_hint(1e9)}


# ------------------------------------------------------------------ codec golden vectors
@pytest.mark.parametrize("name", sorted(GOLDEN["codec"]))
def test_encode_best_frames_match_reference(port, name):
    """encode_best (rea.cpp:178-238): frames byte-identical to the reference's, every hint, with and
    without a shared context; recv_batch (collectives.cpp:304-348) restores the input."""
    g = GOLDEN["codec"][name]
    raw = arrays()[f"raw/{name}"]
    ctx = _port_ctx(port, raw)
    assert list(ctx.len) == arrays()[f"ctxlens/{name}"].tolist()
    for key, want in g["frames"].items():
        hname, c = key.split("/")
        r, frame = port.encode_best(raw, HINTS[hname], ctx if c == "ctx" else None)
        assert (r.codec, r.payload_bytes, r.total_bytes) == (want["codec"], want["payload_bytes"], want["total_bytes"]), key
        assert sha(frame) == want["sha256"], key
        codec, back = port.recv_batch(frame, len(raw), ctx)
        assert codec == want["codec"] and bytes(back) == bytes(raw), key


@pytest.mark.parametrize("name", sorted(GOLDEN["codec"]))
def test_bare_codecs_match_reference(port, name):
    """fixedlen_encode (fixedlen.cpp:15-37) and huffman_encode (huffman.cpp:216-246) payloads."""
    g = GOLDEN["codec"][name]
    raw = arrays()[f"raw/{name}"]
    if "fixedlen_width" in g:
        p, w = port.fixedlen_encode(raw.view(np.int32))
        assert w == g["fixedlen_width"]
        assert bytes(p) == bytes(arrays()[f"fixedlen/{name}"])
    ctx = _port_ctx(port, raw)
    assert bytes(port.huffman_encode(raw, ctx)) == bytes(arrays()[f"huffman/{name}"])


@pytest.mark.parametrize("name", sorted(GOLDEN["codec"]))
def test_profile_sample_matches_reference(port, name):
    """profile_sample (rea.cpp:93-118): 64 KiB prefix histogram, max zig-zag, ctx code length."""
    g = GOLDEN["codec"][name]["profile"]
    raw = arrays()[f"raw/{name}"]
    st = port.profile(raw, _port_ctx(port, raw))
    assert st.sampled_bytes == g["sampled_bytes"] and st.max_zigzag == g["max_zigzag"]
    assert sha(np.array(st.hist, np.uint64)) == g["hist_sha256"]
    assert st.ctx_code_len_valid == g["ctx_code_len_valid"]
    assert st.ctx_code_len_bits == g["ctx_code_len_bits"]  # bit-exact double


def test_selector_decisions_match_reference(port):
    """arbitrate_plan (rea.cpp:145-176), Eq. 1 without FMA: choice, predictions and predicted times
    bit-identical over a beta sweep (cf. test_rea.cpp:186-225, acceptance.cpp:296-412)."""
    for e in GOLDEN["known"]["selector"]:
        raw = arrays()[f"raw/{e['case']}"]
        ctx = port.huff_from_bytes(raw)
        st = port.profile(raw, ctx)
        plan = abi.ArbitrationPlan()
        port.lib.zo_arbitrate_plan(e["raw_bytes"], abi.BATCH_RAW_BYTES, C.byref(st),
                                   C.byref(abi.make_hint(e["beta"])), C.byref(ctx),
                                   C.byref(abi.default_arb_config()), C.byref(plan))
        assert plan.choice == e["choice"], e
        assert [plan.raw.predicted_payload, plan.fixedlen.predicted_payload, plan.huffman.predicted_payload] == e["pred"]
        assert [plan.raw.admissible, plan.fixedlen.admissible, plan.huffman.admissible] == e["admissible"]
        assert [plan.raw.predicted_sec, plan.fixedlen.predicted_sec, plan.huffman.predicted_sec] == e["sec"]


# ------------------------------------------------------------------ known answers (reference unit tests)
def test_quant_hand_example(port):
    """test_quant.cpp:20-30: x = [1.0, 1.05], rel 0.1 -> scale 0.21, symbols [5, 5]."""
    k = GOLDEN["known"]["eb_hand"]
    assert k["symbols"] == [5, 5] and abs(k["scale"] - 0.21) < 1e-12
    out = np.zeros(2, np.int32)
    assert port.lib.zo_eb_quantize_f64(np.array(k["x"]), 2, k["scale"], out) == 0
    assert out.tolist() == [5, 5]


@pytest.mark.parametrize("nm,width,payload", [("hand", 3, [0x50, 0x08]), ("zeros", 1, [0x00]), ("full_width", 32, None)])
def test_fixedlen_known_answers(port, nm, width, payload):
    """test_fixedlen.cpp:51-75 (hand-packed 0x50 0x08; all-zero width 1) and :115-125 (width 32, 16 B)."""
    k = GOLDEN["known"][f"fixedlen_{nm}"]
    assert k["width"] == width and (payload is None or k["payload"] == payload)
    p, w = port.fixedlen_encode(np.array(k["symbols"], np.int32))
    assert w == width and p.tolist() == k["payload"] and len(p) == (len(k["symbols"]) * width + 7) // 8


@pytest.mark.parametrize("nm", ["single42", "two_equal", "geometric8", "fibonacci60"] + [f"random{i}" for i in range(6)])
def test_huffman_context_matches_reference(port, nm):
    """huffman_build_context (huffman.cpp:23-173): lengths, canonical codes, reversed codes, LUT;
    single symbol -> 1 bit, two equal bins -> 1 bit each (test_huffman.cpp:55-76); Fibonacci
    weights exercise the 32-bit cap repair (test_huffman.cpp:205-231)."""
    k = GOLDEN["known"][f"huff_{nm}"]
    h = np.array(k["hist"], np.uint64)
    ctx = port.huff_from_hist(h)
    assert ctx.valid == k["valid"]
    assert list(ctx.len) == k["lens"] and list(ctx.code) == k["code"] and list(ctx.rev) == k["rev"]
    assert sha(np.array(ctx.lut, np.uint16)) == k["lut_sha256"]
    bits = C.c_double()
    ok = port.lib.zo_huff_expected_len(C.byref(ctx), h, C.byref(bits))
    assert (bits.value if ok else None) == k["expected_len"]
    if nm == "single42":
        assert k["lens"][42] == 1 and sum(k["lens"]) == 1
    if nm == "two_equal":
        assert k["lens"][0] == 1 and k["lens"][255] == 1 and k["expected_len"] == 1.0
    if nm == "fibonacci60":
        assert max(k["lens"]) <= abi.HUFF_MAX_CODE_LEN
        assert sum(2.0 ** -l for l in k["lens"] if l) <= 1.0 + 1e-12


def test_huffman_embedded_repeated_byte(port):
    """test_huffman.cpp:112-123: 1000 x byte 7 with embedded codebook -> 256 + ceil(1000/8) bytes."""
    k = GOLDEN["known"]["huff_embedded_repeat"]
    assert k["payload"] == 256 + (1000 + 7) // 8
    raw = np.full(1000, 7, np.uint8)
    ctx = port.huff_from_hist(np.bincount(raw, minlength=256).astype(np.uint64))
    assert len(port.huffman_encode(raw, ctx, embed=True)) == k["payload"]


# ------------------------------------------------------------------ collectives
def test_symbol_sum_and_scale_reconciliation(port):
    """test_collectives.cpp:83-118: {r+1, -(r+1), 100} at 4 ranks -> {10, -10, 400}; rank scales
    {0.5, 1.0} reconcile to 1.0 with llround requantization -> {6, -1, 5, 8}."""
    for nm in ("symsum4", "reconcile2"):
        k = GOLDEN["collectives"][nm]
        rc, out, sc, _ = port.ring_allreduce(np.array(k["in"], np.int32), np.array(k["scales_in"]))
        assert rc == 0
        assert out.tolist() == k["out"] and sc.tolist() == k["scales_out"]
    assert GOLDEN["collectives"]["symsum4"]["out"][0] == [10, -10, 400]
    assert GOLDEN["collectives"]["reconcile2"]["out"][0] == [6, -1, 5, 8]


@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("pin", ["auto", "raw", "fixedlen", "huffman"])
def test_ring_allreduce_matches_reference(port, n, pin):
    """Ring RS (compressed, int32 sum) + AG (collectives.cpp:462-502) over 6 MiB per rank: output
    symbols and WireStats identical to the reference Communicator's."""
    k = GOLDEN["collectives"][f"ring{n}_{pin}"]
    base = ring_input(n)
    assert sha(base) == GOLDEN["collectives"][f"ring{n}_input_sha256"]
    ctx = port.huff_from_bytes(np.ascontiguousarray(base[0].view(np.uint8)[: abi.BATCH_RAW_BYTES]))
    rc, out, _, w = port.ring_allreduce(base, np.full(n, 2e-4), pin=k["pin"], ctx=ctx)
    assert rc == 0
    assert all((out[r] == out[0]).all() for r in range(n))
    assert sha(out[0]) == k["out_sha256"]
    assert list(w.frames_by_codec) == k["wire"]["frames_by_codec"]
    assert (w.raw_bytes, w.payload_bytes, w.total_bytes) == (k["wire"]["raw_bytes"], k["wire"]["payload_bytes"],
                                                              k["wire"]["total_bytes"])


@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("pin", ["auto", "raw", "fixedlen", "huffman"])
def test_ring_allreduce_per_slot_matches_reference(port, n, pin):
    """CollectiveConfig::perSlotFraming: the same ring with 512 KiB batches (collectives.cpp:197-199,
    366-396): symbols and WireStats identical to the reference Communicator's, and the frame count
    is the per-slot one (not the 4 MiB batches')."""
    k = GOLDEN["collectives"][f"ring{n}_{pin}_slot"]
    base = ring_input(n)
    ctx = port.huff_from_bytes(np.ascontiguousarray(base[0].view(np.uint8)[: abi.BATCH_RAW_BYTES]))
    rc, out, _, w = port.ring_allreduce(base, np.full(n, 2e-4), pin=k["pin"], ctx=ctx, per_slot=True)
    assert rc == 0
    assert sha(out[0]) == k["out_sha256"]
    assert list(w.frames_by_codec) == k["wire"]["frames_by_codec"]
    assert (w.raw_bytes, w.payload_bytes, w.total_bytes) == (k["wire"]["raw_bytes"], k["wire"]["payload_bytes"],
                                                              k["wire"]["total_bytes"])
    assert sum(w.frames_by_codec) > sum(GOLDEN["collectives"][f"ring{n}_{pin}"]["wire"]["frames_by_codec"])


@pytest.mark.parametrize("n", [2, 3, 4])
def test_ring_allgather_matches_reference(port, n):
    """RankCtx::allgather (collectives.cpp:525-544)."""
    k = GOLDEN["collectives"][f"allgather{n}"]
    blk = ring_input(n)[:, : k["block"]]
    rc, out, w = port.ring_allgather(blk)
    assert rc == 0 and all(sha(out[r]) == k["out_sha256"] and (out[r] == blk.ravel()).all() for r in range(n))
    assert list(w.frames_by_codec) == k["wire"]["frames_by_codec"]
    assert w.payload_bytes == k["wire"]["payload_bytes"]


# ------------------------------------------------------------------ live differential (compiled reference)
def test_quantizer_differential(port, ref):
    """eb_quantize_with_scale (quant.cpp:22-27, 43-62): symbols and the error on out-of-range."""
    rng = np.random.default_rng(3)
    for scale in (2e-4, 1e-3, 0.21, 1.0, 3.0e-9):
        x = np.concatenate([rng.standard_normal(5000), (np.arange(-50, 50) + 0.5) * scale,
                            np.array([0.0, -0.0, 1e-300, -1e-300])]).astype(np.float32).astype(np.float64)
        a = np.zeros(len(x), np.int32)
        b = np.zeros(len(x), np.int32)
        ra = port.lib.zo_eb_quantize_f64(x, len(x), scale, a)
        rb = ref.lib.zr_eb_quantize_with_scale(x, len(x), scale, b)
        assert (ra == 0) == (rb == 0), scale
        if ra == 0:
            assert (a == b).all(), scale
    for bad in (np.array([2147483647.5]), np.array([np.inf]), np.array([np.nan]), np.array([-2147483648.6])):
        a = np.zeros(1, np.int32)
        b = np.zeros(1, np.int32)
        assert port.lib.zo_eb_quantize_f64(bad, 1, 1.0, a) != 0
        assert ref.lib.zr_eb_quantize_with_scale(bad, 1, 1.0, b) != 0


def test_encode_best_fuzz_differential(port, ref):
    """Random structured batches (fuzz in the spirit of acceptance.cpp:416-496): frames identical."""
    rng = np.random.default_rng(11)
    for t in range(60):
        n = int(rng.choice([1, 3, 4, 4095, 4096, 4097, 65535, 65536, 65537, 200000, 1 << 20]))
        kind = t % 4
        if kind == 0:
            raw = rng.integers(0, 256, n, dtype=np.uint8)
        elif kind == 1:
            raw = rng.geometric(rng.uniform(0.05, 0.9), n).clip(0, 255).astype(np.uint8)
        elif kind == 2:
            raw = (rng.standard_normal((n + 3) // 4) * rng.uniform(1, 1e5)).astype(np.int32).view(np.uint8)[:n].copy()
        else:
            raw = np.zeros(n, np.uint8)
            raw[rng.integers(0, n, max(1, n // 100))] = rng.integers(0, 256, max(1, n // 100))
        hint = abi.make_hint(float(rng.choice([1e9, 1e10, 1.0737e10, 2e11, 9e11])))
        cap = int(rng.choice([abi.STAGE_BANK_BYTES, n + 32, max(33, n // 2), 40]))
        pc = port.huff_from_bytes(raw[: 1 << 16]) if t % 3 else None
        rc = ref.huff_from_bytes(raw[: 1 << 16]) if t % 3 else None
        a, fa = port.encode_best(raw, hint, pc, cap=cap)
        b, fb = ref.encode_best(raw, hint, rc, cap=cap)
        if rc is not None:
            ref.lib.zr_huff_ctx_free(rc)
        assert (a.codec, a.payload_bytes, a.total_bytes) == (b.codec, b.payload_bytes, b.total_bytes), (t, n, cap)
        assert bytes(fa) == bytes(fb), (t, n, cap)


def test_gen_data_matches_reference(port, ref):
    """gen_data (bench.cpp:49-68, 463-476): Uniform / Gaussian / Geometric streams, with offsets."""
    for dist in (0, 1, 2):
        for seed, rank, off in ((1, 0, 0), (5, 3, 1000), (9, 1, 77)):
            a = port.gen_data(dist, seed, rank, 5000, off)
            b = np.zeros(5000)
            assert ref.lib.zr_gen_data(dist, 0.7, seed, rank, off, 5000, b) == 0
            assert (a == b).all(), (dist, seed, rank, off)


def test_qsgd_restatement_matches_reference():
    """zo_qsgd_quantize_f32 / zo_mt19937_64 (zc_oracle.c) against the compiled reference's
    qsgd_quantize / std::mt19937_64 (quant.cpp:64-98), including the C++ standard's known answer."""
    import oracle
    try:
        ref = oracle.ref()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"compiled reference unavailable: {e}")
    port = oracle.port()
    assert int(ref.mt19937_64(5489, 9999, 1)[0]) == 9981545732273789042
    rng = np.random.default_rng(0)
    for n, lv, seed in [(0, 4, 1), (1, 1, 2), (1000, 15, 3), (100003, 255, 1234567), (5000, 1 << 30, 9)]:
        x = rng.standard_normal(n).astype(np.float32)
        a = port.qsgd_quantize_f32(x, lv, seed)
        b = ref.qsgd_quantize(x.astype(np.float64), lv, seed)
        assert a[0] == b[0] == 0 and a[2] == b[2] and np.array_equal(a[1], b[1])
    x = rng.standard_normal(7777).astype(np.float32)
    a = port.qsgd_quantize_chunk_f32(x, 7, 3.5, 42, 1000)
    b = ref.qsgd_quantize_chunk(x.astype(np.float64), 7, 3.5, 42, 1000)
    assert np.array_equal(a[1], b[1])
