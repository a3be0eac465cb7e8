"""GPU parity: quantizer, frame, FixedLen, Huffman, selector and encode_best on sm_100a vs the
oracle (oracle/zc_oracle.c, itself pinned to the compiled reference in test_oracle.py).

Bar: bit-exact symbols, selector decisions, frame bytes; round trips exact."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2605_12396_b200 import abi

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]
DEV = "cuda"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def npy(x):
    return x.cpu().numpy()


def hdr(codec, raw, payload, params, flags=0):
    h = abi.FrameHeader()
    h.magic, h.version, h.codec, h.flags = abi.FRAME_MAGIC, abi.FRAME_VERSION, codec, flags
    h.raw_bytes, h.payload_bytes, h.params = raw, payload, params
    return h


# ------------------------------------------------------------------ quantizer
def _tie_heavy(n, scale, rng):
    """Values whose quotient lands exactly on / right next to half-integers."""
    k = rng.integers(-30000, 30000, n).astype(np.float64)
    x = (k + 0.5) * scale
    x[::3] = np.nextafter(x[::3], np.inf)
    x[1::3] = np.nextafter(x[1::3], -np.inf)
    return x


@pytest.mark.parametrize("scale", [2e-4, 0.21, 1.0, 3.0e-7, 0.1])
def test_quantize_f64_bitexact(zc, port, scale):
    rng = np.random.default_rng(1)
    x = np.concatenate([rng.normal(0, 3, 200001), _tie_heavy(50000, scale, rng), [0.0, -0.0, scale / 2, -scale / 2]])
    got = npy(zc.eb_quantize_with_scale(t(x), scale))
    exp = np.zeros(len(x), np.int32)
    assert port.lib.zo_eb_quantize_f64(x, len(x), scale, exp) == 0
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("scale", [2e-4, 2e-3 * 3.7, 1e-6])
def test_quantize_f32_bitexact(zc, port, scale):
    rng = np.random.default_rng(2)
    x = np.concatenate([rng.normal(0, 1, 1 << 20), _tie_heavy(1 << 16, scale, rng)]).astype(np.float32)
    got = npy(zc.eb_quantize_with_scale(t(x), scale))
    rc, exp = port.eb_quantize_f32(x, scale)
    assert rc == 0 and np.array_equal(got, exp)


def test_quantize_hand_example_and_errors(zc):
    # quant.cpp hand example (test_quant.cpp:20-30): [1.0, 1.05], rel 0.1 -> scale 0.21, symbols [5, 5]
    sym, scale = zc.eb_quantize(t(np.array([1.0, 1.05], np.float32)), 0.1)
    assert abs(scale - 0.21) < 1e-7 and npy(sym).tolist() == [5, 5]
    sym, scale = zc.eb_quantize(t(np.zeros(3, np.float32)), 1e-4)
    assert scale == 1.0 and npy(sym).tolist() == [0, 0, 0]
    with pytest.raises(ValueError):
        zc.eb_quantize_with_scale(t(np.array([1.0, np.nan])), 0.1)
    with pytest.raises(ValueError):
        zc.eb_quantize_with_scale(t(np.array([np.inf])), 0.1)
    with pytest.raises(ValueError):
        zc.eb_quantize_with_scale(t(np.array([3.0e9])), 1.0)
    with pytest.raises(ValueError):
        zc.eb_quantize(t(np.array([1.0], np.float32)), 1.5)
    with pytest.raises(ValueError):
        zc.eb_quantize_with_scale(t(np.array([1.0])), 0.0)


def test_dequantize_bitexact(zc, port):
    rng = np.random.default_rng(3)
    s = rng.integers(-2**31, 2**31, 100003, dtype=np.int64).astype(np.int32)
    for mode, scale, levels in [(0, 2e-4, 0), (1, 3.75, 7), (2, 1.0, 0)]:
        exp = np.zeros(len(s))
        port.lib.zo_dequantize_f64(s, len(s), mode, scale, levels, exp)
        got = npy(zc.dequantize(t(s), mode, scale, levels, torch.float64))
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64))
        got32 = npy(zc.dequantize(t(s), mode, scale, levels, torch.float32))
        assert np.array_equal(got32, exp.astype(np.float32))


# ------------------------------------------------------------------ frame
def test_header_roundtrip_and_validate(zc, port):
    rng = np.random.default_rng(4)
    for _ in range(200):
        h = hdr(int(rng.integers(0, 3)), int(rng.integers(1, 2**40)), int(rng.integers(0, 2**40)),
                int(rng.integers(0, 2**63)), int(rng.integers(0, 2**16)))
        b = zc.write_header(h)
        ob = np.zeros(32, np.uint8)
        port.lib.zo_write_header(C.byref(h), ob)
        assert b == ob.tobytes()
        g = zc.parse_header(b)
        assert (g.magic, g.codec, g.raw_bytes, g.payload_bytes, g.params, g.flags) == \
            (h.magic, h.codec, h.raw_bytes, h.payload_bytes, h.params, h.flags)
        for region in (31, 32, 33, h.payload_bytes + 32, h.payload_bytes + 31):
            assert zc.validate_header(h, region) == bool(port.lib.zo_validate_header(C.byref(h), region))
    assert zc.parse_header(b"\0" * 31) is None


def test_commit_raw_capacity(zc):
    raw = t(np.arange(8, dtype=np.uint8))
    assert zc.frame_commit_raw(raw, torch.zeros(40, dtype=torch.uint8, device=DEV)) == 40
    assert zc.frame_commit_raw(raw, torch.zeros(39, dtype=torch.uint8, device=DEV)) == 0


# ------------------------------------------------------------------ fixedlen
def test_fixedlen_golden(zc):
    # test_fixedlen.cpp:51-75, 115-125
    p, w = zc.fixedlen_encode(t(np.array([0, 1, -1, 2], np.int32)), 8)
    assert w == 3 and npy(p).tolist() == [0x50, 0x08]
    p, w = zc.fixedlen_encode(t(np.zeros(4, np.int32)), 8)
    assert w == 1 and npy(p).tolist() == [0]
    p, w = zc.fixedlen_encode(t(np.array([-2**31, 2**31 - 1, 0, -1], np.int32)), 32)
    assert w == 32 and p.numel() == 16
    ok, back = zc.fixedlen_decode(hdr(1, 16, 16, 32), p, 16)
    assert ok and npy(back).view(np.int32).tolist() == [-2**31, 2**31 - 1, 0, -1]
    p, w = zc.fixedlen_encode(t(np.array([100, -200, 300], np.int32)), 2)
    assert p.numel() == 0


def test_fixedlen_random_vs_oracle(zc, port):
    rng = np.random.default_rng(9)
    for it in range(60):
        n = int(rng.integers(1, 5000)) if it % 3 else int(rng.integers(100000, 300000))
        shift = int(rng.integers(0, 28))
        s = (rng.integers(-2**31, 2**31, n, dtype=np.int64) >> shift).astype(np.int32)
        cap = 4 * n + 8
        out = np.zeros(cap, np.uint8)
        w = C.c_uint32()
        pn = port.lib.zo_fixedlen_encode(s, n, out, cap, C.byref(w))
        got, gw = zc.fixedlen_encode(t(s), cap)
        assert gw == w.value and got.numel() == pn
        assert np.array_equal(npy(got), out[:pn])
        ok, back = zc.fixedlen_decode(hdr(1, 4 * n, pn, gw), got, 4 * n)
        assert ok and np.array_equal(npy(back).view(np.int32), s)


def test_fixedlen_decode_rejects(zc):
    p, w = zc.fixedlen_encode(t(np.array([1, 2, 3, 4, 5], np.int32)), 32)
    assert not zc.fixedlen_decode(hdr(1, 20, p.numel(), 0), p, 20)[0]
    assert not zc.fixedlen_decode(hdr(1, 20, p.numel(), 33), p, 20)[0]
    assert not zc.fixedlen_decode(hdr(1, 18, p.numel(), w), p, 20)[0]
    assert not zc.fixedlen_decode(hdr(1, 20, p.numel() - 1, w), p, 20)[0]
    assert not zc.fixedlen_decode(hdr(1, 20, p.numel(), w), p, 19)[0]


# ------------------------------------------------------------------ huffman
def _hist(b):
    return np.bincount(np.asarray(b, np.uint8), minlength=256).astype(np.uint64)


def test_huffman_context_matches_oracle(zc, port):
    rng = np.random.default_rng(5)
    cases = [np.array([1, 1, 2, 2] + [0] * 252, np.uint64)]
    cases[0] = np.zeros(256, np.uint64)
    cases[0][[10, 20, 30, 40]] = [1, 1, 2, 2]
    fib = np.zeros(256, np.uint64)
    a, b = 1, 1
    for i in range(40):
        fib[i] = a
        a, b = b, a + b
    cases.append(fib)
    for _ in range(60):
        h = np.zeros(256, np.uint64)
        live = int(rng.integers(1, 256))
        h[rng.choice(256, live, replace=False)] = rng.integers(1, 10**6, live)
        cases.append(h)
    for h in cases:
        c = zc.HuffmanContext.from_hist(h)
        o = port.huff_from_hist(h)
        assert c.valid == bool(o.valid)
        assert c.code_lengths == list(o.len)
        code, rev = c.codes()
        assert code == list(o.code) and rev == list(o.rev)
    # tie-break pin: weights {1,1,2,2} on {10,20,30,40} -> all length 2
    c = zc.HuffmanContext.from_hist(cases[0])
    assert [c.code_lengths[s] for s in (10, 20, 30, 40)] == [2, 2, 2, 2]
    assert not zc.HuffmanContext.from_hist(np.zeros(256, np.uint64)).valid


@pytest.mark.parametrize("n", [1, 100, 1023, 1024, 1025, 65536, 300001, 4 << 20])
def test_huffman_encode_decode_vs_oracle(zc, port, n):
    rng = np.random.default_rng(n)
    raw = np.minimum(rng.geometric(0.3, n) - 1, 255).astype(np.uint8)
    sample = raw[: min(n, 1 << 20)]
    c = zc.HuffmanContext.from_bytes(sample)
    o = port.huff_from_bytes(sample)
    cap = 2 * n + 64
    out = np.zeros(cap, np.uint8)
    pn = port.lib.zo_huffman_encode(raw, n, C.byref(o), out, cap, 0)
    got, idx = zc.huffman_encode(t(raw), c, cap, with_index=True)
    assert got.numel() == pn and np.array_equal(npy(got), out[:pn])
    h = hdr(2, n, pn, 0)
    ok, back = zc.huffman_decode(h, got, c, n, index=idx)
    assert ok and np.array_equal(npy(back), raw)
    if n <= 65536:  # sequential path (frames without a companion index)
        ok, back = zc.huffman_decode(h, got, c, n)
        assert ok and np.array_equal(npy(back), raw)


def test_huffman_embedded_and_failures(zc, port):
    raw = np.full(1000, 7, np.uint8)
    c = zc.HuffmanContext.from_hist(_hist(raw))
    p = zc.huffman_encode(t(raw), c, 256 + 1000, embed=True)
    assert p.numel() == 256 + 125  # test_huffman.cpp:112-123
    ok, back = zc.huffman_decode(hdr(2, 1000, p.numel(), 256, abi.FLAG_EMBEDDED_CODEBOOK), p, None, 1000)
    assert ok and np.array_equal(npy(back), raw)
    # unseen symbol under the shared context -> failure sentinel 0
    c2 = zc.HuffmanContext.from_hist(_hist(np.array([1, 2, 3], np.uint8)))
    assert zc.huffman_encode(t(np.array([1, 9], np.uint8)), c2, 64).numel() == 0
    # capacity shortfall
    assert zc.huffman_encode(t(np.arange(256, dtype=np.uint8)), zc.HuffmanContext.from_bytes(b""), 10).numel() == 0
    # shared frame without a context / with params != 0
    p = zc.huffman_encode(t(raw), c, 2000)
    assert not zc.huffman_decode(hdr(2, 1000, p.numel(), 0), p, None, 1000)[0]
    assert not zc.huffman_decode(hdr(2, 1000, p.numel(), 5), p, c, 1000)[0]
    # truncated stream -> overrun
    assert not zc.huffman_decode(hdr(2, 1000, p.numel() - 1, 0), p[:-1], c, 1000)[0]


# ------------------------------------------------------------------ selector
def _stats_equal(a, b):
    return (a.sampled_bytes == b.sampled_bytes and list(a.hist) == list(b.hist) and a.max_zigzag == b.max_zigzag
            and a.ctx_code_len_valid == b.ctx_code_len_valid and a.self_code_len_valid == b.self_code_len_valid
            and (not a.ctx_code_len_valid or a.ctx_code_len_bits == b.ctx_code_len_bits)
            and (not a.self_code_len_valid or a.self_code_len_bits == b.self_code_len_bits))


@pytest.mark.parametrize("n", [0, 3, 4096, 65535, 65536, 65537, 1 << 20])
def test_profile_sample_vs_oracle(zc, port, n):
    rng = np.random.default_rng(n + 11)
    raw = (rng.normal(0, 300, (n + 3) // 4).astype(np.int32)).view(np.uint8)[:n]
    sample = raw[: min(n, 1 << 16)]
    c = zc.HuffmanContext.from_bytes(sample)
    o = port.huff_from_bytes(sample)
    for with_ctx in (False, True):
        got = zc.profile_sample(t(raw) if n else torch.zeros(0, dtype=torch.uint8, device=DEV), c if with_ctx else None)
        exp = port.profile(raw, o if with_ctx else None)
        assert _stats_equal(got, exp)


def test_arbitrate_random_triples_vs_oracle(zc, port):
    """Host build of the selector vs the oracle (test_rea.cpp:186-225 style)."""
    rng = np.random.default_rng(63)
    shared = port.huff_from_bytes(np.minimum(rng.geometric(0.3, 65536) - 1, 255).astype(np.uint8))
    gshared = zc.HuffmanContext.from_lengths(list(shared.len))
    for k in range(300):
        p = 0.05 + 0.9 * rng.random()
        raw = np.minimum(rng.geometric(p, 8192 + int(rng.integers(0, 65536))) - 1, 255).astype(np.uint8)
        use = k % 3 != 0
        st = port.profile(raw, shared if use else None)
        cfg = abi.default_arb_config()
        cfg.min_gain_permil = int(rng.integers(0, 200))
        cfg.lam_enc = int(rng.integers(0, 101)) / 100.0
        cfg.lam_dec = int(rng.integers(0, 101)) / 100.0
        cfg.embed_codebook = 1 if k % 4 == 0 else 0
        cfg.huffman_min_raw_bytes = 1 << int(rng.integers(10, 18))
        hint = abi.make_hint(10 ** (8 + 3.5 * rng.random()), k & 1)
        cap = len(raw) // 2 + int(rng.integers(0, 2 * len(raw)))
        plan = zc.arbitrate_plan(len(raw), cap, st, hint, gshared if use else None, cfg)
        exp = abi.ArbitrationPlan()
        port.lib.zo_arbitrate_plan(len(raw), cap, C.byref(st), C.byref(hint), C.byref(shared) if use else None,
                                   C.byref(cfg), C.byref(exp))
        assert bytes(plan) == bytes(exp)


def _stream_cases():
    rng = np.random.default_rng(79)
    geo = np.minimum(rng.geometric(0.7, 1 << 20) - 1, 255).astype(np.int32)
    return {
        "const0": np.zeros(1 << 20, np.int32),
        "narrow": (rng.integers(0, 7, 60000) - 3).astype(np.int32),
        "wide_skew": np.where(rng.integers(0, 2, 60000) == 1, 0x40000000, -0x40000000).astype(np.int32),
        "noise": rng.integers(0, 256, 240000).astype(np.uint8),
        "geometric": geo,
        "gauss": (rng.normal(0, 1, 1 << 20) / 2e-4).round().astype(np.int32),
        "small": np.arange(1000, dtype=np.int32),
        "odd_bytes": rng.integers(0, 4, 100003).astype(np.uint8),
        "adversarial": np.concatenate([np.zeros(64 * 1024, np.uint8), rng.integers(0, 256, 192 * 1024).astype(np.uint8)]),
    }


@pytest.mark.parametrize("beta", [1.0e9, 10 * 2**30, 200 * 2**30, 900e9])
def test_encode_best_frames_vs_oracle(zc, port, beta):
    cases = _stream_cases()
    sample = cases["wide_skew"].view(np.uint8)
    c, o = zc.HuffmanContext.from_bytes(sample), port.huff_from_bytes(sample)
    cfg = abi.default_arb_config()
    cfg.huffman_min_raw_bytes = 16 * 1024
    hint = abi.make_hint(beta)
    for name, arr in cases.items():
        raw = arr.view(np.uint8)
        for cap in (abi.STAGE_BANK_BYTES, len(raw) + 32, len(raw) // 2 + 40):
            r, frame = zc.encode_best(t(raw), cap, hint, c, cfg)
            er = abi.EncodeResult()
            stage = np.zeros(cap, np.uint8)
            port.lib.zo_encode_best(raw, len(raw), stage, cap, C.byref(hint), C.byref(o), C.byref(cfg), C.byref(er))
            assert (r.codec, r.payload_bytes, r.total_bytes) == (er.codec, er.payload_bytes, er.total_bytes), (name, cap)
            assert np.array_equal(npy(frame), stage[: er.total_bytes]), (name, cap)


def test_encode_best_degenerate(zc):
    hint = abi.make_hint(1e10)
    r, _ = zc.encode_best(torch.zeros(0, dtype=torch.uint8, device=DEV), 1024, hint)
    assert r.total_bytes == 0
    raw = t(np.ones(100, np.uint8))
    assert zc.encode_best(raw, 32, hint)[0].total_bytes == 0
    assert zc.encode_best(raw, 82, hint)[0].total_bytes == 0
    r, f = zc.encode_best(t(np.zeros(4096, np.uint8)), abi.STAGE_BANK_BYTES, abi.make_hint(1e9))
    assert (r.codec, r.payload_bytes, r.total_bytes) == (0, 4096, 4128)


def test_selector_stress_c4(zc, port):
    """BASELINE config 4: constant / low-entropy / uniform batches -> FixedLen / Huffman / RAW at 10 GiB/s."""
    rng = np.random.default_rng(0xC4)
    b0 = np.zeros(1 << 20, np.int32)
    x = port.gen_data(2, 5, 0, 1 << 20, geom_p=0.7)
    amax = np.abs(x).max()
    b1 = np.zeros(1 << 20, np.int32)
    port.lib.zo_eb_quantize_f64(x, len(x), 2 * 1e-4 * amax, b1)
    b2 = rng.integers(0, 2**32, 1 << 20, dtype=np.uint64).astype(np.uint32).view(np.int32)
    msg = np.concatenate([b0, b1, b2])
    sample = msg.view(np.uint8)
    c, o = zc.HuffmanContext.from_bytes(sample), port.huff_from_bytes(sample)
    fr = zc.encode_batches(t(msg), abi.PIN_AUTO, ctx=c)
    codecs = [r.codec for r in fr.encode_results()]
    exp = port.encode_batches(msg, abi.PIN_AUTO, ctx=o)
    assert codecs == [e[0].codec for e in exp] == [abi.CODEC_FIXEDLEN, abi.CODEC_HUFFMAN, abi.CODEC_RAW]
    for b, (er, ef) in enumerate(exp):
        assert np.array_equal(npy(fr.frame(b)), ef)
    back = zc.decode_batches(fr, c)
    assert np.array_equal(npy(back), msg)


# ------------------------------------------------------------------ batched hot path
@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_RAW, abi.PIN_FIXEDLEN, abi.PIN_HUFFMAN])
@pytest.mark.parametrize("count", [1000, 1 << 20, (9 << 20) // 4 + 3])
def test_encode_batches_f32_fused_vs_oracle(zc, port, pin, count):
    rng = np.random.default_rng(count + pin)
    x = rng.normal(0, 1, count).astype(np.float32)
    scale = 2e-4
    rc, sym = port.eb_quantize_f32(x, scale)
    assert rc == 0
    raw = sym.view(np.uint8)
    sample = raw[: 4 << 20]
    c, o = zc.HuffmanContext.from_bytes(sample), port.huff_from_bytes(sample)
    hint = abi.make_hint()
    fr = zc.encode_batches(t(x), pin, scale=scale, hint=hint, ctx=c)
    fr2 = zc.encode_batches(t(sym), pin, hint=hint, ctx=c)
    exp = port.encode_batches(raw, pin, hint, o)
    assert fr.nbatches == len(exp)
    for b, (er, ef) in enumerate(exp):
        for f in (fr, fr2):
            r = f.encode_results()[b]
            assert (r.codec, r.payload_bytes, r.total_bytes) == (er.codec, er.payload_bytes, er.total_bytes)
            assert np.array_equal(npy(f.frame(b)), ef)
    assert np.array_equal(npy(zc.decode_batches(fr, c)), sym)
    y = npy(zc.decode_batches(fr, c, scale=scale))
    deq = np.zeros(count, np.float32)
    port.lib.zo_dequantize_f32(sym, count, 0, scale, 0, deq)
    assert np.array_equal(y, deq)
    assert np.max(np.abs(y.astype(np.float64) - x)) <= scale / 2 * (1 + 1e-6) + 1e-7


def test_decode_fallback_on_corrupt_header(zc, port):
    rng = np.random.default_rng(0xC5)
    sym = (rng.integers(0, 512, 300000) - 256).astype(np.int32)
    fr = zc.encode_batches(t(sym), abi.PIN_AUTO)
    # corrupt the magic of the only frame: raw-copy fallback of the payload region
    fr.stages[0] ^= 0xFF
    codecs = torch.zeros(1, dtype=torch.int32, device=DEV)
    out = zc.decode_batches(fr, None, codecs=codecs)
    frame = npy(fr.stages[: fr.encode_results()[0].total_bytes])
    cdc, exp = port.recv_batch(frame, len(sym) * 4)
    assert cdc == -1 and int(codecs.item()) == -1
    have = len(frame) - 32  # min(dst, have) bytes are the payload region verbatim (collectives.cpp:330-336)
    assert np.array_equal(npy(out).view(np.uint8)[:have], exp[:have])


# ------------------------------------------------------------------ fp32 fast path (zc_fixed.cu)
@pytest.mark.parametrize("sigma,scale", [(0.0, 2e-4), (1e-4, 2e-4), (1.0, 2e-4), (3.0, 1e-3), (1.0, 1e-6),
                                         (100.0, 1e-6), (150.0, 1e-6), (300.0, 1e-6)])
@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_FIXEDLEN, abi.PIN_RAW])
def test_fixed_path_widths_vs_oracle(zc, port, sigma, scale, pin):
    """Every FixedLen width from 1 to 32 (and RAW) through the TMA emit / decode kernels, with
    values placed on exact rounding ties and near the int32 limit, frames byte-compared with the
    oracle and the decoded fp32 compared with dequantize_into."""
    rng = np.random.default_rng(int(sigma * 7) + pin)
    count = (6 << 20) // 4 + 1029  # one full unit, one ragged unit with a partial tile
    x = (rng.normal(0, 1, count) * sigma).astype(np.float32)
    k = rng.integers(-1000, 1000, 4096)
    x[rng.integers(0, count, 4096)] = ((k + 0.5) * scale).astype(np.float32)  # ties (after fp32 rounding: near ties)
    rc, sym = port.eb_quantize_f32(x, scale)
    assert rc == 0
    raw = sym.view(np.uint8)
    hint = abi.make_hint()
    fr = zc.encode_batches(t(x), pin, scale=scale, hint=hint)
    exp = port.encode_batches(raw, pin, hint, None)
    for b, (er, ef) in enumerate(exp):
        r = fr.encode_results()[b]
        assert (r.codec, r.payload_bytes, r.total_bytes) == (er.codec, er.payload_bytes, er.total_bytes)
        assert np.array_equal(npy(fr.frame(b)), ef), f"frame {b}"
    y = npy(zc.decode_batches(fr, None, scale=scale))
    deq = np.zeros(count, np.float32)
    port.lib.zo_dequantize_f32(sym, count, 0, scale, 0, deq)
    assert np.array_equal(y, deq)
    assert np.array_equal(npy(zc.decode_batches(fr, None)), sym)


def test_fixed_path_matches_generic_kernels(zc, monkeypatch):
    """The fast kernels and the generic batch kernels (ZC_NO_FIXED) produce identical frames."""
    rng = np.random.default_rng(11)
    x = rng.laplace(0, 1e-2, (9 << 20) // 4 + 5).astype(np.float32)
    fast = zc.encode_batches(t(x), abi.PIN_AUTO, scale=2e-4)
    monkeypatch.setenv("ZC_NO_FIXED", "1")
    slow = zc.encode_batches(t(x), abi.PIN_AUTO, scale=2e-4)
    ys = npy(zc.decode_batches(slow, None, scale=2e-4))
    monkeypatch.delenv("ZC_NO_FIXED")
    yf = npy(zc.decode_batches(fast, None, scale=2e-4))
    for b in range(fast.nbatches):
        assert np.array_equal(npy(fast.frame(b)), npy(slow.frame(b)))
    assert np.array_equal(yf, ys)


def test_codec_roundtrip_host_pipeline(zc):
    """zc_codec_roundtrip_host_f32 (pinned host in -> frames -> pinned host out) equals the
    device-resident encode + decode, frames included."""
    import ctypes as C
    L = zc.lib()
    rng = np.random.default_rng(5)
    count = (21 << 20) // 4 + 7
    x = rng.normal(0, 1, count).astype(np.float32)
    hx = torch.from_numpy(x).pin_memory()
    hy = torch.empty(count, dtype=torch.float32).pin_memory()
    work = torch.empty(count, dtype=torch.float32, device=DEV)
    fr = zc.alloc_frames(count * 4, DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    hint, cfg = abi.make_hint(), zc.default_arb_config()
    s = torch.cuda.current_stream()
    zc.check(L.zc_codec_roundtrip_host_f32(hx.data_ptr(), count, 2e-4, zc._ptr(work), zc._ptr(fr.stages),
                                           zc.STAGE_STRIDE, abi.STAGE_BANK_BYTES, abi.PIN_AUTO, C.byref(hint), None,
                                           C.byref(cfg), zc._ptr(fr.results), zc._ptr(fr.index), zc._ptr(err),
                                           hy.data_ptr(), 2, C.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    ref = zc.encode_batches(t(x), abi.PIN_AUTO, scale=2e-4)
    for b in range(ref.nbatches):
        assert np.array_equal(npy(fr.frame(b)), npy(ref.frame(b)))
    assert torch.equal(hy, zc.decode_batches(ref, None, scale=2e-4).cpu())


@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_HUFFMAN])
def test_embedded_codebook_batches_vs_oracle(zc, port, pin):
    """cfg.embed_codebook end to end (rea.cpp:214-221, huffman.cpp:256-262): every
    batch builds its own tree from its full histogram and ships the 256 code lengths in the frame;
    frames byte-equal to the reference's send_batch, and recv_batch decodes them without a
    shared context."""
    cases = _stream_cases()
    msg = np.concatenate([cases["geometric"].view(np.uint8), cases["adversarial"], cases["narrow"].view(np.uint8)])
    cfg = abi.default_arb_config()
    cfg.embed_codebook = 1
    hint = abi.make_hint(1e9)
    fr = zc.encode_batches(t(msg), pin, hint=hint, cfg=cfg)
    exp = port.encode_batches(msg, pin, hint, None, cfg)
    assert fr.nbatches == len(exp)
    codecs = []
    for b, (er, ef) in enumerate(exp):
        r = fr.encode_results()[b]
        assert (r.codec, r.payload_bytes, r.total_bytes) == (er.codec, er.payload_bytes, er.total_bytes), b
        assert np.array_equal(npy(fr.frame(b)), ef), b
        codecs.append(r.codec)
    assert abi.CODEC_HUFFMAN in codecs
    assert np.array_equal(npy(zc.decode_batches(fr, None)).view(np.uint8), msg)


@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_FIXEDLEN])
def test_speculative_width_misses_vs_oracle(zc, port, pin, monkeypatch):
    """The single-read encoder packs each unit at its 64 KiB window's width and redoes units whose
    decision differs: an outlier past the window (wider FixedLen), one near the int32 limit (Auto:
    the gain check fails -> RAW; pinned: width 32), a hit, and a tiny last unit (window profile
    skipped).  Frames must equal the oracle's and the two-read path's."""
    scale = 2e-4
    U = (4 << 20) // 4
    rng = np.random.default_rng(pin + 5)
    x = (rng.normal(0, 1, 3 * U + 700) * 2e-3).astype(np.float32)    # |q| ~ tens
    x[U // 2] = 3.0                                                  # unit 0: outlier past the window
    x[U + U // 3] = np.float32(2e9 * scale)                          # unit 1: |q| near 2^31
    rc, sym = port.eb_quantize_f32(x, scale)
    assert rc == 0
    hint = abi.make_hint()
    fr = zc.encode_batches(t(x), pin, scale=scale, hint=hint)
    exp = port.encode_batches(sym.view(np.uint8), pin, hint, None)
    for b, (er, ef) in enumerate(exp):
        r = fr.encode_results()[b]
        assert (r.codec, r.payload_bytes, r.total_bytes) == (er.codec, er.payload_bytes, er.total_bytes), f"unit {b}"
        assert np.array_equal(npy(fr.frame(b)), ef), f"frame {b}"
    assert np.array_equal(npy(zc.decode_batches(fr, None)), sym)
    monkeypatch.setenv("ZC_NO_SPEC", "1")
    two = zc.encode_batches(t(x), pin, scale=scale, hint=hint)
    for b in range(fr.nbatches):
        assert np.array_equal(npy(fr.frame(b)), npy(two.frame(b)))


_RANGE_CASES = {
    # |q| past 2^32: the low word alone looks like a small symbol (858993.5 / 2e-4 = 4294967500)
    "wrap_small": [858993.5],
    "wrap_pos": [np.float32((2.0 ** 32 + 4096) * 2e-4)],
    "wrap_neg": [np.float32(-(2.0 ** 32 - 8192) * 2e-4)],
    "huge": [np.float32(2.0 ** 40 * 2e-4)],
    "just_over": [np.float32(2.0 ** 31 * 2e-4)],
    # inside the int32 range but past the fast path's 2^30: exact, no error
    "inside": [np.float32(2.0e9 * 2e-4), np.float32(-1.5e9 * 2e-4)],
}


@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_FIXEDLEN, abi.PIN_RAW])
@pytest.mark.parametrize("case", sorted(_RANGE_CASES))
def test_int32_range_past_window(zc, port, pin, case):
    """eb_quantize_chunk throws when |x/scale| >= 2147483647.5 (quant.cpp:22-27,
    test_quant.cpp:61-68) wherever the value sits: here past every unit's 64 KiB profile window,
    so the single-read encoder's width guess never saw it.  The fused encoder must raise exactly
    where the oracle does, and otherwise produce the oracle's frames."""
    scale = 2e-4
    U = (4 << 20) // 4
    rng = np.random.default_rng(11)
    x = rng.normal(0, 1, 2 * U + 1000).astype(np.float32)
    vals = _RANGE_CASES[case]
    for i, v in enumerate(vals):
        x[U // 2 + 7919 * i] = v            # unit 0, past the window
        x[U + U - 33 - i] = v               # unit 1, its last full tile
    rc, sym = port.eb_quantize_f32(x, scale)
    hint = abi.make_hint()
    if rc != 0:
        assert rc == 2  # bin index exceeds int32 range
        with pytest.raises(ValueError, match="int32"):
            zc.encode_batches(t(x), pin, scale=scale, hint=hint)
        with pytest.raises(ValueError, match="int32"):
            zc.eb_quantize_with_scale(t(x), scale)
        return
    fr = zc.encode_batches(t(x), pin, scale=scale, hint=hint)
    exp = port.encode_batches(sym.view(np.uint8), pin, hint, None)
    for b, (er, ef) in enumerate(exp):
        assert np.array_equal(npy(fr.frame(b)), ef), f"frame {b}"
    assert np.array_equal(npy(zc.decode_batches(fr, None)), sym)


def test_int32_range_host_roundtrip(zc, port):
    """The same rejection through the C-ABI host round trip (zc_codec_roundtrip_host_f32): the
    device error word carries ZC_DERR_RANGE."""
    L = zc.lib()
    count = 3 * ((4 << 20) // 4) + 5
    x = np.random.default_rng(3).normal(0, 1, count).astype(np.float32)
    x[(4 << 20) // 4 + 300000] = 858993.5
    assert port.eb_quantize_f32(x, 2e-4)[0] == 2
    hx = torch.from_numpy(x).pin_memory()
    hy = torch.empty(count, dtype=torch.float32).pin_memory()
    work = torch.empty(count, dtype=torch.float32, device=DEV)
    fr = zc.alloc_frames(count * 4, DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    hint, cfg = abi.make_hint(), zc.default_arb_config()
    s = torch.cuda.current_stream()
    for pin in (abi.PIN_AUTO, abi.PIN_FIXEDLEN):
        err.zero_()
        zc.check(L.zc_codec_roundtrip_host_f32(hx.data_ptr(), count, 2e-4, zc._ptr(work), zc._ptr(fr.stages),
                                               zc.STAGE_STRIDE, abi.STAGE_BANK_BYTES, pin, C.byref(hint), None,
                                               C.byref(cfg), zc._ptr(fr.results), zc._ptr(fr.index), zc._ptr(err),
                                               hy.data_ptr(), 2, C.c_void_p(s.cuda_stream)))
        torch.cuda.synchronize()
        assert int(err.item()) & abi.DERR_RANGE


@pytest.mark.parametrize("stage_len", [(2 << 20) + 32, (3 << 20) + 100, (4 << 20)])
@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_FIXEDLEN])
def test_small_stage_capacity_vs_oracle(zc, port, pin, stage_len):
    """A caller stage smaller than a unit's raw bytes: the payload cap (stage_len - 32) decides
    FixedLen vs RAW vs failure as in encode_best / send_batch; no store may pass the stage.
    Stages sit at a stride with a guard pattern after each, which must survive."""
    scale = 2e-4
    U = (4 << 20) // 4
    rng = np.random.default_rng(pin + stage_len % 97)
    x = rng.normal(0, 1, 3 * U).astype(np.float32)
    x[U:2 * U] *= 4.0                                         # unit 1: width 18 -> 2.25 MiB
    x[2 * U:] *= 0.01                                         # unit 2: width 9
    rc, sym = port.eb_quantize_f32(x, scale)
    assert rc == 0
    hint = abi.make_hint()
    exp = port.encode_batches(sym.view(np.uint8), pin, hint, None, stage_len=stage_len)
    stride = zc.STAGE_STRIDE
    stages = torch.full((3 * stride,), 0xA5, dtype=torch.uint8, device=DEV)
    results = torch.zeros(3 * 3, dtype=torch.int64, device=DEV)
    index = torch.zeros(3 * abi.HUFF_INDEX_ENTRIES, dtype=torch.int32, device=DEV)
    err = torch.zeros(1, dtype=torch.int32, device=DEV)
    L = zc.lib()
    zc.check(L.zc_encode_batches_f32(zc._ptr(t(x)), x.size, scale, zc._ptr(stages), stride, stage_len, pin,
                                     C.byref(hint), None, C.byref(zc.default_arb_config()), zc._ptr(results),
                                     zc._ptr(index), zc._ptr(err), zc._stream()))
    torch.cuda.synchronize()
    st = npy(stages)
    res = npy(results).reshape(3, 3)
    failed = any(er.total_bytes == 0 for er, _ in exp)
    assert bool(int(err.item()) & abi.DERR_CAPACITY) == failed
    for b, (er, ef) in enumerate(exp):
        assert (res[b, 0] & 0xffffffff, res[b, 1], res[b, 2]) == (er.codec, er.payload_bytes, er.total_bytes), f"unit {b}"
        if er.total_bytes:
            assert np.array_equal(st[b * stride: b * stride + er.total_bytes], ef), f"frame {b}"
        assert np.all(st[b * stride + stage_len:(b + 1) * stride] == 0xA5), f"stage {b} overrun"


@pytest.mark.parametrize("embed", [False, True])
def test_indexless_4mib_reference_frame_parallel_decode(zc, port, embed):
    """A 4 MiB Huffman frame produced by the CPU reference path (no companion index, huffman.cpp:
    216-246) decodes on the device through recv_batch's dispatch: the CTA-parallel
    self-synchronising decoder, bit-exact, in milliseconds (the sequential decoder is the fallback)."""
    import time
    rng = np.random.default_rng(44 + embed)
    sym = np.clip(rng.laplace(0, 40, (4 << 20) // 4), -3000, 3000).astype(np.int32)
    raw = sym.view(np.uint8)
    o = port.huff_from_bytes(raw[: 1 << 20])
    c = zc.HuffmanContext.from_bytes(raw[: 1 << 20])
    cfg = abi.default_arb_config()
    cfg.embed_codebook = 1 if embed else 0
    r, frame = port.send_batch(raw, abi.PIN_HUFFMAN, abi.make_hint(), None if embed else o, cfg)
    assert r.codec == abi.CODEC_HUFFMAN
    h = zc.parse_header(bytes(frame[:32]))
    payload = t(frame[32:32 + h.payload_bytes].copy())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ok, back = zc.huffman_decode(h, payload, None if embed else c, len(raw))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    assert ok and np.array_equal(npy(back), raw)
    assert dt < 1.0, f"index-less 4 MiB decode took {dt:.2f} s"
    # the same frame through the batched receive path with an fp32 sink (dequantize_into)
    fr = zc.alloc_frames(len(raw), DEV)
    fr.stages[: len(frame)] = t(frame)
    er = abi.EncodeResult()
    er.codec, er.payload_bytes, er.total_bytes = abi.CODEC_HUFFMAN, h.payload_bytes, len(frame)
    fr.results[: C.sizeof(er)] = t(np.frombuffer(bytes(er), np.uint8).copy())
    y = zc.decode_batches(fr, None if embed else c, scale=2e-4, use_index=False)
    exp = np.zeros(len(sym), np.float32)
    port.lib.zo_dequantize_f32(sym, len(sym), 0, 2e-4, 0, exp)
    assert np.array_equal(npy(y), exp)


# ------------------------------------------------------------------ warp-staged short-code decoder
def _kraft_lengths(maxlen):
    """A complete prefix code with lengths 1..maxlen plus a second maxlen code (Kraft sum = 1)."""
    lens = [0] * 256
    for s in range(maxlen):
        lens[s] = s + 1
    lens[maxlen] = maxlen
    return lens


@pytest.mark.parametrize("maxlen", [11, 12, 13])
@pytest.mark.parametrize("n", [32 * 1024, 70000, 300001])
def test_huffman_warp_decoder_edges(zc, port, maxlen, n):
    """Codes at / past the root LUT (12 bits: warp-staged vs per-lane decoder), warps with idle lanes
    (grain counts not a multiple of 32), a partial last grain, a corrupted companion index (the
    sequential fixup must reproduce the data) and a truncated payload (failure)."""
    lens = _kraft_lengths(maxlen)
    c = zc.HuffmanContext.from_lengths(lens)
    from oracle import HuffStruct
    o = HuffStruct()
    assert port.lib.zo_huff_from_lengths(np.array(lens, np.uint8), C.byref(o)) == 1
    rng = np.random.default_rng(maxlen * 1000 + n)
    p = np.array([2.0 ** -min(l, 8) for l in lens[: maxlen + 1]])
    raw = rng.choice(maxlen + 1, size=n, p=p / p.sum()).astype(np.uint8)
    cap = 4 * n + 64
    got, idx = zc.huffman_encode(t(raw), c, cap, with_index=True)
    assert got.numel() > 0
    if o is not None:
        out = np.zeros(cap, np.uint8)
        pn = port.lib.zo_huffman_encode(raw, n, C.byref(o), out, cap, 0)
        assert got.numel() == pn and np.array_equal(npy(got), out[:pn])
    h = hdr(2, n, got.numel(), 0)
    ok, back = zc.huffman_decode(h, got, c, n, index=idx)
    assert ok and np.array_equal(npy(back), raw)
    bad = idx.clone()
    bad[len(bad) // 2] += 3  # a start bit that is not a code boundary
    ok, back = zc.huffman_decode(h, got, c, n, index=bad)
    assert ok and np.array_equal(npy(back), raw)
    h2 = hdr(2, n, got.numel() - 8, 0)
    ok, _ = zc.huffman_decode(h2, got[:-8], c, n, index=idx)
    assert not ok
