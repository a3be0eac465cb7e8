"""GPU parity of the ring collectives (collectives.cpp:398-616) on one B200: N ranks in one process
share the GPU (a loopback Group — the analogue of the reference's thread-per-rank Communicator),
exercising the same fused RS-step / AG-relay kernels and flag protocol as the NVLink path.

Bar: symbols bit-identical to the serial oracle for every codec pin; WireStats equal to the
oracle ring's (frames per codec, raw/payload/total bytes)."""
import numpy as np
import pytest
import torch

from paper_2605_12396_b200 import abi

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]
DEV = "cuda"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def npy(x):
    return x.cpu().numpy()


def test_allreduce_hand_vector(zc):
    g = zc.Group(4)
    syms = [t(np.array([r + 1, -(r + 1), 100], np.int32)) for r in range(4)]
    g.allreduce(syms, [1.0] * 4)
    for s in syms:
        assert npy(s).tolist() == [10, -10, 400]  # test_collectives.cpp:83-94


def test_scale_reconciliation(zc):
    g = zc.Group(2)
    syms = [t(np.array([10, -6, 3, 7], np.int32)), t(np.array([1, 2, 3, 4], np.int32))]
    scales = g.allreduce(syms, [0.5, 1.0])
    assert scales == [1.0, 1.0]
    for s in syms:
        assert npy(s).tolist() == [6, -1, 5, 8]  # test_collectives.cpp:103-118


def test_overflow_aborts_and_group_survives(zc):
    g = zc.Group(2)
    syms = [t(np.full(8, 2**31 - 1, np.int32)) for _ in range(2)]
    with pytest.raises(OverflowError):
        g.allreduce(syms, [1.0, 1.0])
    syms = [t(np.array([1, 2], np.int32)) for _ in range(2)]
    g.allreduce(syms, [1.0, 1.0])
    assert [npy(s).tolist() for s in syms] == [[2, 4], [2, 4]]  # test_collectives.cpp:129-146


def test_allreduce_max(zc):
    g = zc.Group(3)
    assert g.allreduce_max([1.5 * r - 1.0 for r in range(3)]) == [2.0] * 3
    with pytest.raises(ValueError):
        g.allreduce_max([1.0, float("nan"), 0.0])


def _serial_eb(port, xs, rel):
    gmax = max(float(np.abs(x.astype(np.float64)).max()) for x in xs)
    scale = 1.0 if gmax == 0.0 else 2.0 * rel * gmax
    acc = np.zeros(len(xs[0]), np.int64)
    syms = []
    for x in xs:
        rc, s = port.eb_quantize_f32(x, scale)
        assert rc == 0
        syms.append(s)
        acc += s
    out = np.zeros(len(acc))
    port.lib.zo_dequantize_f64(acc.astype(np.int32), len(acc), 0, scale, 0, out)
    return scale, syms, out


@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("pin", [abi.PIN_RAW, abi.PIN_FIXEDLEN, abi.PIN_HUFFMAN, abi.PIN_AUTO])
def test_allreduce_eb_bit_identical_across_pins(zc, port, n, pin):
    """test_collectives.cpp:148-174 / acceptance C3: every pin == the serial oracle, bit for bit."""
    rel = 1e-3
    count = 5000
    rng = np.random.default_rng(1000 + n)
    xs = [rng.normal(0, 1.0 + r, count).astype(np.float32) for r in range(n)]
    scale, syms, exp = _serial_eb(port, xs, rel)
    g = zc.Group(n, cfg=zc.collective_config(pin))
    g.set_shared_huffman_from_bytes(syms[0].view(np.uint8))
    outs = g.allreduce_eb([t(x) for x in xs], rel, torch.float64)
    for o in outs:
        assert np.array_equal(npy(o).view(np.uint64), exp.view(np.uint64))


@pytest.mark.parametrize("n,count", [(2, (12 << 20) // 4 + 5), (4, (9 << 20) // 4), (3, 3 << 20)])
@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_FIXEDLEN, abi.PIN_HUFFMAN])
def test_allreduce_sym_multibatch_vs_oracle_ring(zc, port, n, count, pin):
    """Multi-batch chunks: reduced symbols exact; wire stats equal to the oracle ring's."""
    rng = np.random.default_rng(n * 7 + pin)
    syms = [np.clip(rng.laplace(0, 50 * (r + 1), count), -2**20, 2**20).astype(np.int32) for r in range(n)]
    sample = syms[0].view(np.uint8)[: 4 << 20]
    o = port.huff_from_bytes(sample)
    cfgp = abi.default_collective_config(pin)
    rc, exp, _, wire = port.ring_allreduce(np.stack(syms), [1.0] * n, pin, cfgp.hint, o, cfgp.arb,
                                           cfgp.fused_codec_min_msg_bytes)
    assert rc == 0
    assert np.array_equal(exp[0], np.sum(np.stack(syms).astype(np.int64), axis=0).astype(np.int32))
    g = zc.Group(n, cfg=zc.collective_config(pin))
    g.set_shared_huffman(zc.HuffmanContext.from_bytes(sample))
    ts = [t(s) for s in syms]
    g.allreduce(ts, [1.0] * n)
    for r in range(n):
        assert np.array_equal(npy(ts[r]), exp[r])
    w = g.wire_stats()
    assert list(w.frames_by_codec) == list(wire.frames_by_codec)
    assert (w.raw_bytes, w.payload_bytes, w.total_bytes) == (wire.raw_bytes, wire.payload_bytes, wire.total_bytes)


@pytest.mark.parametrize("n", [2, 4])
def test_reduce_scatter_ownership(zc, n):
    count = 10001
    rng = np.random.default_rng(n)
    syms = [rng.integers(-1000, 1000, count).astype(np.int32) for _ in range(n)]
    total = np.sum(np.stack(syms).astype(np.int64), axis=0).astype(np.int32)
    g = zc.Group(n)
    ts = [t(s) for s in syms]
    g.reduce_scatter(ts)
    for r in range(n):
        c = (r + 1) % n  # rank r owns chunk (r+1) mod n, bounds c*count/n (collectives.cpp:465-467)
        lo, hi = c * count // n, (c + 1) * count // n
        assert np.array_equal(npy(ts[r])[lo:hi], total[lo:hi])


@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_HUFFMAN])
def test_allgather_vs_oracle(zc, port, n, pin):
    block = (5 << 20) // 4 + 7
    rng = np.random.default_rng(n + 100)
    blocks = [(rng.integers(-300, 300, block)).astype(np.int32) for _ in range(n)]
    sample = blocks[0].view(np.uint8)[: 1 << 20]
    g = zc.Group(n, cfg=zc.collective_config(pin))
    g.set_shared_huffman(zc.HuffmanContext.from_bytes(sample))
    outs = g.allgather([t(b) for b in blocks])
    full = np.concatenate(blocks)
    for o in outs:
        assert np.array_equal(npy(o), full)
    o = port.huff_from_bytes(sample)
    cfgp = abi.default_collective_config(pin)
    res = np.zeros(n * n * block, np.int32)
    w = abi.WireStats()
    import ctypes as C
    assert port.lib.zo_ring_allgather(n, np.stack(blocks).ravel(), block, pin, C.byref(cfgp.hint), C.byref(o),
                                      C.byref(cfgp.arb), res, C.byref(w)) == 0
    gw = g.wire_stats()
    assert list(gw.frames_by_codec) == list(w.frames_by_codec) and gw.payload_bytes == w.payload_bytes


def test_c2_laplacian_two_ranks_large(zc, port):
    """BASELINE config 2 shape at a test-sized count: Laplacian gradients, abs eb 1e-4, 2 ranks."""
    n, count = 2, 16 << 20
    rng = np.random.default_rng(100)
    xs = [rng.laplace(0, 1e-2, count).astype(np.float32) for _ in range(n)]
    gmax = max(float(np.abs(x).max()) for x in xs)
    rel = 1e-4 / gmax  # abs eb 1e-4 -> scale 2e-4
    scale, syms, exp = _serial_eb(port, xs, rel)
    g = zc.Group(n)
    outs = g.allreduce_eb([t(x) for x in xs], rel, torch.float64)
    for o in outs:
        assert np.array_equal(npy(o).view(np.uint64), exp.view(np.uint64))
    exact = xs[0].astype(np.float64) + xs[1].astype(np.float64)
    assert np.max(np.abs(npy(outs[0]) - exact)) <= n * scale / 2 * (1 + 1e-9)
    w = g.wire_stats()
    assert w.frames_by_codec[abi.CODEC_FIXEDLEN] > 0


def _ring_check(zc, port, g, syms, pin, ctx_np=None, cfg=None):
    """g.allreduce on `syms` == the oracle ring (symbols and WireStats)."""
    n = len(syms)
    cfgp = cfg or abi.default_collective_config(pin)
    rc, exp, _, wire = port.ring_allreduce(np.stack(syms), [1.0] * n, pin, cfgp.hint, ctx_np, cfgp.arb,
                                           cfgp.fused_codec_min_msg_bytes)
    assert rc == 0
    ts = [t(s) for s in syms]
    g.allreduce(ts, [1.0] * n)
    for r in range(n):
        assert np.array_equal(npy(ts[r]), exp[r]), f"rank {r}"
    w = g.wire_stats()
    assert list(w.frames_by_codec) == list(wire.frames_by_codec)
    assert (w.raw_bytes, w.payload_bytes, w.total_bytes) == (wire.raw_bytes, wire.payload_bytes, wire.total_bytes)
    return w


@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_FIXEDLEN, abi.PIN_HUFFMAN])
def test_allreduce_n8_multipiece_vs_oracle_ring(zc, port, pin, monkeypatch):
    """8 ranks, chunks of two 4 MiB batches (one full, one ragged) moved one batch per piece
    (ZC_COMM_REGION_UNITS=1), so every step runs several pieces and the 3 piece regions are
    reused many times over the 7 RS + 7 AG steps.  Count not a multiple of 8."""
    monkeypatch.setenv("ZC_COMM_REGION_UNITS", "1")
    n = 8
    count = n * ((5 << 20) // 4) + 13
    rng = np.random.default_rng(80 + pin)
    syms = [np.clip(rng.laplace(0, 40 * (r + 1), count), -2**19, 2**19).astype(np.int32) for r in range(n)]
    sample = syms[0].view(np.uint8)[: 4 << 20]
    g = zc.Group(n, cfg=zc.collective_config(pin))
    g.set_shared_huffman(zc.HuffmanContext.from_bytes(sample))
    _ring_check(zc, port, g, syms, pin, port.huff_from_bytes(sample))
    g.close()


def _smooth_field(nz, rank, n=512):
    """C3's synthetic scientific field: sin(2 pi i/512) cos(4 pi j/512) +
    0.5 sin(6 pi k/512) with a per-rank phase, on a 512 x 512 x nz slab, fp32."""
    i = np.arange(n, dtype=np.float64)[:, None, None]
    j = np.arange(n, dtype=np.float64)[None, :, None]
    k = np.arange(nz, dtype=np.float64)[None, None, :]
    ph = 0.37 * rank
    f = np.sin(2 * np.pi * i / n + ph) * np.cos(4 * np.pi * j / n) + 0.5 * np.sin(6 * np.pi * k / n + ph)
    return f.astype(np.float32).ravel()


@pytest.mark.parametrize("n", [4, 8])
def test_allreduce_eb_c3_smooth_field(zc, port, n):
    """BASELINE config 3 at a slab size: the 512^3 smooth field's generator on 512 x 512 x 24
    (6 Mi elements per rank), relative bound 1e-3 through allreduce_eb (scale = 2 rel gmax,
    collectives.cpp:505-513).  Output bit-identical to the serial oracle; error <= N eb."""
    rel = 1e-3
    xs = [_smooth_field(24, r) for r in range(n)]
    scale, syms, exp = _serial_eb(port, xs, rel)
    g = zc.Group(n)
    outs = g.allreduce_eb([t(x) for x in xs], rel, torch.float64)
    for o in outs:
        assert np.array_equal(npy(o).view(np.uint64), exp.view(np.uint64))
    exact = np.sum(np.stack([x.astype(np.float64) for x in xs]), axis=0)
    assert np.max(np.abs(npy(outs[0]) - exact)) <= n * scale / 2 * (1 + 1e-9)
    g.close()
    # the same symbols through the ring: wire stats equal the oracle ring's (FixedLen frames)
    g = zc.Group(n)
    w = _ring_check(zc, port, g, syms, abi.PIN_AUTO)
    assert w.frames_by_codec[abi.CODEC_FIXEDLEN] > 0
    g.close()


@pytest.mark.parametrize("n,count", [
    (2, (1 << 20) // 4),            # 1 MiB: RS steps ship RAW below fusedCodecMinMsgBytes
    (2, (4 << 20) // 4 + 3),        # just past one batch
    (2, (64 << 20) // 4),
    (8, (1 << 20) // 4 + 5),        # count % 8 != 0, tiny chunks
    (8, (40 << 20) // 4 + 7),
])
def test_allreduce_c5_sizes_vs_oracle_ring(zc, port, n, count):
    """C5's message-size sweep points against the oracle ring (auto selector, shared context)."""
    rng = np.random.default_rng(count % 1000 + n)
    syms = [np.clip(rng.laplace(0, 30, count), -2**18, 2**18).astype(np.int32) for _ in range(n)]
    sample = syms[0].view(np.uint8)[: 4 << 20]
    g = zc.Group(n)
    g.set_shared_huffman(zc.HuffmanContext.from_bytes(sample))
    _ring_check(zc, port, g, syms, abi.PIN_AUTO, port.huff_from_bytes(sample))
    g.close()


@pytest.mark.slow
def test_allreduce_eb_1gib_two_ranks(zc, port):
    """C5's top end: 1 GiB of fp32 per rank (256 Mi elements), abs eb 1e-4, 2 ranks; exact
    against the symbol sum (int64, checked to fit int32) dequantized as the reference does."""
    n, count = 2, 1 << 28
    rng = np.random.default_rng(5)
    xs = [rng.laplace(0, 1e-2, count).astype(np.float32) for _ in range(n)]
    scale = 2e-4
    gmax = max(float(np.abs(x).max()) for x in xs)
    rel = scale / (2 * gmax)
    acc = np.zeros(count, np.int64)
    for x in xs:
        rc, s = port.eb_quantize_f32(x, 2.0 * rel * gmax)
        assert rc == 0
        acc += s
    g = zc.Group(n)
    outs = g.allreduce_eb([t(x) for x in xs], rel, torch.float32)
    sc = 2.0 * rel * gmax
    exp = (sc * acc.astype(np.int32).astype(np.float64)).astype(np.float32)
    for o in outs:
        assert np.array_equal(npy(o), exp)
    g.close()


def test_embedded_codebook_ring_without_shared_ctx(zc, port):
    """cfg.embedCodebook with no shared table: Auto picks Huffman with a per-frame codebook
    (rea.cpp:160, 214-221).  Every rank must decode those frames (RS adds, AG stores)."""
    n = 3
    count = 3 * ((6 << 20) // 4) + 11
    rng = np.random.default_rng(17)
    syms = []
    for r in range(n):
        s = rng.integers(-2, 3, count).astype(np.int32)
        hit = rng.random(count) < 1e-3
        s[hit] = rng.integers(-(1 << 19), 1 << 19, int(hit.sum()))
        syms.append(s)
    cfg = zc.collective_config(abi.PIN_AUTO)
    cfg.arb.embed_codebook = 1
    g = zc.Group(n, cfg=cfg)
    w = _ring_check(zc, port, g, syms, abi.PIN_AUTO, None, cfg)
    assert w.frames_by_codec[abi.CODEC_HUFFMAN] > 0
    g.close()


# ------------------------------------------------------------------ per-slot framing
@pytest.mark.parametrize("n,count", [(2, (3 << 20) // 4 + 777), (3, (5 << 20) // 4 + 3)])
@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_RAW, abi.PIN_FIXEDLEN, abi.PIN_HUFFMAN])
def test_allreduce_per_slot_framing_vs_reference(zc, port, ref, n, count, pin):
    """CollectiveConfig::perSlotFraming (collectives.hpp:33): every exchange batches at 512 KiB
    (RankCtx::chunk_raw_bytes, collectives.cpp:197-199).  Symbols and WireStats equal to the
    compiled reference Communicator's and to the oracle ring's; more frames than 4 MiB batching."""
    import ctypes as C
    rng = np.random.default_rng(40 + n * 5 + pin)
    syms = [np.clip(rng.laplace(0, 40 * (r + 1), count), -2**20, 2**20).astype(np.int32) for r in range(n)]
    sample = np.ascontiguousarray(syms[0].view(np.uint8)[: 1 << 20])
    cfg = zc.collective_config(pin, per_slot_framing=1)
    exp = np.stack(syms).copy()
    sc = np.ones(n)
    w_ref = abi.WireStats()
    assert ref.lib.zr_allreduce_sym(n, C.byref(cfg), exp.ravel(), count, abi.QUANT_ERROR_BOUNDED, sc, 0,
                                    sample.ctypes.data_as(C.POINTER(C.c_uint8)), len(sample), C.byref(w_ref),
                                    None) == 0
    o = port.huff_from_bytes(sample)
    rc, exp_p, _, w_p = port.ring_allreduce(np.stack(syms), [1.0] * n, pin, cfg.hint, o, cfg.arb,
                                            cfg.fused_codec_min_msg_bytes, per_slot=True)
    assert rc == 0 and np.array_equal(exp_p, exp)
    assert list(w_p.frames_by_codec) == list(w_ref.frames_by_codec) and w_p.payload_bytes == w_ref.payload_bytes
    g = zc.Group(n, cfg=cfg)
    g.set_shared_huffman(zc.HuffmanContext.from_bytes(sample))
    ts = [t(s) for s in syms]
    g.allreduce(ts, [1.0] * n)
    for r in range(n):
        assert np.array_equal(npy(ts[r]), exp[r])
    w = g.wire_stats()
    assert list(w.frames_by_codec) == list(w_ref.frames_by_codec)
    assert (w.raw_bytes, w.payload_bytes, w.total_bytes) == (w_ref.raw_bytes, w_ref.payload_bytes, w_ref.total_bytes)
    g4 = zc.Group(n, cfg=zc.collective_config(pin))  # 4 MiB batches: fewer frames on the same data
    g4.set_shared_huffman(zc.HuffmanContext.from_bytes(sample))
    g4.allreduce([t(s) for s in syms], [1.0] * n)
    assert sum(g4.wire_stats().frames_by_codec) < sum(w.frames_by_codec)


@pytest.mark.parametrize("n", [2, 4])
def test_allgather_and_broadcast_per_slot_framing(zc, port, ref, n):
    """allgather under per-slot framing: outputs exact, WireStats equal to the compiled reference's
    (collectives.cpp:525-544); broadcast's store-and-forward at slot granularity (:569-591) exact."""
    import ctypes as C
    block = (3 << 20) // 4 + 11
    rng = np.random.default_rng(n + 900)
    blocks = [rng.integers(-3000, 3000, block).astype(np.int32) for _ in range(n)]
    cfg = zc.collective_config(abi.PIN_AUTO, per_slot_framing=1)
    out = np.zeros(n * n * block, np.int32)
    w_ref = abi.WireStats()
    assert ref.lib.zr_allgather_sym(n, C.byref(cfg), np.stack(blocks).ravel(), block, None, 0, out,
                                    C.byref(w_ref)) == 0
    g = zc.Group(n, cfg=cfg)
    outs = g.allgather([t(b) for b in blocks])
    full = np.concatenate(blocks)
    for o in outs:
        assert np.array_equal(npy(o), full)
    w = g.wire_stats()
    assert list(w.frames_by_codec) == list(w_ref.frames_by_codec)
    assert (w.raw_bytes, w.payload_bytes, w.total_bytes) == (w_ref.raw_bytes, w_ref.payload_bytes, w_ref.total_bytes)
    data = rng.integers(-2**20, 2**20, (5 << 20) // 4 + 9).astype(np.int32)
    ds = [t(data) if r == 1 else torch.zeros(len(data), dtype=torch.int32, device=DEV) for r in range(n)]
    g.broadcast(ds, 1)
    for d in ds:
        assert np.array_equal(npy(d), data)


@pytest.mark.parametrize("n", [2, 3, 5])
@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_FIXEDLEN, abi.PIN_HUFFMAN])
def test_fused_ring_equals_unfused(zc, port, n, pin, monkeypatch):
    """The fused ring (fp32 quantized inside the first RS send and the RS sinks, sums' range handed
    to the next send, AG frames forwarded verbatim, dequantized inside the AG sinks) produces the
    same outputs and WireStats as the unfused ring (quantize -> re-encoding hops -> dequantize),
    and both equal the serial oracle."""
    count = (11 << 20) // 4 + 5 * n + 1
    rng = np.random.default_rng(70 + n + pin)
    xs = [rng.laplace(0, 1e-2 * (r + 1), count).astype(np.float32) for r in range(n)]
    gmax = max(float(np.abs(x).max()) for x in xs)
    rel = 1e-4 / gmax
    scale, syms, exp = _serial_eb(port, xs, rel)
    outs, wires = [], []
    for unfused in (False, True):
        if unfused:
            monkeypatch.setenv("ZC_RING_UNFUSED", "1")
        g = zc.Group(n, cfg=zc.collective_config(pin))
        g.set_shared_huffman_from_bytes(syms[0].view(np.uint8)[: 1 << 20])
        o = g.allreduce_eb([t(x) for x in xs], rel, torch.float64)
        outs.append([npy(v) for v in o])
        wires.append(g.wire_stats())
    for o in outs[0] + outs[1]:
        assert np.array_equal(o.view(np.uint64), exp.view(np.uint64))
    a, b = wires
    assert list(a.frames_by_codec) == list(b.frames_by_codec)
    assert (a.raw_bytes, a.payload_bytes, a.total_bytes) == (b.raw_bytes, b.payload_bytes, b.total_bytes)


@pytest.mark.parametrize("n", [2, 3, 5])
@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_FIXEDLEN, abi.PIN_RAW])
@pytest.mark.parametrize("fusedk", [True, False])
def test_fused_ring_kernel_vs_oracle(zc, port, n, pin, fusedk, monkeypatch):
    """The fused ring (default; ZC_RING_NOFUSEDK=1 opts out): every reduce-scatter receive is one
    kernel with the next step's send (decode -> reduce -> range -> decide -> pack into the
    successor), the steps and the first
    all-gather hop run as one wavefront over n + 2 piece regions.  Symbols, allreduce_eb outputs and
    WireStats equal the oracle ring; several pieces per chunk (ZC_COMM_REGION_UNITS=1)."""
    monkeypatch.setenv("ZC_COMM_REGION_UNITS", "1")
    if not fusedk:
        monkeypatch.setenv("ZC_RING_NOFUSEDK", "1")
    count = n * ((9 << 20) // 4) + 4 * n  # chunk bases 16-byte aligned (the fused kernel's precondition)
    rng = np.random.default_rng(500 + n + pin)
    syms = [np.clip(rng.laplace(0, 30 * (r + 1), count), -2**20, 2**20).astype(np.int32) for r in range(n)]
    g = zc.Group(n, cfg=zc.collective_config(pin))
    _ring_check(zc, port, g, syms, pin)
    xs = [rng.laplace(0, 1e-2, count).astype(np.float32) for _ in range(n)]
    rel = 1e-4 / max(float(np.abs(x).max()) for x in xs)
    scale, _, exp = _serial_eb(port, xs, rel)
    g2 = zc.Group(n, cfg=zc.collective_config(pin))
    for o in g2.allreduce_eb([t(x) for x in xs], rel, torch.float64):
        assert np.array_equal(npy(o).view(np.uint64), exp.view(np.uint64))
