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
