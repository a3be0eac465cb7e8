"""GPU parity of the QSGD path (quant.cpp:64-98, collectives.cpp:518-523):
std::mt19937_64 draws generated on the device by jump-ahead are the reference's, bit for bit; QSGD
symbols equal the compiled reference's for every chunking of the stream; allreduce_qsgd equals the
reference's N-rank result bit for bit (f64 output)."""
import numpy as np
import pytest
import torch

from paper_2605_12396_b200 import abi

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


@pytest.fixture(scope="module")
def ref():
    import oracle
    try:
        return oracle.ref()
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"compiled reference unavailable: {e}")


@pytest.mark.parametrize("seed,skip,n", [(5489, 0, 1000), (1, 0, 312), (7, 311, 5), (123456789, 1 << 20, 70000),
                                         (2**64 - 1, 12345, 3 << 16)])
def test_mt19937_64_stream(zc, ref, seed, skip, n):
    got = zc.mt19937_64(seed, n, skip).cpu().numpy().view(np.uint64)
    assert np.array_equal(got, ref.mt19937_64(seed, skip, n))


def test_mt19937_64_known_answer(zc):
    # C++ [rand.predef]: the 10000th draw of a default-constructed mt19937_64
    assert int(zc.mt19937_64(5489, 1, 9999).cpu().numpy().view(np.uint64)[0]) == 9981545732273789042


@pytest.mark.parametrize("n,levels,seed", [(0, 4, 1), (1, 1, 2), (4097, 15, 3), (300001, 255, 99),
                                           ((1 << 20) + 3, 1 << 30, 2**40 + 5)])
def test_qsgd_quantize_vs_reference(zc, ref, n, levels, seed):
    rng = np.random.default_rng(n + levels)
    x = (rng.standard_normal(n) * 0.1).astype(np.float32)
    if n > 2:
        x[1] = 0.0
        x[2] = -0.0
    sym, scale = zc.qsgd_quantize(torch.from_numpy(x).cuda(), levels, seed)
    rc, exp, escale = ref.qsgd_quantize(x.astype(np.float64), levels, seed)
    assert rc == 0
    assert scale == escale
    assert np.array_equal(sym.cpu().numpy(), exp)


def test_qsgd_chunk_with_skip_and_zero_norm(zc, ref):
    x = np.random.default_rng(5).standard_normal(50000).astype(np.float32)
    got = zc.qsgd_quantize_chunk(torch.from_numpy(x).cuda(), 7, 3.25, 42, skip=777).cpu().numpy()
    rc, exp = ref.qsgd_quantize_chunk(x.astype(np.float64), 7, 3.25, 42, 777)
    assert rc == 0 and np.array_equal(got, exp)
    z = np.zeros(1000, np.float32)
    sym, scale = zc.qsgd_quantize(torch.from_numpy(z).cuda(), 4, 3)
    assert scale == 1.0 and not sym.any()


def test_qsgd_errors(zc):
    x = torch.ones(10, device="cuda")
    with pytest.raises(ValueError):
        zc.qsgd_quantize(x, 0, 1)
    with pytest.raises(ValueError):
        zc.qsgd_quantize_chunk(x, 4, float("nan"), 1)
    x[3] = float("inf")
    with pytest.raises(ValueError):
        zc.qsgd_quantize(x, 4, 1)


@pytest.mark.parametrize("n", [2, 3])
def test_allreduce_qsgd_vs_reference(zc, ref, n):
    count = 200003
    rng = np.random.default_rng(n)
    xs = [(rng.standard_normal(count) * (r + 1)).astype(np.float32) for r in range(n)]
    seeds = [11 + r for r in range(n)]
    g = zc.Group(n)
    outs = g.allreduce_qsgd([torch.from_numpy(x).cuda() for x in xs], 16, seeds)
    rc, exp = ref.allreduce_qsgd([x.astype(np.float64) for x in xs], 16, seeds)
    assert rc == 0
    for r in range(n):
        assert np.array_equal(outs[r].cpu().numpy().view(np.uint64), exp[r].view(np.uint64))
    g.close()
