"""GPU checks of captured group collectives: a single-process group call is captured as a CUDA
graph on its first call and replayed on later calls with the same arguments (zc_comm.cu,
run_group).  A replay must equal a fresh eager run: the same symbols as the oracle ring on NEW data
in the same buffers, WireStats accumulating exactly one call's worth per replay, and the flag
protocol staying consistent with per-rank (eager) collectives and failures in between."""
import numpy as np
import pytest
import torch

from paper_2605_12396_b200 import abi

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]
DEV = "cuda"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("n,count", [(2, (9 << 20) // 4 + 5), (3, (5 << 20) // 4 + 1)])
@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_FIXEDLEN, abi.PIN_HUFFMAN, abi.PIN_RAW])
def test_replay_on_new_data_vs_oracle_ring(zc, port, n, count, pin):
    rng = np.random.default_rng(40 + n + 7 * pin)
    sample = np.clip(rng.laplace(0, 40, 1 << 20), -2**20, 2**20).astype(np.int32).view(np.uint8)
    cfgp = abi.default_collective_config(pin)
    o = port.huff_from_bytes(sample)
    g = zc.Group(n, cfg=zc.collective_config(pin))
    g.set_shared_huffman(zc.HuffmanContext.from_bytes(sample))
    ts = [torch.empty(count, dtype=torch.int32, device=DEV) for _ in range(n)]
    frames, raw, pay, tot = np.zeros(3, np.int64), 0, 0, 0
    for call in range(3):
        syms = [np.clip(rng.laplace(0, 30 * (r + 1 + call), count), -2**20, 2**20).astype(np.int32) for r in range(n)]
        for x, s in zip(ts, syms):
            x.copy_(t(s))
        rc, exp, _, wire = port.ring_allreduce(np.stack(syms), [1.0] * n, pin, cfgp.hint, o, cfgp.arb,
                                               cfgp.fused_codec_min_msg_bytes)
        assert rc == 0
        g.allreduce(ts, [1.0] * n)
        for r in range(n):
            assert np.array_equal(ts[r].cpu().numpy(), exp[r]), (call, r)
        frames += np.array(list(wire.frames_by_codec))
        raw, pay, tot = raw + wire.raw_bytes, pay + wire.payload_bytes, tot + wire.total_bytes
        w = g.wire_stats()
        assert list(w.frames_by_codec) == frames.tolist()
        assert (w.raw_bytes, w.payload_bytes, w.total_bytes) == (raw, pay, tot)


def test_replay_interleaved_with_rank_threads_and_failures(zc):
    n, count = 2, (6 << 20) // 4 + 3
    rng = np.random.default_rng(9)
    g = zc.Group(n)
    xs = [t(rng.normal(0, 1 + r, count).astype(np.float32)) for r in range(n)]
    outs = [torch.empty(count, dtype=torch.float32, device=DEV) for _ in range(n)]
    g.allreduce_eb(xs, 1e-4, outs=outs)  # captured
    first = [o.clone() for o in outs]
    want = (xs[0].double() + xs[1].double())
    for _ in range(3):
        syms = [t(rng.integers(-1000, 1000, count).astype(np.int32)) for _ in range(n)]
        ref = (syms[0].cpu().numpy().astype(np.int64) + syms[1].cpu().numpy()).astype(np.int32)
        g.run(lambda ctx: ctx.allreduce(syms[ctx.rank()], 1.0))  # per-rank (eager) in between
        for s in syms:
            assert np.array_equal(s.cpu().numpy(), ref)
        g.allreduce_eb(xs, 1e-4, outs=outs)  # replayed
        for o, f in zip(outs, first):
            assert torch.equal(o, f)
        assert float((outs[0].double() - want).abs().max()) <= 2e-4 * float(max(x.abs().max() for x in xs))
    # a failing replay (overflow) poisons and resets; the next replay works
    big = [t(np.full(count, 2**31 - 1, np.int32)) for _ in range(n)]
    good = [t(np.arange(count, dtype=np.int32) % 1000) for _ in range(n)]
    g.allreduce(good, [1.0] * n)  # capture with these buffers
    for b, x in zip(big, good):
        x.copy_(b)
    with pytest.raises(OverflowError):
        g.allreduce(good, [1.0] * n)  # replay on overflowing data
    for x in good:
        x.copy_(t(np.arange(count, dtype=np.int32) % 1000))
    g.allreduce(good, [1.0] * n)
    for x in good:
        assert np.array_equal(x.cpu().numpy(), 2 * (np.arange(count, dtype=np.int32) % 1000))


@pytest.mark.parametrize("n", [2, 4])
def test_replay_allgather_broadcast_alltoall(zc, n):
    rng = np.random.default_rng(n)
    g = zc.Group(n)
    block = (3 << 20) // 4 + 11
    for call in range(3):
        blocks = [rng.integers(-5000 * (call + 1), 5000, block).astype(np.int32) for _ in range(n)]
        outs = [torch.zeros(n * block, dtype=torch.int32, device=DEV) for _ in range(n)]
        # fixed output buffers across calls so the replay path is taken
        if call == 0:
            keep = outs
        for r in range(n):
            keep[r].zero_()
            keep[r][r * block:(r + 1) * block] = t(blocks[r])
        from paper_2605_12396_b200.zcomm import lib, check
        check(lib().zc_group_allgather_sym(g._h, n, g._ptrs(keep), block))
        want = np.concatenate(blocks)
        for o in keep:
            assert np.array_equal(o.cpu().numpy(), want), call
        data = [t(blocks[0]) if r == 1 else torch.zeros(block, dtype=torch.int32, device=DEV) for r in range(n)]
        if call == 0:
            bkeep = data
        else:
            for r in range(n):
                bkeep[r].copy_(data[r])
        g.broadcast(bkeep, 1)
        for d in bkeep:
            assert np.array_equal(d.cpu().numpy(), blocks[0]), call
        sends = [rng.integers(-3000, 3000, n * 4099).astype(np.int32) for _ in range(n)]
        if call == 0:
            skeep = [t(s) for s in sends]
            rkeep = [torch.empty(n * 4099, dtype=torch.int32, device=DEV) for _ in range(n)]
        else:
            for a, s in zip(skeep, sends):
                a.copy_(t(s))
        check(lib().zc_group_alltoall_sym(g._h, n, g._ptrs(skeep), g._ptrs(rkeep), 4099))
        for d in range(n):
            want = np.concatenate([sends[s][d * 4099:(d + 1) * 4099] for s in range(n)])
            assert np.array_equal(rkeep[d].cpu().numpy(), want), call
