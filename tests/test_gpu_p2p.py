"""GPU parity of the point-to-point path and of Communicator::run (collectives.cpp:137-173,
350-364): RankCtx::send_encoded / recv_decoded between any two ranks of a loopback Group, the
sender's WireStats equal to the oracle's send_batch accounting over the same batches (4 MiB, or
512 KiB slots under per-slot framing), and the reference's failure semantics (a rank whose body
throws poisons the links; run re-raises the root cause; the communicator stays usable)."""
import numpy as np
import pytest
import torch

from paper_2605_12396_b200 import abi

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]
DEV = "cuda"


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _oracle_send_wire(port, raw, pin, ctx, step):
    """send_encoded's accounting (collectives.cpp:285-296) over `raw` cut at `step` bytes."""
    frames, pay, tot = [0, 0, 0], 0, 0
    for off in range(0, len(raw), step):
        r, _ = port.send_batch(raw[off:off + step], pin, abi.make_hint(), ctx, None, cap=abi.STAGE_BANK_BYTES)
        frames[r.codec] += 1
        pay += r.payload_bytes
        tot += r.total_bytes
    return frames, pay, tot


@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_RAW, abi.PIN_FIXEDLEN, abi.PIN_HUFFMAN])
@pytest.mark.parametrize("per_slot", [0, 1])
def test_send_recv_vs_oracle(zc, port, pin, per_slot):
    rng = np.random.default_rng(11 + pin + 4 * per_slot)
    count = (10 << 20) // 4 + 13  # three 4 MiB batches (the last ragged), or 21 slots
    x = np.clip(rng.laplace(0, 60, count), -2**20, 2**20).astype(np.int32)
    sample = x.view(np.uint8)[: 1 << 20]
    g = zc.Group(2, cfg=zc.collective_config(pin, per_slot_framing=per_slot))
    g.set_shared_huffman(zc.HuffmanContext.from_bytes(sample))
    src = t(x)
    dst = torch.zeros(count, dtype=torch.int32, device=DEV)

    def body(ctx):
        if ctx.rank() == 0:
            ctx.send_encoded(1, src)
        else:
            ctx.recv_decoded(0, dst)

    g.run(body)
    assert np.array_equal(dst.cpu().numpy(), x)
    frames, pay, tot = _oracle_send_wire(port, x.view(np.uint8), pin, port.huff_from_bytes(sample),
                                         abi.SLOT_BYTES if per_slot else abi.BATCH_RAW_BYTES)
    w = g.wire_stats()
    assert list(w.frames_by_codec) == frames
    assert (w.raw_bytes, w.payload_bytes, w.total_bytes) == (4 * count, pay, tot)


def test_send_recv_many_pieces_all_pairs(zc):
    """Messages of several pieces (more than the pair's two channel regions, so sender and receiver
    run concurrently) between every ordered pair of 3 ranks, one pair at a time (a barrier between
    transfers): each directed pair keeps its own channel and counters."""
    import threading
    n = 3
    rng = np.random.default_rng(5)
    count = (70 << 20) // 4 + 5
    pairs = [(a, b) for a in range(n) for b in range(n) if a != b]
    data = {k: rng.integers(-5000, 5000, count).astype(np.int32) for k in pairs}
    src = {k: t(v) for k, v in data.items()}
    dst = {k: torch.zeros(count, dtype=torch.int32, device=DEV) for k in pairs}
    g = zc.Group(n)
    bar = threading.Barrier(n)

    def body(ctx):
        r = ctx.rank()
        for rep in range(2):  # twice: the pair counters carry over between messages
            for (a, b) in pairs:
                if r == a:
                    ctx.send_encoded(b, src[(a, b)])
                elif r == b:
                    ctx.recv_decoded(a, dst[(a, b)])
                bar.wait()

    g.run(body)
    for k, v in data.items():
        assert np.array_equal(dst[k].cpu().numpy(), v), k


def test_point_to_point_reference_cases(zc):
    """test_collectives.cpp:221-265: a 12 MiB message of narrow symbols goes as 3 FixedLen frames;
    per-slot framing with a RAW pin carries 3 MiB in 6 frames."""
    rng = np.random.default_rng(7)
    src = (rng.integers(0, 100, 3 << 20) - 50).astype(np.int32)
    dst = torch.zeros(len(src), dtype=torch.int32, device=DEV)
    g = zc.Group(2)
    ts = t(src)
    g.run(lambda ctx: ctx.send_encoded(1, ts) if ctx.rank() == 0 else ctx.recv_decoded(0, dst))
    assert np.array_equal(dst.cpu().numpy(), src)
    w = g.wire_stats()
    assert list(w.frames_by_codec) == [0, 3, 0]
    assert w.raw_bytes == 12 << 20 and w.payload_bytes < (12 << 20) // 4
    raw = (np.arange(3 << 20, dtype=np.uint64) * 31 % 256).astype(np.uint8)
    out = torch.zeros(len(raw), dtype=torch.uint8, device=DEV)
    g2 = zc.Group(2, cfg=zc.collective_config(abi.PIN_RAW, per_slot_framing=1))
    tr = t(raw)
    g2.run(lambda ctx: ctx.send_encoded(1, tr) if ctx.rank() == 0 else ctx.recv_decoded(0, out))
    assert np.array_equal(out.cpu().numpy(), raw)
    assert list(g2.wire_stats().frames_by_codec) == [6, 0, 0]


def test_run_root_cause_and_recovery(zc):
    """A rank whose body raises poisons the links: the peer blocked in recv_decoded fails with
    LinkPoisoned, run re-raises the root cause, and the group works afterwards
    (test_collectives.cpp:129-146 semantics)."""
    g = zc.Group(2)
    dst = torch.zeros(1 << 20, dtype=torch.int32, device=DEV)

    def body(ctx):
        if ctx.rank() == 1:
            raise ValueError("rank 1 fails before sending")
        ctx.recv_decoded(1, dst)

    with pytest.raises(ValueError, match="rank 1 fails"):
        g.run(body)
    syms = [t(np.array([1, 2, 3], np.int32)) for _ in range(2)]
    g.run(lambda ctx: ctx.allreduce(syms[ctx.rank()], 1.0))
    assert [s.cpu().tolist() for s in syms] == [[2, 4, 6], [2, 4, 6]]


def test_run_collectives_per_rank_threads(zc, port):
    """Collectives issued from the rank threads (the reference's usage) equal the group calls."""
    n, count = 4, (9 << 20) // 4 + 3
    rng = np.random.default_rng(3)
    syms = [rng.integers(-3000, 3000, count).astype(np.int32) for _ in range(n)]
    g = zc.Group(n)
    ts = [t(s) for s in syms]
    scales = g.run(lambda ctx: ctx.allreduce(ts[ctx.rank()], 1.0))
    assert scales == [1.0] * n
    want = np.sum(np.stack(syms).astype(np.int64), axis=0).astype(np.int32)
    for x in ts:
        assert np.array_equal(x.cpu().numpy(), want)
    assert g.run(lambda ctx: ctx.allreduce_max(float(ctx.rank()))) == [float(n - 1)] * n
