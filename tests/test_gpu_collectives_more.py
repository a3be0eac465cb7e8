"""GPU parity of the remaining collectives on the frame path: alltoall
(collectives.cpp:546-567), broadcast (:569-591) and group_execute (:593-616), as loopback Groups
(N ranks in one process sharing the GPU, like the reference's thread-per-rank Communicator).

Bar: received symbols bit-identical to the data movement the reference performs; WireStats equal
to the frames the oracle's send path (encode_best / pinned send_batch per 4 MiB batch) produces
for every block each rank sends.  Small piece regions (ZC_COMM_REGION_UNITS=1) make every
exchange span several pieces, so region reuse across steps with a changing peer is exercised."""
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


def _frames_wire(port, blocks, pin, octx):
    """Expected WireStats of sending each int32 block once (oracle send path, batch by batch)."""
    cfgp = abi.default_collective_config(pin)
    fr = [0, 0, 0]
    raw = pay = tot = 0
    for b in blocks:
        for er, _ in port.encode_batches(b.view(np.uint8), pin, cfgp.hint, octx, cfgp.arb):
            fr[er.codec] += 1
            pay += er.payload_bytes
            tot += er.total_bytes
        raw += b.nbytes
    return fr, raw, pay, tot


def _check_wire(g, exp):
    w = g.wire_stats()
    assert list(w.frames_by_codec) == exp[0]
    assert (w.raw_bytes, w.payload_bytes, w.total_bytes) == exp[1:]


def _syms(rng, n):
    return np.clip(rng.laplace(0, 40, n), -2**20, 2**20).astype(np.int32)


@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_FIXEDLEN, abi.PIN_HUFFMAN, abi.PIN_RAW])
def test_alltoall_vs_reference_semantics(zc, port, monkeypatch, n, pin):
    monkeypatch.setenv("ZC_COMM_REGION_UNITS", "1")
    block = (9 << 20) // 4 + 3  # three pieces per exchange, the last one ragged
    rng = np.random.default_rng(31 * n + pin)
    sends = [_syms(rng, n * block) for _ in range(n)]
    sample = sends[0].view(np.uint8)[: 1 << 20]
    g = zc.Group(n, cfg=zc.collective_config(pin))
    g.set_shared_huffman(zc.HuffmanContext.from_bytes(sample))
    outs = g.alltoall([t(s) for s in sends])
    for r in range(n):
        want = np.concatenate([sends[j][r * block:(r + 1) * block] for j in range(n)])
        assert np.array_equal(npy(outs[r]), want)
    octx = port.huff_from_bytes(sample)
    sent = [sends[r][((r + k) % n) * block:((r + k) % n + 1) * block] for r in range(n) for k in range(1, n)]
    _check_wire(g, _frames_wire(port, sent, pin, octx))
    g.close()


def test_alltoall_uneven_rejected(zc):
    g = zc.Group(3)
    with pytest.raises(ValueError):
        g.alltoall([t(np.zeros(10, np.int32)) for _ in range(3)])


@pytest.mark.parametrize("n,root", [(2, 0), (3, 1), (4, 3)])
@pytest.mark.parametrize("pin", [abi.PIN_AUTO, abi.PIN_HUFFMAN])
def test_broadcast_chain(zc, port, monkeypatch, n, root, pin):
    monkeypatch.setenv("ZC_COMM_REGION_UNITS", "1")
    count = (10 << 20) // 4 + 5
    rng = np.random.default_rng(7 * n + root)
    data = _syms(rng, count)
    sample = data.view(np.uint8)[: 1 << 20]
    g = zc.Group(n, cfg=zc.collective_config(pin))
    g.set_shared_huffman(zc.HuffmanContext.from_bytes(sample))
    bufs = [t(data) if r == root else torch.full((count,), -7, dtype=torch.int32, device=DEV) for r in range(n)]
    g.broadcast(bufs, root)
    for b in bufs:
        assert np.array_equal(npy(b), data)
    # n-1 hops, each ships the message's frames (collectives.cpp:579-590)
    _check_wire(g, _frames_wire(port, [data] * (n - 1), pin, port.huff_from_bytes(sample)))
    with pytest.raises(ValueError):
        g.broadcast(bufs, n)
    g.close()


def test_mixed_sequence_keeps_protocol_consistent(zc, monkeypatch):
    """broadcast (ring edges only) then alltoall (every pair) then allreduce / allgather: the piece
    counters must stay consistent across collectives of different shapes."""
    monkeypatch.setenv("ZC_COMM_REGION_UNITS", "1")
    n = 3
    rng = np.random.default_rng(5)
    g = zc.Group(n)
    msg = _syms(rng, (9 << 20) // 4)
    bufs = [t(msg) if r == 2 else torch.zeros(msg.size, dtype=torch.int32, device=DEV) for r in range(n)]
    g.broadcast(bufs, 2)
    for b in bufs:
        assert np.array_equal(npy(b), msg)
    block = (5 << 20) // 4
    sends = [_syms(rng, n * block) for _ in range(n)]
    outs = g.alltoall([t(s) for s in sends])
    for r in range(n):
        assert np.array_equal(npy(outs[r]), np.concatenate([sends[j][r * block:(r + 1) * block] for j in range(n)]))
    syms = [_syms(rng, (13 << 20) // 4 + 1) for _ in range(n)]
    ts = [t(s) for s in syms]
    g.allreduce(ts, [1.0] * n)
    total = np.sum(np.stack(syms).astype(np.int64), axis=0).astype(np.int32)
    for x in ts:
        assert np.array_equal(npy(x), total)
    g.broadcast(ts, 0)
    outs = g.allgather([x[:1000] for x in ts])
    for o in outs:
        assert np.array_equal(npy(o), np.tile(total[:1000], n))
    g.close()


def test_group_execute_matches_one_by_one(zc):
    """group_execute runs the requests in order with the results of running them one by one."""
    n = 3
    rng = np.random.default_rng(11)
    ar = [_syms(rng, 300001) for _ in range(n)]
    a2a = [_syms(rng, n * 50000) for _ in range(n)]
    ag = [_syms(rng, 7000) for _ in range(n)]
    bc = _syms(rng, 123457)
    g = zc.Group(n)
    reqs = []
    for r in range(n):
        reqs.append([
            dict(op=abi.COLL_ALLREDUCE, sym=t(ar[r]), scale=0.5 * (r + 1)),
            dict(op=abi.COLL_ALLTOALL, sym=t(a2a[r]), recv=torch.empty(n * 50000, dtype=torch.int32, device=DEV),
                 nranks=n),
            dict(op=abi.COLL_BROADCAST, sym=t(bc) if r == 1 else torch.zeros(bc.size, dtype=torch.int32, device=DEV),
                 root=1),
            dict(op=abi.COLL_ALLGATHER, sym=t(ag[r]), recv=torch.empty(n * 7000, dtype=torch.int32, device=DEV)),
        ])
    g.group_execute(reqs)
    # allreduce with scale reconciliation: shared scale 1.5, symbols requantized llround(s * f)
    want = np.zeros(300001, np.int64)
    for r in range(n):
        f = (0.5 * (r + 1)) / 1.5
        x = ar[r].astype(np.float64) * f  # llround(s * f), half away from zero (collectives.cpp:454-456)
        want += (np.sign(x) * np.floor(np.abs(x) + 0.5)).astype(np.int64) if f != 1.0 else ar[r]
    for r in range(n):
        assert reqs[r][0]["scale"] == 1.5
        assert np.array_equal(npy(reqs[r][0]["sym"]), want.astype(np.int32))
        assert np.array_equal(npy(reqs[r][1]["recv"]),
                              np.concatenate([a2a[j][r * 50000:(r + 1) * 50000] for j in range(n)]))
        assert np.array_equal(npy(reqs[r][2]["sym"]), bc)
        assert np.array_equal(npy(reqs[r][3]["recv"]), np.concatenate(ag))
    bad = [[dict(op=abi.COLL_ALLGATHER, sym=t(ag[r]))] for r in range(n)]
    with pytest.raises(ValueError):
        g.group_execute(bad)
    g.close()


def test_measured_timeline(zc, monkeypatch):
    """zc_comm_timeline_*: one send row per batch with its frame, joined with the receiver's decode
    of the same piece; the times are causally ordered and the CSV has the reference's columns."""
    from paper_2605_12396_b200 import report
    monkeypatch.setenv("ZC_COMM_REGION_UNITS", "1")
    n = 2
    rng = np.random.default_rng(3)
    syms = [_syms(rng, (12 << 20) // 4 + 9) for _ in range(n)]
    g = zc.Group(n)
    g.timeline_enable(256)
    ts = [t(s) for s in syms]
    g.allreduce(ts, [1.0] * n)
    rows = g.timeline()
    w = g.wire_stats()
    # every frame the ring sent has a row (meta frames are host-counted control frames, not pieces)
    assert len(rows) == sum(1 for _ in rows) == w.frames_by_codec[0] + w.frames_by_codec[1] + w.frames_by_codec[2] - 2
    for r in rows:
        assert r["enc_start_sec"] <= r["enc_end_sec"] <= r["dec_end_sec"] + 1e-6
        assert r["dec_start_sec"] <= r["dec_end_sec"]
        assert r["total_bytes"] > 32 and r["raw_bytes"] <= 4 << 20
    csv = report.emit_timeline_csv(rows)
    assert csv.splitlines()[0] == report.TIMELINE_HEADER and len(csv.splitlines()) == len(rows) + 1
    s = report.overlap_summary(rows)
    assert s["overlap_sec"] >= 0 and s["span_sec"] > 0
    g.close()
