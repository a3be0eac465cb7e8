"""GPU, two processes: the multi-process Communicator (one process per rank, CUDA IPC peer memory,
torch.distributed/gloo only for the rendezvous).  On the single-GPU test box both ranks share
device 0 — the same IPC mappings, flag protocol and kernels as two NVLink peers, time-sliced.
Results must equal the reference Communicator's (tests/golden)."""
import os
import socket
import sys
import traceback

import pytest
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, pin_name, q):
    try:
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), ZC_COMM_TIMEOUT_MS="60000")
        import numpy as np
        import torch
        import torch.distributed as dist
        from golden_data import GOLDEN, ring_input, sha
        from paper_2605_12396_b200 import abi, zcomm
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        k = GOLDEN["collectives"][f"ring{world}_{pin_name}"]
        base = ring_input(world)
        comm = zcomm.Communicator(rank, world, 0, zcomm.collective_config(k["pin"]))
        comm.set_shared_huffman(zcomm.HuffmanContext.from_bytes(base[0].view(np.uint8)[: abi.BATCH_RAW_BYTES].tobytes()))
        s = torch.from_numpy(base[rank].copy()).cuda()
        sc = comm.allreduce(s, 2e-4)
        torch.cuda.synchronize()
        w = comm.wire_stats()
        res = {"sha": sha(s.cpu().numpy()), "scale": sc, "frames": list(w.frames_by_codec),
               "payload": int(w.payload_bytes), "want": k}
        # the max ring and the eb AllReduce through the same communicator
        res["max"] = comm.allreduce_max(1.5 * rank - 1.0)
        comm.close()
        dist.destroy_process_group()
        q.put((rank, res, None))
    except Exception:
        q.put((rank, None, traceback.format_exc()))


@pytest.mark.parametrize("pin_name", ["auto", "huffman"])
def test_two_process_allreduce_equals_reference(pin_name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, pin_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, out, err = q.get(timeout=500)
        assert err is None, err
        res[rank] = out
    for p in procs:
        p.join(timeout=60)
    want = res[0]["want"]
    for r in range(world):
        assert res[r]["sha"] == want["out_sha256"]
        assert res[r]["scale"] == 2e-4
        assert res[r]["max"] == 0.5
    # wire stats are per rank here; their sum is the reference Communicator's total
    assert [res[0]["frames"][i] + res[1]["frames"][i] for i in range(3)] == want["wire"]["frames_by_codec"]
    assert res[0]["payload"] + res[1]["payload"] == want["wire"]["payload_bytes"]


def _worker_more(rank, world, port, q):
    """broadcast -> alltoall -> group_execute -> allreduce_qsgd through one multi-process communicator
    (the piece protocol across processes with a changing peer)."""
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), ZC_COMM_TIMEOUT_MS="60000",
                          ZC_COMM_REGION_UNITS="1")
        import numpy as np
        import torch
        import torch.distributed as dist
        from paper_2605_12396_b200 import abi, zcomm
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        comm = zcomm.Communicator(rank, world, 0, zcomm.collective_config(abi.PIN_AUTO))
        rng = np.random.default_rng(77)
        msg = rng.integers(-5000, 5000, (9 << 20) // 4 + 3).astype(np.int32)
        buf = torch.from_numpy(msg.copy() if rank == 1 else np.zeros_like(msg)).cuda()
        comm.broadcast(buf, 1)
        ok_b = bool(np.array_equal(buf.cpu().numpy(), msg))
        block = (5 << 20) // 4 + 1
        sends = [rng.integers(-900, 900, world * block).astype(np.int32) for _ in range(world)]
        out = comm.alltoall(torch.from_numpy(sends[rank]).cuda())
        want = np.concatenate([sends[j][rank * block:(rank + 1) * block] for j in range(world)])
        ok_a = bool(np.array_equal(out.cpu().numpy(), want))
        ar = [rng.integers(-100, 100, 100001).astype(np.int32) for _ in range(world)]
        reqs = [dict(op=abi.COLL_ALLREDUCE, sym=torch.from_numpy(ar[rank]).cuda(), scale=1.0),
                dict(op=abi.COLL_BROADCAST, sym=torch.from_numpy(msg[:1000].copy() if rank == 0 else
                                                                 np.zeros(1000, np.int32)).cuda(), root=0)]
        comm.group_execute(reqs)
        ok_g = bool(np.array_equal(reqs[0]["sym"].cpu().numpy(), ar[0] + ar[1])) and \
            bool(np.array_equal(reqs[1]["sym"].cpu().numpy(), msg[:1000]))
        xs = [rng.standard_normal(50001).astype(np.float32) for _ in range(world)]
        y = comm.allreduce_qsgd(torch.from_numpy(xs[rank]).cuda(), 8, 100 + rank)
        comm.close()
        dist.destroy_process_group()
        q.put((rank, {"b": ok_b, "a": ok_a, "g": ok_g, "qsgd": y.cpu().numpy(), "xs": xs}, None))
    except Exception:
        q.put((rank, None, traceback.format_exc()))


def test_two_process_more_collectives():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_more, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, out, err = q.get(timeout=500)
        assert err is None, err
        res[rank] = out
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert res[r]["b"] and res[r]["a"] and res[r]["g"], res[r]
    import numpy as np
    try:
        import oracle
        ref = oracle.ref()
    except Exception:  # noqa: BLE001
        ref = None
    if ref is not None:
        rc, exp = ref.allreduce_qsgd([x.astype(np.float64) for x in res[0]["xs"]], 8, [100, 101])
        assert rc == 0
        for r in range(world):
            assert np.array_equal(res[r]["qsgd"].view(np.uint64), exp[r].view(np.uint64))
