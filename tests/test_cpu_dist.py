"""CPU, world_size 2 over gloo: the multi-process host logic of the N>1 path.

The data path (ring steps over peer memory) needs GPUs; what runs on the host per rank is the
rendezvous — CollectiveConfig agreement (a mismatch raises ValueError on every rank, like the
reference's stream-meta check, collectives.cpp:428-452), the rank-ordered exchange of the CUDA IPC
blobs, and bench.py's max-over-ranks timing.  These are exercised here with two real processes.
"""
import os
import socket
import sys
import traceback

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, scenario, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import torch.distributed as dist
        from paper_2605_12396_b200 import abi, zcomm
        dist.init_process_group("gloo", rank=rank, world_size=world)
        out = None
        if scenario == "exchange":
            got = zcomm._dist_allgather_bytes(bytes([rank]) * (3 + rank))
            out = [bytes(b) for b in got]
        elif scenario == "config_ok":
            zcomm.check_consistent_config(abi.default_collective_config(), rank, zcomm._dist_allgather_bytes)
            out = "ok"
        elif scenario == "config_mismatch":
            cfg = abi.default_collective_config()
            if rank == 1:
                cfg.hint.beta_eff_bytes_per_sec = 900e9
            try:
                zcomm.check_consistent_config(cfg, rank, zcomm._dist_allgather_bytes)
                out = "no error"
            except ValueError as e:
                out = f"ValueError: {e}"
        elif scenario == "pin_mismatch":
            cfg = abi.default_collective_config(abi.PIN_FIXEDLEN if rank == 0 else abi.PIN_AUTO)
            try:
                zcomm.check_consistent_config(cfg, rank, zcomm._dist_allgather_bytes)
                out = "no error"
            except ValueError as e:
                out = f"ValueError: {e}"
        elif scenario == "max":
            import bench
            out = bench.max_over_ranks(1.5 + rank)
        dist.destroy_process_group()
        q.put((rank, out, None))
    except Exception:
        q.put((rank, None, traceback.format_exc()))


def _run(scenario, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, scenario, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, out, err = q.get(timeout=120)
        assert err is None, err
        res[rank] = out
    for p in procs:
        p.join(timeout=60)
    return res


def test_ipc_blob_exchange_is_rank_ordered():
    res = _run("exchange")
    for r in (0, 1):
        assert res[r] == [b"\x00" * 3, b"\x01" * 4]


def test_matching_configs_pass():
    assert _run("config_ok") == {0: "ok", 1: "ok"}


@pytest.mark.parametrize("scenario", ["config_mismatch", "pin_mismatch"])
def test_mismatched_configs_raise_on_every_rank(scenario):
    res = _run(scenario)
    for r in (0, 1):
        assert res[r].startswith("ValueError") and "differs on rank" in res[r], res


def test_bench_max_over_ranks():
    assert _run("max") == {0: 2.5, 1: 2.5}
