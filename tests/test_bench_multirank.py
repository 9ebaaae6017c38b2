"""bench.py's N>1 host logic on CPU with gloo, world_size 2: the step time is the max over ranks
and the value is the whole-job aggregate (replicas only)."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    local = [12.5, 40.0][rank]
    m = bench.max_over_ranks(local, "cpu")
    assert bench.dist_env() == (ws, rank, 0)
    q.put((rank, m, bench.whole_job_value(10, ws, m)))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [o[1] for o in out] == [40.0, 40.0]
    assert out[0][2] == pytest.approx(10 * 2 / 0.040)


def test_single_process_is_identity():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.max_over_ranks(3.0, "cpu") == 3.0
    assert bench.whole_job_value(50, 1, 100.0) == pytest.approx(500.0)
