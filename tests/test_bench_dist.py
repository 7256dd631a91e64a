"""CPU (gloo, world_size 2) coverage of bench.py's multi-process host logic: whole-job iterations are
summed over ranks and the time is the max over ranks (replicas, weak scaling)."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    dist = bench.init_dist(world, "gloo")
    it, ms = bench.reduce_job(100.0 + rank, 10.0 * (rank + 1), dist)
    bench.barrier(dist)
    q.put((rank, it, ms))
    dist.destroy_process_group()


def test_reduce_job_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, it, ms in out:
        assert it == pytest.approx(201.0)
        assert ms == pytest.approx(20.0)


def test_reduce_job_single_process():
    import bench
    assert bench.reduce_job(5.0, 2.0, None) == (5.0, 2.0)
