"""N > 1 path of bench.py on CPU (gloo, world size 2): every rank runs its own
replica, the job time is the max over ranks and the
job rate counts the work of all ranks."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = 100.0 * (rank + 1)  # rank 1 is the slow one
    m = bench.max_over_ranks(ms, dist)
    r = bench.job_rate(1e9, world, m)
    out[rank] = (m, r)
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for rank in range(world):
        m, r = out[rank]
        assert m == pytest.approx(200.0)
        assert r == pytest.approx(2 * 1e9 / 0.2)


def test_single_process_is_identity():
    import bench
    assert bench.max_over_ranks(12.5) == 12.5
    assert bench.job_rate(3e9, 1, 1500.0) == pytest.approx(2e9)
