"""Multi-rank host logic on CPU (gloo, world_size 2): replicas each time their
own HoMLN; the job value is units summed over ranks / max-over-ranks time."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    units = [10.0, 20.0][rank]
    ms = [100.0, 200.0][rank]
    val, tmax = bench.job_value(units, ms, device="cpu")
    out[rank] = (val, tmax)
    dist.barrier()
    dist.destroy_process_group()


def test_job_value_two_ranks():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        val, tmax = out[r]
        assert tmax == 200.0                       # max over ranks
        assert abs(val - 30.0 / 0.2) < 1e-9        # summed units / max time


def test_job_value_single_process():
    import bench
    val, tmax = bench.job_value(50.0, 250.0)
    assert tmax == 250.0 and abs(val - 200.0) < 1e-9
