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


def _shard_worker(rank, world, port, out):
    """--shard host logic: each rank holds the target-side distance sums of its own
    sources (here sources s = rank mod world, distances by a plain BFS); one int64
    all-reduce (the uint64 sums viewed as int64, as bench.py does on NCCL) must give
    the oracle's S for every vertex."""
    import sys
    from collections import deque
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from synth import random_graph
    V = 80
    E = [tuple(e) for e in random_graph(V, 110, seed=5, kind="er").tolist()]
    adj = [[] for _ in range(V)]
    for u, v in E:
        adj[u].append(v)
        adj[v].append(u)
    part = np.zeros(V, np.uint64)
    for s in range(rank, V, world):
        dist_s = [-1] * V
        dist_s[s] = 0
        q = deque([s])
        while q:
            u = q.popleft()
            for w in adj[u]:
                if dist_s[w] < 0:
                    dist_s[w] = dist_s[u] + 1
                    q.append(w)
        for v in range(V):
            if dist_s[v] > 0:
                part[v] += np.uint64(dist_s[v])          # target side: S(v) += d(s, v)
    t = torch.from_numpy(part.view(np.int64).copy())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    out[rank] = t.numpy().view(np.uint64).tolist()
    dist.barrier()
    dist.destroy_process_group()


def test_shard_allreduce_two_ranks():
    from oracle import oracle as O
    from synth import random_graph
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_shard_worker, args=(2, port, out), nprocs=2, join=True)
    V = 80
    E = {tuple(e) for e in random_graph(V, 110, seed=5, kind="er").tolist()}
    S_ref = O.analyze(V, E)["S"]
    assert out[0] == S_ref and out[1] == S_ref
