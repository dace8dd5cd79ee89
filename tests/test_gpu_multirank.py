"""Source-batch sharding through bench.py on ONE GPU with two ranks (
VERDICT r1 item 7).

torchrun starts 2 ranks of bench.py --shard, both on cuda:0, over the gloo backend (host-staged
all-reduce of CUDA tensors: the ranks' kernels never wait on each other on the device).  Each rank
runs the source batches i = rank, rank + 2, ... of every graph through hm_closeness_partial, one
all-reduce sums the partial sums, hm_closeness_combine finalises, and every rank composes.  Rank 0
dumps one more step's results (bench.py --dump); they must equal the oracle's."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O
from synth import build_config

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name,V", [("C5", 8192), ("C4", 4096), ("C1", 1000)])
def test_shard_two_ranks_gloo_one_gpu(tmp_path, name, V):
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    dump = tmp_path / "dump.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--shard", "--backend", "gloo", "--same-device", "--config", name, "--V", str(V),
           "--steps", "1", "--warmup", "1", "--no-e2e", "--no-cpu-baseline", "--words", "8",
           "--dump", str(dump)]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([ln for ln in p.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["value"] > 0
    d = np.load(dump)
    h = build_config(name, V=V)
    Es = [set(map(tuple, L.tolist())) for L in h.layers]
    res = []
    for i, E in enumerate(Es):
        r = O.analyze(h.V, E)
        res.append(r)
        assert d[f"L{i}_S"].tolist() == r["S"] and d[f"L{i}_k"].tolist() == r["k"]
        assert d[f"L{i}_pen"].tolist() == r["pen"] and d[f"L{i}_c"].tolist() == r["c"]
    K = h.K
    for T in h.subsets:
        tag = "".join(map(str, T))
        ra = O.analyze(h.V, O.and_aggregate([Es[i] for i in T]))
        assert d[f"AND{tag}_S"].tolist() == ra["S"] and d[f"AND{tag}_c"].tolist() == ra["c"]
        rs = [res[i] for i in T]
        assert d[f"gt_{tag}"].tolist() == O.topk_closeness(ra["c"], K)
        assert d[f"cc2_{tag}"].tolist() == O.cc2(rs, K)[0]
        assert d[f"cc1_{tag}"].tolist() == O.cc1(rs, K)[0]
        assert d[f"naive_{tag}"].tolist() == O.naive(rs, K)[0]
