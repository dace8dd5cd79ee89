"""GPU parity at BASELINE.json's full sizes, EVERY output, in the launch
configuration bench.py times (library defaults: 4096 sources per batch, 16-lane
row teams, L2 policy hints, interleaved work units, 2-core pruning; layers
loaded from device tensors; every graph of the step through one hm_closeness_multi
call, as bench.py's Psi -- plus the fused / separate variants of that call).

Expected values come from tests/golden/fullsize_<C>.json, written by
tools/oracle_golden.py, which runs ONLY the oracle (oracle/) on the inputs of
synth/ at full size and stores SHA-256 digests of every output in the byte
layouts of tests/_digest.py, keyed by the SHA-256 of the inputs.  Compared
bit-exactly here:
  * per layer and per AND subset: S, k, closeness (IEEE bits), n-penalty sums,
    degrees, the CC-node set and its mean mu;
  * per subset: the AND and OR edge sets, the ground-truth top-K
    (PAPER.md:205-209), CC2 top-K (Alg. 1), CC1's whole ranked set R (K = V;
    Eq. 2-3 and the pseudocode), the naive set
    and the CC2 above-average set, and the accuracy metrics of each heuristic's
    top-K against the GT top-K;
  * mu == math.fsum(c) / V on the GPU's own closeness values (Z6).
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O
from oracle import _bfs
from synth import build_config
from _digest import sha, input_sha

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def Context():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2207_11662_b200 import build as B
    B.build()
    from paper_2207_11662_b200 import Context
    return Context


def cc1_name(T):
    return "cc1" if len(T) == 2 else "cc1_rary"


def golden(name):
    path = os.path.join(GOLDEN, f"fullsize_{name}.json")
    assert os.path.exists(path), f"{path} missing: run tools/oracle_golden.py {name}"
    return json.load(open(path))


def check_graph(ctx, g, V, want, what):
    got = ctx.closeness_results(g)                   # cached by the step's hm_closeness_multi
    deg = ctx.degrees(g)
    nodes, cnt, mu = ctx.cc_nodes(g)
    assert cnt == len(nodes) == want["n_CH"], what
    for key, arr, kind in (("S", got["S"], "S"), ("k", got["k"], "k"), ("c", got["c"], "c"),
                           ("pen", got["pen"], "pen"), ("deg", deg, "deg"), ("CH", nodes, "ids")):
        assert sha(arr, kind) == want[key], f"{what}: {key} differs from the oracle"
    assert int(got["S"].sum(dtype=np.uint64)) == want["sum_S"]
    assert mu.hex() == want["mu"], what
    # the mean is the correctly rounded sum / V of the GPU's own closeness values (Z6)
    assert mu == math.fsum(got["c"].tolist()) / V, what
    return got


KNOBS = {"default": {}, "noprune-w32-contig": {"bfs_prune": 0, "bfs_interleave": 0, "bfs_words": 32},
         "separate": {"bfs_fuse": 0}, "fused": {"bfs_fuse": 1}, "torder2": {"bfs_torder": 2}}


@pytest.mark.parametrize("name,knobs", [("C1", "default"), ("C2", "default"), ("C3", "default"),
                                        ("C4", "default"), ("C5", "default"),
                                        ("C4", "noprune-w32-contig"), ("C5", "noprune-w32-contig"),
                                        ("C2", "separate"), ("C3", "fused"), ("C1", "fused"), ("C4", "torder2")],
                         ids=["C1", "C2", "C3", "C4", "C5", "C4-noprune-w32", "C5-noprune-w32",
                              "C2-separate", "C3-fused", "C1-fused", "C4-torder2"])
def test_fullsize_config(Context, name, knobs):
    import torch
    gold = golden(name)
    h = build_config(name)
    assert input_sha(h) == gold["input_sha256"], "synthetic inputs changed since the digests were written"
    V, K = h.V, h.K
    with Context() as ctx:
        for k, v in KNOBS[knobs].items():
            ctx.set_param(k, v)
        ctx.load_layers(V, [torch.from_numpy(L).cuda() for L in h.layers])
        # bench's Psi: every layer and AND graph of the step in one hm_closeness_multi call (one fused
        # pass or one pass per graph, bfs_fuse)
        ands = [ctx.and_aggregate(want["T"]) for want in gold["ands"]]
        ctx.closeness_multi(list(range(len(h.layers))) + ands)
        for i in range(len(h.layers)):
            check_graph(ctx, i, V, gold["layers"][i], f"{name} layer {i}")
        for want, g in zip(gold["ands"], ands):
            T = want["T"]
            tag = f"{name} AND{T}"
            rp, col = ctx.graph_csr(g)
            src = np.repeat(np.arange(V, dtype=np.int64), np.diff(rp))
            keep = src < col
            keys = np.sort(src[keep] * V + col[keep])
            assert len(keys) == want["m"] and sha(keys, "edges") == want["edges"], tag
            check_graph(ctx, g, V, want, tag)
            assert ctx.topk_closeness(g, K).tolist() == want["gt_topk"], tag
            ids2, n2 = ctx.compose("cc2", T, K)
            assert ids2.tolist() == want["cc2_topk"] and n2 == K, tag
            ids1, n1 = ctx.compose(cc1_name(T), T, V)            # the whole ranked set R
            assert n1 == want["cc1_n"] and sha(ids1, "ids") == want["cc1_ranked"], tag
            ids1k, n1k = ctx.compose(cc1_name(T), T, K)          # bench's call
            assert ids1k.tolist() == want["cc1_topk"] and n1k == want["cc1_n"], tag
            idsn, nn = ctx.compose("naive", T, V)
            assert nn == want["naive_n"] and sha(idsn, "ids") == want["naive"], tag
            idsa, na = ctx.compose("cc2_avg", T, V)
            assert na == want["cc2_avg_n"] and sha(idsa, "ids") == want["cc2_avg"], tag
            # the paper's evaluation: each heuristic's top-K against the GT top-K, on the
            # GPU's lists and set-metric kernel vs the oracle's plain Jaccard / P / R / F1 of its lists
            gt = ctx.topk_closeness(g, K)
            for heur, key in (("cc2", "cc2_topk"), (cc1_name(T), "cc1_topk"), ("naive", "naive_topk")):
                est, _ = ctx.compose(heur, T, K)
                m = ctx.set_metrics(V, est, gt)
                p_, r_, f_ = O.prf1(want[key], want["gt_topk"])
                assert (m["jaccard"], m["precision"], m["recall"], m["f1"]) == \
                    (O.jaccard(want[key], want["gt_topk"]), p_, r_, f_), (tag, heur)
            ctx.free_graph(g)
            # OR aggregation: the edge set
            go = ctx.or_aggregate(T)
            rp, col = ctx.graph_csr(go)
            src = np.repeat(np.arange(V, dtype=np.int64), np.diff(rp))
            keep = src < col
            keys = np.sort(src[keep] * V + col[keep])
            assert len(keys) == want["or_m"] and sha(keys, "edges") == want["or_edges"], tag + " OR"
            ctx.free_graph(go)


def test_large_vertex_count(Context):
    """The top of the supported range, V = 2^26 - 1 (67 M vertices, mostly isolated; R2 in
    DESIGN.md): 64-bit offsets, the relabelling of 67 M keys, the pruning paths, and frontier
    state sized by the vertices that can be BFS rows rather than by V.  A random forest plus
    cycles on 300 K scattered vertices (many components, long hanging trees) and one
    4097-vertex path; sampled vertices checked with the oracle's plain BFS, isolated vertices
    by definition."""
    V = (1 << 26) - 1
    rng = np.random.default_rng(24)
    verts = rng.choice(V, size=300_000, replace=False).astype(np.int64)
    E = []
    for i in range(1, len(verts)):                       # random forest on the scattered vertices
        if rng.random() < 0.97:
            E.append((verts[rng.integers(0, i)], verts[i]))
    for _ in range(60_000):                               # cycles
        a, b = rng.choice(len(verts), 2, replace=False)
        E.append((verts[a], verts[b]))
    path = np.arange(V - 4097, V, dtype=np.int64)          # ids up to V - 1
    E += list(zip(path[:-1], path[1:]))
    E = np.array(E, dtype=np.int64)
    E = np.sort(E, axis=1)
    E = np.unique(E[E[:, 0] != E[:, 1]], axis=0).astype(np.int32)
    with Context() as ctx:
        ctx.load_layers(V, [E])
        got = ctx.closeness(0)
        src = np.concatenate([rng.choice(verts, 24, replace=False), path[[0, 1, 2048, 4095, 4096]],
                              [0, V - 4098]]).astype(np.int32)
        S, k = _bfs.bfs_sources(V, E, np.sort(src), 0)
        src = np.sort(src)
        assert got["S"][src].tolist() == [int(x) for x in S]
        assert got["k"][src].tolist() == [int(x) for x in k]
        assert got["c"][src].tolist() == O.closeness_wf(V, [int(x) for x in S], [int(x) for x in k])
        deg = np.bincount(E.reshape(-1), minlength=V)
        iso = np.nonzero(deg == 0)[0][:1000]
        assert not got["S"][iso].any() and (got["k"][iso] == 1).all() and not got["c"][iso].any()
