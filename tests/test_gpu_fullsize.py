"""GPU parity at BASELINE.json's full sizes, in the launch configuration
bench.py times (the library defaults: 4096 sources per batch, 16-lane row teams,
L2 policy hints, interleaved work units).

The oracle cannot run all-sources BFS at these sizes in test time, so:
  * S, k, closeness, pen: exact on seeded samples of vertices, each checked
    with one plain oracle BFS (the target-side accumulation makes every
    vertex's value independent of the sample);
  * AND edge sets: exact, full (oracle set intersection);
  * top-K lists (GT, CC2, CC1, naive): properties that hold at any size --
    ids distinct, in rank order under the paper's key, and no vertex outside
    the list beats the last one; CC1 invariants (common CC nodes included,
    added vertices are common neighbours).
"""
import numpy as np
import pytest

from oracle import oracle as O
from oracle import _bfs
from synth import build_config

pytestmark = pytest.mark.gpu

N_SAMPLE = 48


@pytest.fixture(scope="module")
def Context():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2207_11662_b200 import build as B
    B.build()
    from paper_2207_11662_b200 import Context
    return Context


def sample_vertices(V, seed, n=N_SAMPLE):
    rng = np.random.default_rng(seed)
    s = rng.choice(V, size=min(n, V), replace=False)
    return np.sort(np.concatenate([s, [0, V - 1]])).astype(np.int32)


def check_sampled(V, E_arr, got, seed):
    src = sample_vertices(V, seed)
    S, k = _bfs.bfs_sources(V, E_arr, src, 0)
    S = [int(x) for x in S]
    k = [int(x) for x in k]
    c = O.closeness_wf(V, S, k)
    pen = O.pen_sum(V, S, k)
    assert got["S"][src].tolist() == S
    assert got["k"][src].tolist() == k
    assert got["c"][src].tolist() == c           # bit-exact (and within 1e-12 rel.)
    assert got["pen"][src].tolist() == pen


def check_ranked(ids, key, K):
    """ids must be the K smallest (key, id) pairs, in order."""
    ids = np.asarray(ids, dtype=np.int64)
    assert len(ids) == K and len(set(ids.tolist())) == K
    pairs = [(key[i], int(i)) for i in ids]
    assert pairs == sorted(pairs)
    mask = np.ones(len(key), bool)
    mask[ids] = False
    last = pairs[-1]
    rest_key = key[mask]
    rest_id = np.nonzero(mask)[0]
    # no excluded vertex precedes the last selected one
    better = (rest_key < last[0]) | ((rest_key == last[0]) & (rest_id < last[1]))
    assert not better.any()


def edges_of(rp, col):
    V = len(rp) - 1
    src = np.repeat(np.arange(V, dtype=np.int64), np.diff(rp))
    keep = src < col
    return src[keep] * V + col[keep]


@pytest.mark.parametrize("name,knobs", [("C1", {}), ("C2", {}), ("C3", {}), ("C4", {}), ("C5", {}),
                                        ("C4", {"bfs_prune": 0, "bfs_interleave": 0, "bfs_words": 32})],
                         ids=["C1", "C2", "C3", "C4", "C5", "C4-noprune-w32"])
def test_fullsize_config(Context, name, knobs):
    h = build_config(name)
    V, K = h.V, h.K
    with Context() as ctx:
        for k, v in knobs.items():
            ctx.set_param(k, v)
        ctx.load_layers(V, h.layers)
        res = []
        for i, L in enumerate(h.layers):
            got = ctx.closeness(i)
            check_sampled(V, L, got, seed=100 + i)
            res.append(got)
        degs = [ctx.degrees(i) for i in range(len(h.layers))]
        chs = []
        for i in range(len(h.layers)):
            nodes, cnt, mu = ctx.cc_nodes(i)
            c = res[i]["c"]
            assert cnt == len(nodes)
            assert set(nodes.tolist()) == set(np.nonzero(c > mu)[0].tolist())
            chs.append(set(nodes.tolist()))
        Es = None
        for t_i, T in enumerate(h.subsets[:4]):          # C3 has 10 subsets: test 4 of them here
            T = list(T)
            g = ctx.and_aggregate(T)
            rp, col = ctx.graph_csr(g)
            got_keys = np.sort(edges_of(rp, col))
            if Es is None:
                Es = [set(map(tuple, L.tolist())) for L in h.layers]
            A = O.and_aggregate([Es[i] for i in T])
            want = np.sort(np.array([u * V + v for u, v in A], dtype=np.int64))
            assert np.array_equal(got_keys, want)
            A_arr = np.array(sorted(A), dtype=np.int32).reshape(-1, 2)
            ga = ctx.closeness(g)
            check_sampled(V, A_arr, ga, seed=200 + t_i)
            # ground truth top-K: closeness descending, id ascending
            gt = ctx.topk_closeness(g, K)
            check_ranked(gt, -ga["c"], K)
            # CC2: est = max pen over the subset, ascending
            est = np.max(np.stack([res[i]["pen"] for i in T]), axis=0)
            ids2, n2 = ctx.compose("cc2", T, K)
            assert n2 == K
            check_ranked(ids2, est, K)
            # naive: common CC nodes, by id
            common = set.intersection(*[chs[i] for i in T])
            idsn, nn = ctx.compose("naive", T, K)
            assert nn == len(common) and idsn.tolist() == sorted(common)[:K]
            # CC1: R contains the common CC nodes; added vertices are common neighbours
            # of a common CC node (candidates lie in every layer's NBD); ranked by
            # RN(est / mindeg), id
            ids1, n1 = ctx.compose("cc1", T, min(V, max(K, n2)))
            assert n1 >= len(common)
            mindeg = np.min(np.stack([degs[i] for i in T]), axis=0)
            key1 = np.full(V, np.inf)
            sel = np.asarray(ids1, dtype=np.int64)
            key1[sel] = est[sel].astype(np.float64) / mindeg[sel].astype(np.float64)
            pairs = [(key1[i], int(i)) for i in sel]
            assert pairs == sorted(pairs)
            if n1 <= len(sel):
                Rset = set(sel.tolist())
                assert common <= Rset
                adjA = {}
                src = np.repeat(np.arange(V), np.diff(rp))
                for u in common:
                    adjA[u] = set(col[rp[u]:rp[u + 1]].tolist())
                for v in Rset - common:
                    assert any(v in adjA[u] for u in common)
            ctx.free_graph(g)


def test_large_vertex_count(Context):
    """The top of the supported range, V = 2^26 - 1 (67 M vertices, mostly isolated; R2 in
    DESIGN.md): 64-bit offsets, the relabelling of 67 M keys, the pruning paths, and frontier
    state sized by the vertices that can be BFS rows rather than by V.  A random forest plus cycles on 300 K scattered
    vertices (many components, long hanging trees) and one 4097-vertex path; sampled
    vertices checked with the oracle's plain BFS, isolated vertices by definition."""
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
