"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by
element, on the same seeded inputs.

Bars (BASELINE.json north_star): S, k, pen, AND edge sets, CC-node sets and
every top-K list bit-exact; closeness within 1e-12 relative (the pinned
formula is also expected, and asserted, to be bit-exact).
"""
import random

import numpy as np
import pytest

from oracle import oracle as O
from synth import build_config, random_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hm():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2207_11662_b200 import build as B
    B.build()
    from paper_2207_11662_b200 import Context
    return Context


def cc1_name(T):
    """CC1 is the paper's two-layer heuristic; r > 2 uses the opt-in flat r-ary form (Z12)."""
    return "cc1" if len(T) == 2 else "cc1_rary"


def edges_arr(E):
    return np.array(sorted(E), dtype=np.int32).reshape(-1, 2)


def check_psi(V, E, got, res=None):
    """compare the GPU closeness outputs with the oracle on (V, E)."""
    if res is None:
        res = O.analyze(V, E)
    assert got["S"].tolist() == res["S"]
    assert got["k"].tolist() == res["k"]
    assert got["pen"].tolist() == res["pen"]
    c_ref = np.array(res["c"], dtype=np.float64)
    rel = np.abs(got["c"] - c_ref) / np.maximum(np.abs(c_ref), 1e-300)
    assert np.all(rel <= 1e-12)
    assert np.array_equal(got["c"].view(np.uint64), c_ref.view(np.uint64))   # bit-exact
    return res


def run_graph(ctx, V, E):
    ctx.load_layers(V, [edges_arr(E)])
    return ctx.closeness(0)


# ---------------------------------------------------------------------------
# Psi on small graphs: edge cases and random shapes
# ---------------------------------------------------------------------------
def special_graphs():
    gs = []
    gs.append(("V1", 1, set()))
    gs.append(("V2-empty", 2, set()))
    gs.append(("V2-edge", 2, {(0, 1)}))
    gs.append(("empty-100", 100, set()))
    gs.append(("path-1500", 1500, {(i, i + 1) for i in range(1499)}))   # > 1000 levels
    gs.append(("star-3000", 3000, {(0, i) for i in range(1, 3000)}))    # degree >> 64
    gs.append(("cycle-777", 777, {(i, (i + 1) % 777) for i in range(777)} | set()))
    gs.append(("K40", 40, {(u, v) for u in range(40) for v in range(u + 1, 40)}))
    # two stars + isolated + a path (components of very different size)
    E = {(0, i) for i in range(1, 200)} | {(300, i) for i in range(301, 340)} | {(i, i + 1) for i in range(500, 900)}
    gs.append(("mixed-1000", 1000, E))
    # component exactly B, B+1 and 2B-1 sources (batch-window edges, W=16 -> B=1024)
    for n in (1024, 1025, 2047, 2049):
        gs.append((f"path-{n}", n, {(i, i + 1) for i in range(n - 1)}))
    gs.append(("tree-3000", 3000, {(i, (i - 1) // 2) for i in range(1, 3000)}))
    # hubs of degree 1100..3300 inside a sparse random core: heavy rows of 2-4 work items
    # (BFS_HEAVY_CHUNK = 1024 arcs) that stay unpeeled and change over several levels
    rng = random.Random(11662)
    E = {(rng.randrange(4000), rng.randrange(4000)) for _ in range(6000)}
    for h, deg in ((0, 3300), (1, 2100), (2, 1100), (3, 1025)):
        E |= {(h, u) for u in rng.sample(range(4, 4000), deg)}
    gs.append(("hubs-4000", 4000, E))
    return gs


@pytest.mark.parametrize("name,V,E", special_graphs(), ids=[g[0] for g in special_graphs()])
def test_psi_special(hm, name, V, E):
    E = {(min(u, v), max(u, v)) for u, v in E if u != v}
    res = O.analyze(V, E)
    # narrow batches (B = 512: several batches per component), other team widths and occupancies
    for words, team, bps, unit, prune, fbar in ((8, 0, 0, 8, 1, 1), (16, 4, 0, 16, 0, 0), (64, 32, 1, 32, 1, 0),
                                                (64, 16, 1, 4, 0, 1), (32, 16, 1, 2, 1, 1), (64, 16, 0, 8, 1, 1),
                                                (64, 0, 0, 2, 0, 1), (128, 0, 0, 0, 1, 1), (128, 0, 0, 4, 0, 0)):
        with hm() as ctx:
            if words == 128:                     # 8192 sources per batch: no heavy rows
                ctx.set_param("bfs_heavy", 1 << 30)
            ctx.set_param("bfs_fbar", fbar)
            ctx.set_param("bfs_prune", prune)
            ctx.set_param("bfs_words", words)
            ctx.set_param("bfs_unit", unit)
            ctx.set_param("bfs_team", team)
            ctx.set_param("bfs_blocks_per_sm", bps)
            check_psi(V, E, run_graph(ctx, V, E), res)
    with hm() as ctx:
        got = run_graph(ctx, V, E)
        check_psi(V, E, got, res)
        nodes, cnt, mu = ctx.cc_nodes(0)
        assert set(nodes.tolist()) == res["CH"] and cnt == len(res["CH"])
        assert mu == res["mu"]
        K = min(V, 17)
        assert ctx.topk_closeness(0, K).tolist() == O.topk_closeness(res["c"], K)


def test_psi_random_graphs(hm):
    rng = random.Random(2022)
    with hm() as ctx:
        for t in range(40):
            V = rng.choice([5, 33, 64, 65, 200, 513, 1000, 2500])
            m = rng.choice([0, V // 4, V // 2, V, 2 * V, 4 * V])
            kind = rng.choice(["er", "rmat"])
            E = {tuple(e) for e in random_graph(V, m, seed=1000 + t, kind=kind).tolist()}
            got = run_graph(ctx, V, E)
            res = check_psi(V, E, got)
            nodes, cnt, mu = ctx.cc_nodes(0)
            assert set(nodes.tolist()) == res["CH"], (t, V, m, kind)
            assert mu == res["mu"]
            assert ctx.degrees(0).tolist() == res["deg"]


def test_tuning_invariance(hm):
    """results do not depend on batch width, heavy-row threshold or grid size."""
    V = 3000
    E = {tuple(e) for e in random_graph(V, 6 * V, seed=77, kind="rmat").tolist()}
    res = O.analyze(V, E)
    for words in (8, 16, 32, 64, 128):
        for heavy in ((4, 64, 100000) if words < 128 else (1 << 30,)):
            for bps in ((0, 1) if words < 128 else (0,)):
                for chg_smem, unit, inter, prune, fbar in ((0, 32, 0, 0, 1), (1, 8, 1, 1, 0), (0, 2, 1, 1, 1)):
                    with hm() as ctx:
                        ctx.set_param("bfs_fbar", fbar)
                        ctx.set_param("bfs_prune", prune)
                        ctx.set_param("bfs_interleave", inter)
                        ctx.set_param("bfs_unit", unit)
                        ctx.set_param("bfs_words", words)
                        ctx.set_param("bfs_heavy", heavy)
                        ctx.set_param("bfs_blocks_per_sm", bps)
                        ctx.set_param("bfs_chg_smem", chg_smem)
                        check_psi(V, E, run_graph(ctx, V, E), res)


def test_loader_canonicalises(hm):
    """self-loops and duplicates dropped, either direction accepted."""
    V = 6
    raw = np.array([[0, 1], [1, 0], [2, 2], [1, 2], [2, 1], [4, 5], [0, 1]], dtype=np.int32)
    with hm() as ctx:
        _, dropped = ctx.load_layers(V, [raw])
        assert dropped == [4]
        rp, col = ctx.graph_csr(0)
        assert rp.tolist() == [0, 1, 3, 4, 4, 5, 6]
        assert col.tolist() == [1, 0, 2, 1, 5, 4]


def test_errors(hm):
    from paper_2207_11662_b200 import HmError
    with hm() as ctx:
        with pytest.raises(HmError, match="HM_ERANGE"):
            ctx.load_layers(4, [np.array([[0, 4]], np.int32)])
        with pytest.raises(HmError, match="HM_EINVAL"):
            ctx.load_layers(0, [np.zeros((0, 2), np.int32)])
        ctx.load_layers(5, [np.array([[0, 1]], np.int32), np.array([[0, 1], [1, 2]], np.int32)])
        with pytest.raises(HmError, match="HM_ESTATE"):
            ctx.compose("cc2", [0, 1], 2)                 # before closeness
        with pytest.raises(HmError, match="HM_EINVAL"):
            ctx.and_aggregate([0])
        with pytest.raises(HmError, match="HM_EINVAL"):
            ctx.and_aggregate([0, 0])
        with pytest.raises(HmError, match="HM_ESTATE"):
            ctx.and_aggregate([0, 7])
        ctx.closeness(0)
        with pytest.raises(HmError, match="HM_EINVAL"):
            ctx.topk_closeness(0, 6)
        with pytest.raises(HmError, match="HM_ESTATE"):
            ctx.free_graph(0)
        # tuning knobs: out-of-range values, and a combination with no compiled kernel
        for name, bad in (("bfs_words", 7), ("bfs_unit", 3), ("bfs_unit", 64), ("bfs_gd", 3), ("bfs_team", 2)):
            with pytest.raises(HmError, match="HM_EINVAL"):
                ctx.set_param(name, bad)
        with pytest.raises(HmError, match="HM_EINVAL"):
            ctx.set_param("no_such_knob", 1)
        ctx.set_param("bfs_team", 8)
        ctx.set_param("bfs_gd", 4)
        with pytest.raises(HmError, match="HM_EINVAL.*no MS-BFS kernel"):
            ctx.closeness(1)
        ctx.set_param("bfs_team", 0)
        ctx.set_param("bfs_gd", 0)
        # context stays usable after errors
        ctx.closeness(1)
        g = ctx.and_aggregate([0, 1])
        assert ctx.graph_info(g) == (5, 1)


# ---------------------------------------------------------------------------
# full pipeline on HoMLNs: AND, GT top-K, CC1, CC2, naive (exact)
# ---------------------------------------------------------------------------
def homln_cases():
    return [("C1", None), ("C2", 2048), ("C2", None), ("C3", 1024), ("C4", 2048), ("C5", 4096)]


def run_pipeline_and_compare(ctx, h, check_layers=True):
    V = h.V
    ids, _ = ctx.load_layers(V, h.layers)
    Es = [set(map(tuple, L.tolist())) for L in h.layers]
    refs = []
    for i in ids:
        got = ctx.closeness(i)
        refs.append(check_psi(V, Es[i], got) if check_layers else O.analyze(V, Es[i]))
        nodes, _, mu = ctx.cc_nodes(i)
        assert set(nodes.tolist()) == refs[-1]["CH"] and mu == refs[-1]["mu"]
    for T in h.subsets:
        K = min(h.K, V)
        g = ctx.and_aggregate(list(T))
        rp, col = ctx.graph_csr(g)
        A = O.and_aggregate([Es[i] for i in T])
        src = np.repeat(np.arange(V), np.diff(rp))
        gotE = {(int(a), int(b)) for a, b in zip(src, col) if a < b}
        assert gotE == A
        ra = check_psi(V, A, ctx.closeness(g))
        assert ctx.topk_closeness(g, K).tolist() == O.topk_closeness(ra["c"], K)
        rs = [refs[i] for i in T]
        ids2, n2 = ctx.compose("cc2", list(T), K)
        assert ids2.tolist() == O.cc2(rs, K)[0] and n2 == K
        ids1, n1 = ctx.compose(cc1_name(T), list(T), K)
        r1, nr1, _ = O.cc1(rs, K)
        assert n1 == nr1 and ids1.tolist() == r1
        idsn, nn = ctx.compose("naive", list(T), K)
        rn, nrn, _ = O.naive(rs, K)
        assert nn == nrn and idsn.tolist() == rn
        # CC2 "above average" selection: the whole set, ids ascending
        avg = sorted(O.cc2_above_average(rs))
        idsa, na = ctx.compose("cc2_avg", list(T), V)
        assert na == len(avg) and idsa.tolist() == avg
        # accuracy metrics of each estimate against the GT top-K
        gt = O.topk_closeness(ra["c"], K)
        for est in (ids2.tolist(), ids1.tolist(), idsn.tolist(), avg):
            m = ctx.set_metrics(V, est, gt)
            p, r, f = O.prf1(est, gt)
            assert (m["jaccard"], m["precision"], m["recall"], m["f1"]) == (O.jaccard(est, gt), p, r, f)
        ctx.free_graph(g)
        # OR aggregation, edge set exact
        go = ctx.or_aggregate(list(T))
        rp, col = ctx.graph_csr(go)
        src = np.repeat(np.arange(V), np.diff(rp))
        assert {(int(a), int(b)) for a, b in zip(src, col) if a < b} == O.or_aggregate([Es[i] for i in T])
        ctx.free_graph(go)


@pytest.mark.parametrize("name,V", homln_cases(), ids=[f"{n}@{v or 'full'}" for n, v in homln_cases()])
def test_pipeline_scaled_configs(hm, name, V):
    h = build_config(name, V=V)
    with hm() as ctx:
        run_pipeline_and_compare(ctx, h)


def test_cc1_golden_on_gpu(hm):
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cc1_six_vertex.json")))
    with hm() as ctx:
        ctx.load_layers(6, [np.array(g["L1"], np.int32), np.array(g["L2"], np.int32)])
        ctx.closeness(0)
        ctx.closeness(1)
        ids, n = ctx.compose("cc1", [0, 1], 6)
        assert ids.tolist() == g["CC1_ranked"] and n == 4
        assert ctx.compose("cc2", [0, 1], 3)[0].tolist() == g["CC2_top3"]
        assert ctx.compose("naive", [0, 1], 6)[0].tolist() == g["naive"]
        a = ctx.and_aggregate([0, 1])
        assert ctx.closeness(a)["S"].tolist() == g["AND_S"]
        assert ctx.topk_closeness(a, 3).tolist() == g["GT_top3"]


def test_cc1_golden_eight_vertex_on_gpu(hm):
    """the second hand-executed instance (isolated vertices, avgAND tie, |I| = 1)."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cc1_eight_vertex.json")))
    V = g["V"]
    with hm() as ctx:
        ctx.load_layers(V, [np.array(g["L1"], np.int32), np.array(g["L2"], np.int32)])
        for i, t in ((0, "1"), (1, "2")):
            got = ctx.closeness(i)
            assert got["S"].tolist() == g["S" + t] and got["pen"].tolist() == g["pen" + t]
            assert ctx.cc_nodes(i)[0].tolist() == g["CH" + t]
        ids, n = ctx.compose("cc1", [0, 1], V)
        assert ids.tolist() == g["CC1_ranked"] and n == len(g["CC1_R"])
        assert ctx.compose("cc1_rary", [1, 0], V)[0].tolist() == g["CC1_ranked"]
        assert ctx.compose("cc2", [0, 1], 4)[0].tolist() == g["CC2_top4"]
        assert ctx.compose("cc2_avg", [0, 1], V)[0].tolist() == g["CC2_avg"]
        assert ctx.compose("naive", [0, 1], V)[0].tolist() == g["naive"]
        a = ctx.and_aggregate([0, 1])
        ra = ctx.closeness(a)
        assert ra["S"].tolist() == g["AND_S"] and ra["pen"].tolist() == g["AND_pen"]
        assert ctx.cc_nodes(a)[0].tolist() == g["GT_CH"]
        assert ctx.topk_closeness(a, 3).tolist() == g["GT_top3"]


def test_cc1_pair_only_and_rary_opt_in(hm):
    """HM_CC1 is the paper's pair heuristic: r > 2 is rejected;
    HM_CC1_RARY is the explicit flat r-ary reading (Z12) and equals HM_CC1 at r = 2."""
    from paper_2207_11662_b200 import HmError
    h = build_config("C2", V=1024)
    with hm() as ctx:
        ctx.load_layers(h.V, h.layers)
        for i in range(3):
            ctx.closeness(i)
        with pytest.raises(HmError, match="HM_EINVAL"):
            ctx.compose("cc1", [0, 1, 2], 10)
        for T in ([0, 1], [1, 2], [2, 0]):
            assert ctx.compose("cc1", T, 50)[0].tolist() == ctx.compose("cc1_rary", T, 50)[0].tolist()
        Es = [set(map(tuple, L.tolist())) for L in h.layers]
        rs = [O.analyze(h.V, E) for E in Es]
        r1, n1, _ = O.cc1(rs, 50)
        ids, n = ctx.compose("cc1_rary", [0, 1, 2], 50)
        assert ids.tolist() == r1 and n == n1


def test_compose_device_outputs_sync_free(hm):
    """device ids + device count: K entries, -1 past |R|, same ranking as the host path."""
    import torch
    h = build_config("C5", V=4096)
    with hm() as ctx:
        ctx.load_layers(h.V, h.layers)
        for i in range(3):
            ctx.closeness(i)
        T = [0, 1, 2]
        for heur in ("cc1_rary", "cc2", "naive", "cc2_avg"):
            for K in (1, 7, 500, h.V):
                ref, n = ctx.compose(heur, T, K)
                out = torch.full((K,), -7, dtype=torch.int32, device="cuda")
                cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
                ctx.compose(heur, T, K, out=out, count_out=cnt)
                torch.cuda.synchronize()
                got = out.cpu().numpy()
                assert int(cnt.item()) == n
                m = min(K, n)
                assert got[:m].tolist() == ref.tolist()
                assert (got[m:] == -1).all()


def test_exact_mean_adversarial_on_gpu(hm):
    """GPU pin of the exact-sum reducer (the mean behind "higher than the
    average", and Eq. 3's averages): hm_exact_mean must equal
    math.fsum(x) / n (correctly rounded sum, one IEEE division), checked with Fraction, on arrays
    where plain summation is wrong: long tails of tiny terms, spans from 2^-1074 to 2^37,
    round-half-even ties, and sticky bits below the top three 32-bit limbs."""
    import math
    from fractions import Fraction
    import torch
    from paper_2207_11662_b200 import HmError

    def want(xs):
        exact = sum((Fraction(x) for x in xs), Fraction(0))
        s = float(exact)                                  # Fraction -> float rounds half to even
        assert s == math.fsum(xs)
        return s / len(xs) if xs else 0.0

    rng = random.Random(6)
    tiny = 5e-324                                          # 2^-1074
    cases = [
        [1.0] + [2.0 ** -53] * 1000,                       # tail that left-to-right drops
        [1.0, 2.0 ** -53],                                 # exact tie -> even (1.0)
        [1.0 + 2.0 ** -52, 2.0 ** -53],                    # tie -> even (rounds up)
        [1.0, 2.0 ** -53, 2.0 ** -140],                    # tie broken by a sticky bit far below
        [1.0, 2.0 ** -53, tiny],                           # ... by a subnormal
        [2.0 ** 37, 2.0 ** -16, 2.0 ** -70, tiny],         # 2^37 .. 2^-1074
        [2.0 ** 37] * 999 + [2.0 ** -1000] * 3,
        [1.0 / 3.0] * 999 + [2.0 ** -106],
        [0.1] * 10,
        [tiny] * 12345,                                    # subnormals only
        [2.0 ** -1022 - tiny, tiny],                       # subnormal carry into the normal range
        [float(2 ** 53 - 1), 0.5],                         # 2^53 - 1/2: tie at the top -> even
        [float(2 ** 53 - 1), 0.5, 2.0 ** -200],
        [rng.random() * 2.0 ** -rng.randint(0, 1074) for _ in range(20000)],
        [rng.random() * 2.0 ** rng.randint(-60, 37) for _ in range(100000)],
        [rng.randint(1, 10 ** 6) / rng.randint(10 ** 6, 10 ** 12) for _ in range(262144)],
        [0.0] * 5,
    ]
    with hm() as ctx:
        for xs in cases:
            mu, n = ctx.exact_mean(np.array(xs, dtype=np.float64))
            assert n == len(xs)
            assert mu == want(xs), (xs[:4], mu, want(xs))
        # masked mean over the selected values only (Eq. 3's finite ratios, Z8), device input
        x = np.array([rng.random() * 2.0 ** rng.randint(-30, 30) for _ in range(5000)])
        m = (np.arange(5000) % 3 != 0).astype(np.uint8)
        sel = [float(v) for v, k in zip(x, m) if k]
        mu, n = ctx.exact_mean(torch.from_numpy(x).cuda(), torch.from_numpy(m).cuda())
        assert n == len(sel) and mu == want(sel)
        assert ctx.exact_mean(np.zeros(0)) == (0.0, 0)
        assert ctx.exact_mean(x, np.zeros(5000, np.uint8)) == (0.0, 0)
        for bad in (-1.0, math.inf, math.nan):
            with pytest.raises(HmError, match="HM_EINVAL"):
                ctx.exact_mean(np.array([1.0, bad]))


def test_set_metrics_edge_cases(hm):
    """Jaccard / P / R / F1 incl. empty sets, duplicates, device
    lists and out-of-range ids (SPEC.md:370, :379 conventions)."""
    import torch
    from paper_2207_11662_b200 import HmError
    rng = random.Random(5)
    cases = [([], []), ([], [1, 2]), ([3], []), ([1, 1, 2], [2, 2]), (list(range(100)), list(range(50, 150)))]
    for _ in range(30):
        V = rng.choice([1, 31, 32, 33, 1000, 70000])
        cases.append(([rng.randrange(V) for _ in range(rng.randrange(0, 300))],
                      [rng.randrange(V) for _ in range(rng.randrange(0, 300))]))
    with hm() as ctx:
        for a, b in cases:
            V = max([0] + a + b) + 1
            m = ctx.set_metrics(V, a, b)
            p, r, f = O.prf1(a, b)
            assert (m["jaccard"], m["precision"], m["recall"], m["f1"]) == (O.jaccard(a, b), p, r, f), (a, b)
            assert (m["n_est"], m["n_gt"], m["n_common"]) == (len(set(a)), len(set(b)), len(set(a) & set(b)))
        a = torch.tensor([0, 5, 9], dtype=torch.int32, device="cuda")
        b = torch.tensor([5, 9, 11], dtype=torch.int32, device="cuda")
        assert ctx.set_metrics(12, a, b)["jaccard"] == 0.5
        with pytest.raises(HmError, match="HM_ERANGE"):
            ctx.set_metrics(10, [0, 10], [1])
        with pytest.raises(HmError, match="HM_EINVAL"):
            ctx.set_metrics(0, [], [])


@pytest.mark.parametrize("V", [4097, 8192, 8193, 40000, 300000])
def test_topk_paths_with_ties(hm, V):
    """top-K (ties to the lower id, Z14) on tie-heavy closeness vectors, through the
    one-launch tile select (topk_tiles 1: tiles of 8192, a ragged last tile, candidates G * K up to
    the 16384 limit) and the cooperative radix select (0): identical lists, equal to the oracle's
    ranking of the same closeness values.  The graph is many identical 6-cycles (equal closeness),
    isolated vertices (closeness 0) and a random sparse part."""
    rng = np.random.default_rng(V)
    E = set()
    n_cyc = V // 12
    for c in range(n_cyc):                              # identical 6-cycles: 6 * n_cyc tied vertices
        b = 6 * c
        E |= {(b + i, b + (i + 1) % 6) for i in range(6)}
    lo = 6 * n_cyc
    rest = np.arange(lo, V)
    sparse = rest[: len(rest) // 2]                      # the other half of `rest` stays isolated
    for _ in range(len(sparse)):
        a, b = rng.choice(sparse, 2)
        if a != b:
            E.add((int(min(a, b)), int(max(a, b))))
    with hm() as ctx:
        ctx.load_layers(V, [edges_arr(E)])
        c = ctx.closeness(0)["c"].tolist()
        G = (V + 8191) // 8192
        for K in sorted({1, 2, 7, 100, 1000, 4096, min(V, 16384 // G)}):
            if K > V or K > 4096:
                continue
            want = O.topk_closeness(c, K)
            got = {}
            for tiles in (1, 0):
                ctx.set_param("topk_tiles", tiles)
                got[tiles] = ctx.topk_closeness(0, K).tolist()
            assert got[1] == want and got[0] == want, (V, K)
        ctx.set_param("topk_tiles", 1)


def test_device_tensors_roundtrip(hm):
    import torch
    h = build_config("C5", V=2048)
    with hm() as ctx:
        layers = [torch.from_numpy(L).cuda() for L in h.layers]
        ctx.load_layers(h.V, layers)
        out = {"S": torch.zeros(h.V, dtype=torch.int64, device="cuda"),
               "k": torch.zeros(h.V, dtype=torch.int32, device="cuda"),
               "c": torch.zeros(h.V, dtype=torch.float64, device="cuda"),
               "pen": torch.zeros(h.V, dtype=torch.int64, device="cuda")}
        ctx.closeness(0, out=out)
        ctx.sync()
        res = O.analyze(h.V, set(map(tuple, h.layers[0].tolist())))
        assert out["S"].cpu().numpy().astype(np.uint64).tolist() == res["S"]
        assert out["c"].cpu().numpy().tolist() == res["c"]
        ids = torch.zeros(10, dtype=torch.int32, device="cuda")
        ctx.topk_closeness(0, 10, out=ids)
        ctx.sync()
        assert ids.cpu().tolist() == O.topk_closeness(res["c"], 10)


@pytest.mark.parametrize("name,V,fuse", [("C3", 1024, 1), ("C5", 4096, 1), ("C4", 2048, 1), ("C1", 1000, 1),
                                         ("C2", 4096, 2), ("C1", 1000, 2), ("C5", 2048, 0)])
def test_closeness_multi_fused(hm, name, V, fuse):
    """hm_closeness_multi over layers + AND graphs (one fused pass: bfs_fuse 1; automatic: 2; one pass
    per graph: 0) == separate passes == oracle; the fused pass makes no host round trip."""
    h = build_config(name, V=V)
    Es = [set(map(tuple, L.tolist())) for L in h.layers]
    with hm() as ctx:
        ctx.set_param("bfs_fuse", fuse)
        ids, _ = ctx.load_layers(h.V, h.layers)
        ands = [ctx.and_aggregate(list(T)) for T in h.subsets]
        gids = list(ids) + ands
        ctx.sync()
        ctx.stats(reset=True)
        ctx.closeness_multi(gids)
        st = ctx.stats(reset=True)
        fused_expected = len(gids) > 1 and (fuse == 1 or (fuse == 2 and V * len(gids) <= (1 << 17)))
        assert st["bfs_launches"] == (1 if fused_expected else len(gids))
        if fused_expected:
            assert st["host_syncs"] == 0
        fused = {g: ctx.closeness_results(g) for g in gids}
        fused_ch = {g: ctx.cc_nodes(g) for g in gids}
        for g in gids:
            sep = ctx.closeness(g)
            for key in ("S", "k", "c", "pen"):
                assert np.array_equal(fused[g][key], sep[key]), (g, key)
            nodes, cnt, mu = ctx.cc_nodes(g)
            assert np.array_equal(nodes, fused_ch[g][0]) and mu == fused_ch[g][2]
        for i in ids:
            check_psi(h.V, Es[i], fused[i])
        for T, g in zip(h.subsets, ands):
            check_psi(h.V, O.and_aggregate([Es[i] for i in T]), fused[g])


def test_closeness_multi_groups_unpruned(hm):
    """automatic fusing above 2^17 vertices: graphs whose cached pruning decision is "unpruned" are fused
    in groups of <= 2^17 vertices, pruned ones run alone; every result equals one pass per graph."""
    h = build_config("C3", V=40000)
    with hm() as ctx:
        ids, _ = ctx.load_layers(h.V, h.layers)
        ands = [ctx.and_aggregate(list(T)) for T in h.subsets]
        gids = list(ids) + ands
        ctx.set_param("bfs_fuse", 0)
        ctx.closeness_multi(gids)                      # caches every graph's pruning decision
        sep = {g: ctx.closeness_results(g) for g in gids}
        ctx.set_param("bfs_fuse", 2)
        ctx.sync()
        ctx.stats(reset=True)
        ctx.closeness_multi(gids)
        st = ctx.stats(reset=True)
        assert st["host_syncs"] == 0
        assert st["bfs_launches"] < len(gids)          # the ER layers share a pass
        for g in gids:
            got = ctx.closeness_results(g)
            for key in ("S", "k", "c", "pen"):
                assert np.array_equal(got[key], sep[g][key]), (g, key)


def test_closeness_multi_fresh_graphs_grouped(hm):
    """automatic fusing on graphs met for the first time: their pruning decisions are taken first in the
    same call, the unpruned ones fused; results equal one pass per graph (computed in another context)."""
    h = build_config("C5", V=65536)
    with hm() as ref:
        ids, _ = ref.load_layers(h.V, h.layers)
        ands = [ref.and_aggregate(list(T)) for T in h.subsets]
        ref.set_param("bfs_fuse", 0)
        ref.closeness_multi(list(ids) + ands)
        want = {g: ref.closeness_results(g) for g in list(ids) + ands}
    with hm() as ctx:
        ids, _ = ctx.load_layers(h.V, h.layers)
        ands = [ctx.and_aggregate(list(T)) for T in h.subsets]
        gids = list(ids) + ands
        ctx.sync()
        ctx.stats(reset=True)
        ctx.closeness_multi(gids)                      # fresh graphs: decide, then group
        st = ctx.stats(reset=True)
        assert st["bfs_launches"] < len(gids)          # the C5 layers (unpruned) share one pass
        for g in gids:
            got = ctx.closeness_results(g)
            for key in ("S", "k", "c", "pen"):
                assert np.array_equal(got[key], want[g][key]), (g, key)


# ---------------------------------------------------------------------------
# Top-down push phase on the first levels of a batch (bfs_push; north_star direction optimisation):
# the per-source push step and the hand-over to the bit-parallel bottom-up levels change no result
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,V", [("C5", 8192), ("C5", 16384), ("C4", 8192)])
def test_push_phase(hm, name, V):
    h = build_config(name, V=V)
    Es = [set(map(tuple, L.tolist())) for L in h.layers]
    T = list(h.subsets[0])
    Es.append(O.and_aggregate([Es[i] for i in T]))
    refs = [O.analyze(h.V, E) for E in Es]
    with hm() as ctx:
        ctx.load_layers(h.V, h.layers)
        gids = list(range(len(h.layers))) + [ctx.and_aggregate(T)]
        pushed = 0
        for words, prune, heavy in ((0, 2, 0), (64, 0, 1 << 20), (128, 1, 1 << 20), (64, 1, 1 << 20)):
            levels = {}
            for push in (0, 1, 4, 8, 64, 4096):
                for k, v in (("bfs_words", words), ("bfs_prune", prune), ("bfs_heavy", heavy), ("bfs_push", push)):
                    ctx.set_param(k, v)
                for g, E, res in zip(gids, Es, refs):
                    ctx.stats(reset=True)
                    check_psi(h.V, E, ctx.closeness(g), res)
                    st = ctx.stats(reset=True)
                    pushed += st["bfs_td_levels"]
                    assert levels.setdefault(g, st["bfs_levels"]) == st["bfs_levels"]   # the same levels either way
                if name == "C5" and words == 0 and push == 8:      # sharded and fused passes, same knob
                    for g, E, res in zip(gids, Es, refs):
                        tot = sum(ctx.closeness_partial(g, r, 2).astype(np.uint64) for r in range(2))
                        ctx.closeness_combine(g, tot)
                        check_psi(h.V, E, ctx.closeness_results(g), res)
                    ctx.set_param("bfs_fuse", 1)
                    ctx.closeness_multi(gids)
                    ctx.set_param("bfs_fuse", 2)
                    for g, E, res in zip(gids, Es, refs):
                        check_psi(h.V, E, ctx.closeness_results(g), res)
        assert pushed > 0                                 # push levels ran


def test_push_phase_small_components(hm):
    """batches that end inside the push phase (paths, cycles and cliques of <= 200 vertices) and a star
    whose hub row is walked by one lane: same results, same level count."""
    rng = random.Random(7)
    V, E, start = 6000, set(), 0
    while start < V - 1:
        n = min(V - start, rng.choice([2, 3, 5, 17, 64, 200]))
        vs = list(range(start, start + n))
        if n <= 17 and rng.random() < 0.3:
            E |= {(a, b) for i, a in enumerate(vs) for b in vs[i + 1:]}
        else:
            E |= {(vs[i], vs[i + 1]) for i in range(n - 1)}
            if n > 2 and rng.random() < 0.5:
                E.add((vs[0], vs[-1]))
        start += n + rng.choice([0, 1, 3])
    star = (5000, {(0, v) for v in range(1, 5000)} | {(v, v + 1) for v in range(1, 4999, 7)})
    for V, E in ((V, E), star):
        res = O.analyze(V, E)
        with hm() as ctx:
            ctx.load_layers(V, [edges_arr(E)])
            for words in (64, 128):
                levels = None
                for push in (0, 1, 8, 4096):
                    for k, v in (("bfs_words", words), ("bfs_prune", 0), ("bfs_heavy", 1 << 20), ("bfs_push", push)):
                        ctx.set_param(k, v)
                    ctx.stats(reset=True)
                    check_psi(V, E, ctx.closeness(0), res)
                    st = ctx.stats(reset=True)
                    assert push < 8 or st["bfs_td_levels"] > 0       # (threshold 1: the sources alone exceed it)
                    levels = st["bfs_levels"] if levels is None else levels
                    assert st["bfs_levels"] == levels


# ---------------------------------------------------------------------------
# Sharded Psi: partial sums over source-batch shards add up
# to S exactly, and finalising from the sum reproduces every cached result
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,V", [("C5", 8192), ("C3", 2048), ("C4", 2048)])
def test_sharded_closeness(hm, name, V):
    h = build_config(name, V=V)
    with hm() as ctx:
        ctx.set_param("bfs_words", 8)                   # B = 512: several batches per graph
        ctx.load_layers(h.V, h.layers)
        T = list(h.subsets[0])
        gids = list(range(len(h.layers))) + [ctx.and_aggregate(T)]
        full = {}
        for g in gids:
            full[g] = ctx.closeness(g)
            full[g]["topk"] = ctx.topk_closeness(g, h.K).tolist()
        ref_cc2 = ctx.compose("cc2", T, h.K)[0].tolist()
        ref_cc1 = ctx.compose(cc1_name(T), T, h.K)
        whole = {g: ctx.closeness_partial(g, 0, 1) for g in gids}
        for nshards in (1, 2, 3):
            for g in gids:
                parts = [ctx.closeness_partial(g, r, nshards) for r in range(nshards)]
                tot = np.sum(np.stack(parts).astype(np.uint64), axis=0, dtype=np.uint64)
                # the shards add up to the unsharded pre-finalisation sums (with 2-core pruning these
                # are the core's weighted sums; without it they are S itself)
                assert tot.tolist() == whole[g].tolist(), (g, nshards)
                ctx.closeness_combine(g, tot)
                got = ctx.closeness_results(g)
                for key in ("S", "k", "pen"):
                    assert got[key].tolist() == full[g][key].tolist()
                assert np.array_equal(got["c"].view(np.uint64), full[g]["c"].view(np.uint64))
                assert ctx.topk_closeness(g, h.K).tolist() == full[g]["topk"]
            assert ctx.compose("cc2", T, h.K)[0].tolist() == ref_cc2
            ids, n = ctx.compose(cc1_name(T), T, h.K)
            assert n == ref_cc1[1] and ids.tolist() == ref_cc1[0].tolist()
        with pytest.raises(Exception):
            ctx.closeness_partial(gids[0], 2, 2)
        ctx.set_param("bfs_prune", 0)                   # unpruned: the partial sums are S itself
        for g in gids:
            tot = ctx.closeness_partial(g, 0, 2) + ctx.closeness_partial(g, 1, 2)
            assert tot.tolist() == full[g]["S"].tolist()


# ---------------------------------------------------------------------------
# Randomised sweep: graph shapes x every tuning knob (results never depend on them)
# ---------------------------------------------------------------------------
def _shape(rng, t):
    """seeded test graphs with the structures that stress different paths: ER / R-MAT
    (hubs -> heavy rows), forests with a few cycles (deep hanging trees -> pruning),
    disjoint pieces of different size (component batching)."""
    V = rng.choice([2, 3, 7, 31, 32, 33, 100, 257, 700, 1500, 3000])
    kind = rng.choice(["er", "rmat", "forest", "pieces"])
    if kind in ("er", "rmat"):
        m = rng.choice([V // 2, V, 2 * V, 5 * V])
        return V, {tuple(e) for e in random_graph(V, max(m, 1), seed=5000 + t, kind=kind).tolist()}
    E = set()
    if kind == "forest":
        for v in range(1, V):
            if rng.random() < 0.95:
                u = rng.randrange(v)
                E.add((u, v))
        for _ in range(rng.randrange(0, max(1, V // 10))):
            a, b = rng.sample(range(V), 2)
            E.add((min(a, b), max(a, b)))
        return V, E
    start = 0
    while start < V - 1:                         # pieces: paths, cycles, cliques of random sizes
        n = min(V - start, rng.choice([2, 3, 5, 17, 64, 200]))
        shape = rng.choice(["path", "cycle", "clique"])
        vs = list(range(start, start + n))
        if shape == "clique" and n <= 17:
            E |= {(a, b) for i, a in enumerate(vs) for b in vs[i + 1:]}
        else:
            E |= {(vs[i], vs[i + 1]) for i in range(n - 1)}
            if shape == "cycle" and n > 2:
                E.add((vs[0], vs[-1]))
        start += n + rng.choice([0, 1, 3])
    return V, E


def test_random_sweep_all_knobs(hm):
    rng = random.Random(20220722)
    knobs = dict(bfs_words=[0, 8, 16, 32, 64, 128], bfs_prune=[0, 1, 2], bfs_interleave=[0, 1], bfs_hints=[0, 3, 11, 31],
                 bfs_chg_smem=[0, 1], bfs_unit=[0, 2, 4, 8, 16, 32], bfs_heavy=[0, 2, 16, 256], bfs_blocks_per_sm=[0, 1],
                 bfs_fbar=[0, 1], cc_init=[0, 1, 2, 3, 4], bfs_td=[0, 2, 8, 32, 1 << 20], bfs_torder=[0, 1, 2],
                 bfs_push=[-1, 0, 0, 1, 8, 64, 4096])
    with hm() as ctx:
        for t in range(200):
            V, E = _shape(rng, t)
            res = O.analyze(V, E)
            pick = {k: rng.choice(vals) for k, vals in knobs.items()}
            # gathers in flight: every instantiated value at W = 64, 2 CTAs/SM (the bench path)
            pick["bfs_gd"] = rng.choice([0, 2, 4, 8]) if pick["bfs_words"] == 64 and pick["bfs_blocks_per_sm"] != 1 else 0
            if pick["bfs_words"] == 128:           # 8192 sources per batch: graphs without heavy rows only
                pick.update(bfs_heavy=1 << 30, bfs_blocks_per_sm=0, bfs_gd=rng.choice([0, 4]))
            for k, v in pick.items():
                ctx.set_param(k, v)
            ctx.load_layers(V, [edges_arr(E)])
            check_psi(V, E, ctx.closeness(0), res)
            if t % 6 == 0 and V >= 3:                 # sharded path, same knobs
                n = rng.choice([2, 3])
                tot = sum(ctx.closeness_partial(0, r, n).astype(np.uint64) for r in range(n))
                ctx.closeness_combine(0, tot)
                check_psi(V, E, ctx.closeness_results(0), res)


# ---------------------------------------------------------------------------
# Steady state without host round trips: cached pruning decisions and CUDA-graph replay
# ---------------------------------------------------------------------------
def _step(ctx, h, outs):
    """one bench-style step into device tensors: closeness of every layer and of the AND graph,
    GT top-K and the three compositions."""
    T = list(h.subsets[0])
    g = ctx.and_aggregate(T)
    for i in range(len(h.layers)):
        ctx.closeness(i, out={"S": outs[f"S{i}"]})
    ctx.closeness(g, out={"S": outs["Sand"], "c": outs["cand"]})
    ctx.topk_closeness(g, h.K, out=outs["gt"])
    ctx.compose("cc2", T, h.K, out=outs["cc2"], count_out=outs["n2"])
    ctx.compose("cc1" if len(T) == 2 else "cc1_rary", T, h.K, out=outs["cc1"], count_out=outs["n1"])
    ctx.compose("naive", T, h.K, out=outs["naive"], count_out=outs["nn"])
    ctx.free_graph(g)


def _outs(h):
    import torch
    d = {f"S{i}": torch.zeros(h.V, dtype=torch.int64, device="cuda") for i in range(len(h.layers))}
    d.update(Sand=torch.zeros(h.V, dtype=torch.int64, device="cuda"),
             cand=torch.zeros(h.V, dtype=torch.float64, device="cuda"))
    for k in ("gt", "cc2", "cc1", "naive"):
        d[k] = torch.zeros(h.K, dtype=torch.int32, device="cuda")
    for k in ("n2", "n1", "nn"):
        d[k] = torch.zeros(1, dtype=torch.int32, device="cuda")
    return d


@pytest.mark.parametrize("name,V", [("C5", 8192), ("C4", 8192), ("C3", 4100)])
def test_steady_state_no_sync_and_graph_replay(hm, name, V):
    """The second step on the same layers makes no host round trip (the pruning decisions of the
    layers and of the AND aggregate are cached), its results equal the oracle's, and the same step
    captured in a CUDA graph and replayed writes identical results."""
    import torch
    h = build_config(name, V=V)
    Es = [set(map(tuple, L.tolist())) for L in h.layers]
    refs = [O.analyze(h.V, E) for E in Es]
    T = list(h.subsets[0])
    ra = O.analyze(h.V, O.and_aggregate([Es[i] for i in T]))
    rs = [refs[i] for i in T]
    with hm() as ctx:
        ctx.load_layers(h.V, [torch.from_numpy(L).cuda() for L in h.layers])
        a = _outs(h)
        _step(ctx, h, a)                                  # first step: decisions computed (round trips)
        ctx.sync()
        ctx.stats(reset=True)
        b = _outs(h)
        _step(ctx, h, b)                                  # second step: none
        ctx.sync()
        assert ctx.stats(reset=True)["host_syncs"] == 0
        for k in a:
            assert torch.equal(a[k], b[k]), k
        for i in range(len(h.layers)):
            assert b[f"S{i}"].cpu().tolist() == refs[i]["S"]
        assert b["Sand"].cpu().tolist() == ra["S"]
        assert b["gt"].cpu().tolist() == O.topk_closeness(ra["c"], h.K)
        assert b["cc2"].cpu().tolist() == O.cc2(rs, h.K)[0]
        r1, n1, _ = O.cc1(rs, h.K)
        assert int(b["n1"].item()) == n1 and b["cc1"].cpu().tolist()[:min(h.K, n1)] == r1
        c = _outs(h)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=ctx.stream):
            _step(ctx, h, c)
        for k in c:
            c[k].zero_()
        torch.cuda.synchronize()
        with torch.cuda.stream(ctx.stream):
            graph.replay()
            graph.replay()
        torch.cuda.synchronize()
        for k in a:
            assert torch.equal(a[k], c[k]), k
