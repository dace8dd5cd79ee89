"""ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU definition of what the B200 path computes
for arXiv 2207.11662 (*Closeness Centrality Detection in Homogeneous
Multilayer Networks*).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this module.  It shares no code with ``paper_2207_11662_b200/``: plain Python
sets, lists, ``math.fsum`` and ``sorted``; per-source BFS in
``oracle/bfs_oracle.c`` (plain queue BFS, one per source).

Floating point: every closeness value and ratio is a Python float (IEEE
binary64, round-to-nearest-even), evaluated in the order written below.

Readings of silent / ambiguous passages are the SURVEY.md §8(c) ledger (Z1-Z21),
listed in DESIGN.md §3.  Each function names the passage it follows.

Pinned by tests/test_oracle_*.py against: Floyd-Warshall brute force, closed
forms (path, star, cycle, complete, complete bipartite), networkx
``closeness_centrality`` (the paper's own tool), the paper's CC2
worked example, a hand-executed CC1 instance (SPEC.md:222,
tests/golden/cc1_six_vertex.json), and invariants.  Every function below is
pinned; none is "parity unpinned".
"""
import math
from collections import deque

import numpy as np

from . import _bfs


# ---------------------------------------------------------------------------
# graphs
# ---------------------------------------------------------------------------
def canonical_edges(V, pairs):
    """Canonical simple undirected edge set of one layer.

    PAPER.md:55 (§1): a HoMLN is G_1(V,E_1)...G_l(V,E_l) over one vertex set;
    PAPER.md:186: undirected graphs.  Self-loops dropped, (u,v) -> (min,max),
    duplicates removed; all V vertices kept, isolated ones included
    (Z16).  Raises ValueError on an id outside [0, V).
    """
    E = set()
    for u, v in pairs:
        u = int(u)
        v = int(v)
        if not (0 <= u < V and 0 <= v < V):
            raise ValueError(f"vertex id out of range: ({u},{v}) with V={V}")
        if u == v:
            continue
        E.add((u, v) if u < v else (v, u))
    return E


def adjacency(V, E):
    """One-hop neighbourhoods NBD(u), as sorted lists."""
    adj = [[] for _ in range(V)]
    for u, v in E:
        adj[u].append(v)
        adj[v].append(u)
    for a in adj:
        a.sort()
    return adj


def degrees(V, E):
    """deg(u) = |NBD(u)|."""
    d = [0] * V
    for u, v in E:
        d[u] += 1
        d[v] += 1
    return d


def and_aggregate(edge_sets):
    """Boolean AND aggregation (PAPER.md:150 §3.1; :205 §4 GT step i): an edge
    is present iff it is present in every chosen layer.  Vertex set unchanged."""
    it = iter(edge_sets)
    out = set(next(it))
    for E in it:
        out &= E
    return out


def or_aggregate(edge_sets):
    """Boolean OR aggregation (§3.1): present in at least one layer."""
    out = set()
    for E in edge_sets:
        out |= E
    return out


# ---------------------------------------------------------------------------
# Psi: all-sources BFS distance sums (§4)
# ---------------------------------------------------------------------------
def bfs_python(V, adj, s):
    """One plain queue BFS from s.  Returns (S(s), k(s)):
    S = sum of d(s,w) over reachable w; k = reachable count incl. s."""
    dist = {s: 0}
    q = deque([s])
    while q:
        x = q.popleft()
        for y in adj[x]:
            if y not in dist:
                dist[y] = dist[x] + 1
                q.append(y)
    return sum(dist.values()), len(dist)


def bfs_sums(V, E, sources=None, threads=0, use_c=True):
    """S(s), k(s) for every source (default: all V).  PAPER.md:209.

    ``use_c`` runs the same plain BFS in oracle/bfs_oracle.c (threads over
    sources); ``use_c=False`` runs ``bfs_python``.  Returns (S uint64[n],
    k int32[n]) numpy arrays in source order."""
    if sources is None:
        sources = range(V)
    sources = np.asarray(list(sources) if not isinstance(sources, np.ndarray) else sources,
                         dtype=np.int32)
    if not use_c:
        adj = adjacency(V, E)
        S = np.zeros(len(sources), np.uint64)
        k = np.zeros(len(sources), np.int32)
        for i, s in enumerate(sources):
            S[i], k[i] = bfs_python(V, adj, int(s))
        return S, k
    return _bfs.bfs_sources(V, E, sources, threads)


def closeness_wf(V, S, k):
    """Wasserman-Faust closeness, as the paper's tool computes it.

    PAPER.md:183 (Eq. 1) CC(u) = (n-1)/sum_v d(u,v); for
    disconnected graphs "a distance of 0 is assumed" for unreachable nodes and
    scores are "normalized using Wasserman and Faust" (reading Z1: the exact
    NetworkX wf_improved formula).  In binary64, in this order:
        t1 = (k-1)/S ; t2 = (k-1)/(V-1) ; c = t1*t2
    c = 0 when S == 0 or V <= 1 (Z17).  For k == V this equals Eq. 1 exactly.
    """
    out = []
    for Su, ku in zip(S, k):
        Su = int(Su)
        ku = int(ku)
        if Su > 0 and V > 1:
            t1 = (ku - 1.0) / float(Su)
            t2 = (ku - 1.0) / float(V - 1)
            out.append(t1 * t2)
        else:
            out.append(0.0)
    return out


def pen_sum(V, S, k):
    """n-penalty distance sum sumDist(u) (§5.1): an unreachable
    v contributes dist(u,v) = n.  pen = S + (V - k) * V  (integer)."""
    return [int(Su) + (V - int(ku)) * V for Su, ku in zip(S, k)]


def mean_fsum(xs):
    """Mean as the correctly-rounded exact sum divided by the count (Z6):
    math.fsum(xs) / len(xs) -- one rounding for the sum, one IEEE division."""
    n = len(xs)
    return math.fsum(xs) / n if n else 0.0


def cc_nodes(c):
    """CC nodes: "closeness centrality score higher than the average"
    (PAPER.md:186 §4; :155 "greater than average").  Strict > (Z4); mean over
    all V vertices, isolated ones included at 0 (Z5)."""
    mu = mean_fsum(c)
    return {u for u, x in enumerate(c) if x > mu}, mu


def analyze(V, E, threads=0, use_c=True):
    """Psi on one graph (PAPER.md:121-122 §3; :431 retained data).  Returns a
    dict with S, k, c, pen, deg, adj, mu, CH (all plain Python containers)."""
    S, k = bfs_sums(V, E, threads=threads, use_c=use_c)
    S = [int(x) for x in S]
    k = [int(x) for x in k]
    c = closeness_wf(V, S, k)
    CH, mu = cc_nodes(c)
    return {
        "V": V, "E": E, "S": S, "k": k, "c": c, "pen": pen_sum(V, S, k),
        "deg": degrees(V, E), "adj": adjacency(V, E), "mu": mu, "CH": CH,
    }


# ---------------------------------------------------------------------------
# ground truth and composition (Theta)
# ---------------------------------------------------------------------------
def topk_closeness(c, K):
    """Ground-truth ranking: top-K by closeness descending,
    lower vertex id first on ties (Z14)."""
    return sorted(range(len(c)), key=lambda u: (-c[u], u))[:K]


def cc2(results, K):
    """Heuristic CC2, Alg. 1.

    estSumDist(u) = max over the chosen layers of sumDist_i(u) (the n-penalty
    sum, Z3); CC value by Eq. 1 on estSumDist; "take the top-k CC nodes"
    (PAPER.md:593).  (V-1)/est is strictly decreasing in est, so top-K by
    Eq. 1 = the K smallest (est, id) pairs (Z14).  r-ary max (Z12).
    Returns (topK ids, est list)."""
    V = results[0]["V"]
    est = [max(r["pen"][u] for r in results) for u in range(V)]
    return sorted(range(V), key=lambda u: (est[u], u))[:K], est


def cc2_above_average(results):
    """CC2 with the "above-average" selection: scores by Eq. 1,
    (n-1)/estSumDist, CC nodes = strictly above the fsum mean (Z4-Z6)."""
    V = results[0]["V"]
    _, est = cc2(results, 1)
    score = [(V - 1.0) / float(e) if e > 0 else 0.0 for e in est]
    mu = mean_fsum(score)
    return {u for u in range(V) if score[u] > mu}


def degdist_ratios(results):
    """Eq. 2: degDistRatio_i(u) = sumDist_i(u) / min_j deg_j(u),
    one IEEE division; +inf when the min degree is 0 (Z8).  Flat r-ary (Z12).
    Returns (mindeg, ratios per layer)."""
    V = results[0]["V"]
    mindeg = [min(r["deg"][u] for r in results) for u in range(V)]
    ratios = []
    for r in results:
        ratios.append([float(r["pen"][u]) / float(mindeg[u]) if mindeg[u] >= 1 else math.inf
                       for u in range(V)])
    return mindeg, ratios


def cc1(results, K):
    """Heuristic CC1 (Eq. 2, Eq. 3; pseudocode PAPER.md:477-507
    and the companion appendix :1222-1252), flat r-ary (Z12):

      ratio_i(u) = pen_i(u) / mindeg(u)                    (Eq. 2; Z8)
      avg_i      = fsum of finite ratio_i / their count      (line 483-484; Z6)
      avgAND     = max_i avg_i                               (Eq. 3)
      cand_i(u)  = {v in NBD_i(u) : ratio_i(v) < avgAND}     (lines 486-501; Z7, Z11)
      for u in  CH_1 ∩ ... ∩ CH_r :                          (line 502)
          I = ∩_i cand_i(u); if |I| > 1: R |= I              (lines 503-505; Z9)
          R |= {u}                                           (line 506; Z10)

    Ranking (Z13): by RN(est(u)/mindeg(u)) ascending, id ascending, where
    est = max_i pen_i.  Returns (ranked[:K], |R|, R)."""
    V = results[0]["V"]
    mindeg, ratios = degdist_ratios(results)
    avgs = []
    for rat in ratios:
        finite = [x for x in rat if x != math.inf]
        avgs.append(math.fsum(finite) / len(finite) if finite else 0.0)
    avg_and = max(avgs)
    common = set(results[0]["CH"])
    for r in results[1:]:
        common &= r["CH"]
    R = set()
    for u in sorted(common):
        I = None
        for r, rat in zip(results, ratios):
            cand = {v for v in r["adj"][u] if rat[v] < avg_and}
            I = cand if I is None else (I & cand)
        if len(I) > 1:
            R |= I
        R.add(u)
    est = [max(r["pen"][u] for r in results) for u in range(V)]
    ranked = sorted(R, key=lambda u: (float(est[u]) / float(mindeg[u]), u))
    return ranked[:K], len(R), R


def naive(results, K):
    """Naive composition: intersection of the layers' CC-node
    sets.  Ranked by vertex id; returns (first K ids, |set|, set)."""
    common = set(results[0]["CH"])
    for r in results[1:]:
        common &= r["CH"]
    s = sorted(common)
    return s[:K], len(s), common


# ---------------------------------------------------------------------------
# evaluation (§5)
# ---------------------------------------------------------------------------
def jaccard(a, b):
    """|a ∩ b| / |a ∪ b|; both empty -> 1.0."""
    a, b = set(a), set(b)
    if not a and not b:
        return 1.0
    return len(a & b) / len(a | b)


def prf1(est, gt):
    """precision, recall, F1 (empty-set conventions SPEC.md:379)."""
    est, gt = set(est), set(gt)
    tp = len(est & gt)
    if est:
        p = tp / len(est)
    else:
        p = 1.0 if not gt else 0.0
    r = tp / len(gt) if gt else 1.0
    f = 2 * p * r / (p + r) if (p + r) > 0 else 0.0
    return p, r, f
