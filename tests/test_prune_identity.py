"""CPU check of the identities the GPU's exact 2-core pruning relies on
(paper_2207_11662_b200/csrc/prune.cu):

  core u:    S(u) = sum_{core s} (1 + T(s)) d(s, u) + sum_{core c} A(c)      (1)
  peeled x:  S(x) = S(p(x)) + k - 2 size(x)                                 (2)

Peeling follows the kernel's rule (rounds; of two degree-1 ends of the last
edge only the larger id goes).  Distances come from a plain BFS written here;
the expected S is the oracle's.  Exactness of the pruned path
on the GPU itself is covered by the GPU parity tests (bfs_prune on and off)."""
import random
from collections import deque

from oracle import oracle as O


def bfs(adj, s, alive):
    d = {s: 0}
    q = deque([s])
    while q:
        u = q.popleft()
        for w in adj[u]:
            if alive[w] and w not in d:
                d[w] = d[u] + 1
                q.append(w)
    return d


def peel(V, adj, comp):
    """kernel rule on one component `comp` (a set); returns rem (round or 0), par, size, A"""
    rem = [0] * V
    par = [-1] * V
    size = [1] * V
    A = [0] * V
    degl = [len(adj[v]) for v in range(V)]
    r = 0
    while True:
        r += 1
        marked = []
        for v in sorted(comp):
            if rem[v] or degl[v] != 1:
                continue
            u = next(w for w in adj[v] if rem[w] == 0)
            if degl[u] == 1 and u > v:
                continue
            marked.append(v)
        if not marked:
            return rem, par, size, A, r - 1
        for v in marked:
            rem[v] = r
        for v in marked:
            u = next(w for w in adj[v] if rem[w] == 0)
            par[v] = u
            degl[u] -= 1
            size[u] += size[v]
            A[u] += A[v] + size[v]


def pruned_sums(V, E):
    adj = [[] for _ in range(V)]
    for u, v in E:
        adj[u].append(v)
        adj[v].append(u)
    seen, comps = set(), []
    for s in range(V):
        if s not in seen and adj[s]:
            c = set(bfs(adj, s, [True] * V))
            seen |= c
            comps.append(c)
    S = [0] * V
    for comp in comps:
        k = len(comp)
        rem, par, size, A, R = peel(V, adj, comp)
        alive = [rem[v] == 0 for v in range(V)]
        core = [v for v in comp if alive[v]]
        C = sum(A[c] for c in core)
        for u in core:                                           # (1)
            d = bfs(adj, u, alive)
            S[u] = sum((1 + size[s] - 1) * d[s] for s in core) + C
        for rr in range(R, 0, -1):                               # (2), top-down
            for x in comp:
                if rem[x] == rr:
                    S[x] = S[par[x]] + k - 2 * size[x]
    return S


def test_pruning_identities_random_graphs():
    rng = random.Random(11)
    for t in range(60):
        V = rng.randint(3, 60)
        E = set()
        for v in range(1, V):                 # random tree ...
            if rng.random() < 0.9:
                u = rng.randrange(v)
                E.add((u, v))
        for _ in range(rng.randint(0, V // 3)):   # ... plus a few cycle-closing edges
            u, v = rng.sample(range(V), 2)
            E.add((min(u, v), max(u, v)))
        assert pruned_sums(V, E) == O.analyze(V, E)["S"], t


def test_pruning_identities_special_shapes():
    cases = [
        (2, {(0, 1)}),                                                     # K2: last edge kept
        (4, {(0, 1), (1, 2), (2, 3)}),                                     # bicentral path
        (7, {(0, i) for i in range(1, 7)}),                                # star
        (9, {(i, (i + 1) % 5) for i in range(5)} | {(0, 5), (5, 6), (6, 7), (2, 8)}),   # cycle + trees
    ]
    for V, E in cases:
        assert pruned_sums(V, E) == O.analyze(V, E)["S"], (V, E)
