"""Synthetic HoMLN recipes (BASELINE.json ``configs``; readings in SURVEY.md §8(d)).

Every recipe is a deterministic function of its seed.  Edge draws follow one
rule: candidates come from a counter-based stream in order; a candidate is
accepted iff it is not a self-loop, not a duplicate of an earlier accepted
edge, and not in a forbidden set; drawing stops at the target count.  The
chunked numpy implementation below is equivalent to that sequential rule for
any chunk size.

Edges are returned canonical, as int32 arrays of shape (m, 2) with u < v.
"""
from dataclasses import dataclass, field
import numpy as np

from .prng import Stream, stream_key

RMAT_ABCD = (0.57, 0.19, 0.19, 0.05)


# --------------------------------------------------------------------------
# candidate generators: each returns (u, v) int64 arrays of length n
# --------------------------------------------------------------------------
def er_candidates(stream: Stream, V: int):
    def f(n):
        u = stream.next_below(n, V)
        v = stream.next_below(n, V)
        return u, v
    return f


def rmat_candidates(stream: Stream, V: int, perm=None, abcd=RMAT_ABCD):
    """Recursive-quadrant R-MAT on a 2^s domain (s = ceil(log2 V)), bits MSB
    first; ids >= V are rejected as self-loops would be (mapped to u == v)."""
    s = max(1, int(np.ceil(np.log2(V))))
    a, b, c, _ = abcd

    def f(n):
        r = stream.next_uniform(n * s).reshape(n, s)
        bu = (r >= a + b).astype(np.int64)                       # quadrants c, d
        bv = (((r >= a) & (r < a + b)) | (r >= a + b + c)).astype(np.int64)  # b, d
        w = (np.int64(1) << np.arange(s - 1, -1, -1, dtype=np.int64))
        u = (bu * w).sum(axis=1)
        v = (bv * w).sum(axis=1)
        bad = (u >= V) | (v >= V)
        u[bad] = 0
        v[bad] = 0
        if perm is not None:
            u = perm[u]
            v = perm[v]
            v[bad] = u[bad]
        return u, v
    return f


def sbm_candidates(stream: Stream, V: int, n_comm: int, in_over_out: float):
    """Planted partition: community(v) = v // (V // n_comm) (contiguous);
    intra-pair probability = in_over_out x inter-pair probability."""
    csz = V // n_comm
    assert csz * n_comm == V
    intra_pairs = n_comm * csz * (csz - 1) // 2
    inter_pairs = V * (V - 1) // 2 - intra_pairs
    f_intra = in_over_out * intra_pairs / (in_over_out * intra_pairs + inter_pairs)

    def f(n):
        u = stream.next_below(n, V)
        pick = stream.next_uniform(n)
        r_in = stream.next_below(n, csz)
        r_out = stream.next_below(n, V - csz)
        cu = u // csz
        v_in = cu * csz + r_in
        v_out = np.where(r_out < cu * csz, r_out, r_out + csz)
        v = np.where(pick < f_intra, v_in, v_out)
        return u, v
    f.f_intra = f_intra
    return f


def _keys(u, v, V):
    a = np.minimum(u, v)
    b = np.maximum(u, v)
    return a * np.int64(V) + b


def draw_unique_edges(V: int, m: int, cand, forbidden=None, chunk=None):
    """First m accepted candidates (see module docstring).  Returns sorted-by-
    draw-order canonical keys (int64, u*V+v with u<v)."""
    if m <= 0:
        return np.zeros(0, dtype=np.int64)
    forb = np.zeros(0, np.int64) if forbidden is None else np.asarray(forbidden, np.int64)
    forb = np.unique(forb)
    chunk = chunk or max(1024, int(m * 1.15) + 64)
    out = []
    seen = np.zeros(0, dtype=np.int64)
    need = m
    while need > 0:
        u, v = cand(chunk)
        ok = u != v
        k = _keys(u[ok], v[ok], V)
        _, first = np.unique(k, return_index=True)
        first.sort()
        k = k[first]
        keep = ~np.isin(k, seen, assume_unique=True) & ~np.isin(k, forb, assume_unique=True)
        k = k[keep][:need]
        out.append(k)
        seen = np.union1d(seen, k)
        need -= len(k)
        chunk = max(1024, int(need * 1.3) + 64)
    return np.concatenate(out)


def keep_bernoulli(stream: Stream, keys: np.ndarray, p: float):
    """One Bernoulli(p) draw per base edge, in base order."""
    r = stream.next_uniform(len(keys))
    return keys[r < p]


def keys_to_pairs(keys, V):
    keys = np.asarray(keys, dtype=np.int64)
    return np.stack([keys // V, keys % V], axis=1).astype(np.int32)


@dataclass
class HoMLN:
    name: str
    V: int
    layers: list                       # list of int32 (m_i, 2) arrays, canonical u<v
    subsets: list                      # list of tuples of layer indices (r >= 2)
    K: int
    seed: int
    recipe: str = ""
    meta: dict = field(default_factory=dict)


def random_graph(V: int, m: int, seed: int, kind: str = "er"):
    """A single seeded simple graph (for tests): kind in {er, rmat}."""
    st = Stream(stream_key(seed, 0, "graph"))
    m = min(m, V * (V - 1) // 2)
    if kind == "er":
        cand = er_candidates(st, V)
    else:
        cand = rmat_candidates(st, V)
    return keys_to_pairs(draw_unique_edges(V, m, cand), V)


# --------------------------------------------------------------------------
# the five BASELINE configs (optionally scaled down in V, same avg degrees)
# --------------------------------------------------------------------------
CONFIG_NAMES = ("C1", "C2", "C3", "C4", "C5")
FULL_V = {"C1": 1000, "C2": 16384, "C3": 65536, "C4": 131072, "C5": 262144}
FULL_K = {"C1": 10, "C2": 50, "C3": 100, "C4": 200, "C5": 500}


def _layered(name, V, seed, base_keys, keep_ps, pad, K, subsets, recipe):
    layers = []
    for i, p in enumerate(keep_ps):
        kept = keep_bernoulli(Stream(stream_key(seed, i, "keep")), base_keys, p)
        n_add, cand_fn = pad(i, len(kept))
        add = draw_unique_edges(V, n_add, cand_fn(Stream(stream_key(seed, i, "unique"))),
                                forbidden=base_keys)
        layers.append(keys_to_pairs(np.concatenate([kept, add]), V))
    return HoMLN(name, V, layers, subsets, K, seed, recipe)


def build_config(name: str, V: int = None, K: int = None) -> HoMLN:
    """Build config ``name`` (C1..C5).  ``V`` scales the vertex count keeping
    every average degree (parity tests use small V; bench uses the full V)."""
    full = V is None or V == FULL_V[name]
    V = FULL_V[name] if V is None else int(V)
    K = (FULL_K[name] if K is None else K)
    K = min(K, V)
    seed = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5}[name]
    sfx = "" if full else f"@V={V}"

    if name == "C1":
        base = draw_unique_edges(V, 4 * V, er_candidates(Stream(stream_key(seed, 0, "base")), V))
        return _layered(
            "C1" + sfx, V, seed, base, (0.7, 0.7),
            lambda i, kept: (V, lambda st: er_candidates(st, V)),
            K, [(0, 1)],
            "ER base avg deg 8; keep w.p. 0.7 + V unique ER edges per layer")

    if name == "C2":
        perm = np.argsort(Stream(stream_key(seed, 0, "perm")).next_uniform(V), kind="stable")
        m = 8 * V
        base = draw_unique_edges(V, m, rmat_candidates(Stream(stream_key(seed, 0, "base")), V, perm))
        return _layered(
            "C2" + sfx, V, seed, base, (0.6, 0.6, 0.6),
            lambda i, kept: (int(round(0.2 * m)), lambda st: rmat_candidates(st, V, perm)),
            K, [(0, 1, 2)],
            "R-MAT base m=8V; keep 0.6 + round(0.2 m) unique R-MAT per layer")

    if name == "C3":
        perm = np.argsort(Stream(stream_key(seed, 0, "perm")).next_uniform(V), kind="stable")
        m = 8 * V
        base = draw_unique_edges(V, m, rmat_candidates(Stream(stream_key(seed, 0, "base")), V, perm))

        def pad(i, kept):
            if i < 2:
                return m - kept, (lambda st: rmat_candidates(st, V, perm))
            return m - kept, (lambda st: er_candidates(st, V))
        subs = [(a, b) for a in range(4) for b in range(a + 1, 4)]
        subs += [(a, b, c) for a in range(4) for b in range(a + 1, 4) for c in range(b + 1, 4)]
        return _layered("C3" + sfx, V, seed, base, (0.5,) * 4, pad, K, subs,
                        "R-MAT base avg deg 16; keep 0.5; pad to m: R-MAT (L1-2), ER (L3-4)")

    if name == "C4":
        perm = np.argsort(Stream(stream_key(seed, 0, "perm")).next_uniform(V), kind="stable")
        m = 6 * V
        base = draw_unique_edges(V, m, rmat_candidates(Stream(stream_key(seed, 0, "base")), V, perm))
        return _layered("C4" + sfx, V, seed, base, (0.9, 0.8, 0.6, 0.5, 0.4),
                        lambda i, kept: (m - kept, lambda st: er_candidates(st, V)),
                        K, [(0, 1, 2, 3, 4)],
                        "R-MAT base avg deg 12; keep .9/.8/.6/.5/.4; pad with unique ER to m")

    if name == "C5":
        n_comm = 64 if V % 64 == 0 else 1
        m = 4 * V
        base = draw_unique_edges(V, m, sbm_candidates(Stream(stream_key(seed, 0, "base")), V, n_comm, 10.0))
        return _layered("C5" + sfx, V, seed, base, (0.7, 0.7, 0.7),
                        lambda i, kept: (V, lambda st: er_candidates(st, V)),
                        K, [(0, 1, 2)],
                        "SBM base avg deg 8, 64 contiguous communities, p_in=10 p_out; "
                        "keep 0.7 + V unique ER edges per layer")
    raise ValueError(name)
