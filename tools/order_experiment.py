"""dev experiment: does a locality-preserving vertex order (BFS / reverse Cuthill-McKee) speed up the
MS-BFS?  Loads a C5 graph (layer 0 or the AND of all layers) as a single layer under several vertex
relabellings and times hm_closeness (MS-BFS ms per launch)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee, breadth_first_order, connected_components
from synth import build_config
from paper_2207_11662_b200 import Context

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
h = build_config(name)
V = h.V
keys = [set((L[:, 0].astype(np.int64) * V + L[:, 1]).tolist()) for L in h.layers]
A = set.intersection(*keys)
Akeys = np.array(sorted(A), dtype=np.int64)
graphs = {"and": np.stack([Akeys // V, Akeys % V], 1).astype(np.int32), "L0": h.layers[0]}


def perms(E):
    M = sp.coo_matrix((np.ones(len(E)), (E[:, 0], E[:, 1])), shape=(V, V)).tocsr()
    M = M + M.T
    out = {"orig": np.arange(V)}
    r = reverse_cuthill_mckee(M, symmetric_mode=True)          # r[i] = old id at new position i
    p = np.empty(V, np.int64); p[r] = np.arange(V); out["rcm"] = p
    nc, lab = connected_components(M, directed=False)
    big = np.bincount(lab).argmax()
    root = int(np.nonzero(lab == big)[0][0])
    order = breadth_first_order(M, root, directed=False, return_predecessors=False)
    rest = np.setdiff1d(np.arange(V), order)
    full = np.concatenate([order, rest])
    p = np.empty(V, np.int64); p[full] = np.arange(V); out["bfs"] = p
    rng = np.random.default_rng(0)
    out["random"] = rng.permutation(V)
    return out


with Context(0) as ctx:
    ctx.set_param("timing", 1)
    for gname, E in graphs.items():
        for pname, p in perms(E).items():
            Ep = np.sort(p[E.astype(np.int64)], axis=1).astype(np.int32)
            ctx.load_layers(V, [Ep])
            ctx.closeness(0, out={}); ctx.sync(); ctx.stats(reset=True)
            for _ in range(2):
                ctx.closeness(0, out={})
            ctx.sync()
            st = ctx.stats()
            print(f"{name} {gname} order={pname}: {st['bfs_ms'] / st['bfs_launches']:.2f} ms/launch, "
                  f"levels/launch {st['bfs_levels'] / st['bfs_launches']:.0f}", flush=True)
