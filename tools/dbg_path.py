"""dev script: path parity + per-level change counts under debug settings"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context
from oracle import oracle as O

for n in (40, 100, 300, 700, 1500):
    E = np.array([[i, i + 1] for i in range(n - 1)], np.int32)
    ref = O.bfs_sums(n, set(map(tuple, E.tolist())))[0].astype(np.int64)
    words = 32
    B = 64 * words
    src = np.arange(min(B, n))
    exp = np.zeros(4096, np.int64)
    v = np.arange(n)
    D = np.abs(v[:, None] - src[None, :])
    for d in range(1, n):
        exp[d] = int((D == d).any(axis=1).sum())
    for bps in (1, 0):
        with Context(0) as ctx:
            ctx.set_param("bfs_dbg", 2); ctx.set_param("bfs_words", words); ctx.set_param("bfs_blocks_per_sm", bps)
            ctx.load_layers(n, [E])
            S = ctx.closeness(0)["S"].astype(np.int64)
            st = ctx.stats()
            dc = ctx.debug_counts().astype(np.int64)
        ch = dc[:4096]
        bad = np.nonzero(ch[1:n] != exp[1:n])[0]
        msg = ""
        if len(bad):
            d0 = int(bad[0] + 1)
            lo = max(1, d0 - 2)
            msg = f"first bad level {d0}: got {ch[lo:d0+3].tolist()} exp {exp[lo:d0+3].tolist()}"
            wrong = np.nonzero(S != ref)[0]
            msg += f" | wrong rows {wrong[:8].tolist()} S {S[wrong[:4]].tolist()} ref {ref[wrong[:4]].tolist()}"
        print(f"n={n} bps={bps} mism={(S!=ref).sum()} levels={st['bfs_levels']} {msg}", flush=True)
