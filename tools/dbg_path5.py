import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context
from oracle import oracle as O
n = 1500
E = np.array([[i, i + 1] for i in range(n - 1)], np.int32)
ref = O.bfs_sums(n, set(map(tuple, E.tolist())))[0].astype(np.int64)
for dbg in (2, 2 | 32, 2 | 32 | 8 | 16):
    res = []
    for rep in range(6):
        with Context(0) as ctx:
            ctx.set_param("bfs_dbg", dbg); ctx.set_param("bfs_words", 32); ctx.set_param("bfs_blocks_per_sm", 1)
            ctx.load_layers(n, [E])
            S = ctx.closeness(0)["S"].astype(np.int64)
            dc = ctx.debug_counts()
        rows = dc[8192:8192 + n]
        miss1 = np.nonzero((rows & np.uint64(2)) == 0)[0]
        res.append((int((S != ref).sum()), miss1[:4].tolist()))
    print("dbg", dbg, res, flush=True)
