import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context
for n in (1500, 1100, 1025, 1024):
    E = np.array([[i, i + 1] for i in range(n - 1)], np.int32)
    with Context(0) as ctx:
        ctx.set_param("bfs_dbg", 2); ctx.set_param("bfs_words", 32); ctx.set_param("bfs_blocks_per_sm", 1)
        ctx.load_layers(n, [E])
        S = ctx.closeness(0)["S"]
        dc = ctx.debug_counts()
    rows = dc[8192:8192 + n]
    miss1 = np.nonzero((rows & np.uint64(2)) == 0)[0]
    print(n, "rows not changed at level 1:", miss1[:40].tolist(), "count", len(miss1), flush=True)
    miss2 = np.nonzero((rows & np.uint64(4)) == 0)[0]
    print(n, "rows not changed at level 2:", miss2[:40].tolist(), "count", len(miss2), flush=True)
