import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context
from oracle import oracle as O
n = 1500
E = np.array([[i, i + 1] for i in range(n - 1)], np.int32)
ref = O.bfs_sums(n, set(map(tuple, E.tolist())))[0].astype(np.int64)
for rep in range(6):
    with Context(0) as ctx:
        ctx.set_param("bfs_dbg", 2); ctx.set_param("bfs_words", 32); ctx.set_param("bfs_blocks_per_sm", 1)
        ctx.load_layers(n, [E])
        S = ctx.closeness(0)["S"].astype(np.int64)
        dc = ctx.debug_counts()
    rows = dc[8192:8192 + n]
    miss1 = np.nonzero((rows & np.uint64(2)) == 0)[0]
    info = dc[73728:73728 + n].astype(np.uint64)
    print("rep", rep, "mism", int((S != ref).sum()), "miss@1", miss1[:6].tolist())
    for v in list(miss1[:6]) + [0, 1, 1498]:
        x = int(info[v])
        print("   row", v, "seen", x & 1, "have", (x >> 1) & 1, "nm", (x >> 8) & 0xff, "deg", (x >> 16) & 0xff,
              "acc", (x >> 24) & 0xffff, "Fc_own", (x >> 40) & 0xff, "blk", x >> 48)
