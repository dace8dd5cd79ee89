import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context
from oracle import oracle as O
order = [int(x) for x in sys.argv[1:]] or [1500, 1100, 1025, 1024, 1024, 1024, 700, 1500]
for n in order:
    E = np.array([[i, i + 1] for i in range(n - 1)], np.int32)
    ref = O.bfs_sums(n, set(map(tuple, E.tolist())))[0].astype(np.int64)
    with Context(0) as ctx:
        ctx.set_param("bfs_dbg", 2); ctx.set_param("bfs_words", 32); ctx.set_param("bfs_blocks_per_sm", 1)
        ctx.load_layers(n, [E])
        S = ctx.closeness(0)["S"].astype(np.int64)
        dc = ctx.debug_counts()
    rows = dc[8192:8192 + n]
    miss1 = np.nonzero((rows & np.uint64(2)) == 0)[0]
    print(n, "mism", int((S != ref).sum()), "hi", dc[6000:6003].tolist(), "scal", dc[6100:6104].tolist(),
          "miss@1", miss1[:10].tolist(), flush=True)
