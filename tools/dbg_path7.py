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
    n2o = dc[139264:139264 + 65536].view(np.int32)[:n]
    nrp = dc[139264 + 65536:139264 + 2 * 65536].view(np.int32)[:n]
    k2 = dc[139264 + 2 * 65536:139264 + 3 * 65536][:n]
    bad = np.nonzero(n2o != np.arange(n))[0]
    print("rep", rep, "mism", int((S != ref).sum()), "n2o non-identity at", bad[:10].tolist(), n2o[bad[:10]].tolist(),
          "keys", [hex(int(x)) for x in k2[bad[:4]]], "nrp tail", nrp[-4:].tolist(), flush=True)
