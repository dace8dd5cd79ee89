import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context
from oracle import oracle as O
n = 1500
E = np.array([[i, i + 1] for i in range(n - 1)], np.int32)
ref = O.bfs_sums(n, set(map(tuple, E.tolist())))[0].astype(np.int64)
mode = sys.argv[1]
res = []
for rep in range(8):
    with Context(0, stream=(False if mode == "own" else None)) as ctx:
        ctx.set_param("bfs_words", 32); ctx.set_param("bfs_blocks_per_sm", 1)
        ctx.load_layers(n, [E])
        S = ctx.closeness(0)["S"].astype(np.int64)
    res.append(int((S != ref).sum()))
print(mode, os.environ.get("CUDA_LAUNCH_BLOCKING"), res, flush=True)
