import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context
n = 1024
E = np.array([[i, i + 1] for i in range(n - 1)], np.int32)
for words in (32, 16):
  with Context(0) as ctx:
    ctx.set_param("bfs_dbg", 2); ctx.set_param("bfs_words", words); ctx.set_param("bfs_blocks_per_sm", 1)
    ctx.load_layers(n, [E])
    rp, col = ctx.graph_csr(0)
    print("csr ok:", rp[:4].tolist(), rp[-4:].tolist(), col[-6:].tolist())
    S = ctx.closeness(0)["S"]
    dc = ctx.debug_counts()
    st = ctx.stats()
  print("words", words, "levels", st["bfs_levels"], "batches", st["bfs_batches"])
  print("level counts 1..12:", dc[1:13].tolist())
  rows = dc[8192:8192 + n]
  for v in list(range(0, 4)) + list(range(1012, 1024)):
    print(v, format(int(rows[v]) & ((1 << 20) - 1), '020b')[::-1], int(S[v]))
