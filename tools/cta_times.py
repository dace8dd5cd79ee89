import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context
from synth import build_config
h = build_config("C5")
words = int(sys.argv[1]) if len(sys.argv) > 1 else 16
with Context(0) as ctx:
    ctx.set_param("bfs_words", words)
    ctx.load_layers(h.V, h.layers)
    ctx.closeness(0, out={})
    ctx.set_param("bfs_dbg", 2)
    ctx.closeness(0, out={})
    dc = ctx.debug_counts(8192 + 64 * 512).astype(np.int64)
work = dc[8192:8192 + 32 * 512].reshape(32, 512)[:, :296]
start = dc[8192 + 32 * 512:8192 + 64 * 512].reshape(32, 512)[:, :296]
for d in range(1, 14):
    w = work[d] / 1e3; s = (start[d] - start[d].min()) / 1e3
    if w.max() == 0: continue
    print(f"W={words} level {d:2d}: CTA work us min {w.min():6.1f} med {np.median(w):6.1f} p90 {np.percentile(w,90):6.1f} max {w.max():6.1f} | start skew max {s.max():5.1f}us | slowest CTAs {np.argsort(-w)[:4].tolist()}")
