import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context
from synth import build_config
h = build_config("C5")
for words in [int(x) for x in (sys.argv[1:] or ["16", "32"])]:
    with Context(0) as ctx:
        ctx.set_param("bfs_words", words)
        ctx.load_layers(h.V, h.layers)
        ctx.closeness(0, out={})
        for g in (0, "and"):
            gid = ctx.and_aggregate([0, 1, 2]) if g == "and" else 0
            ctx.set_param("bfs_dbg", 2)
            ctx.closeness(gid, out={})
            dc = ctx.debug_counts(8192).astype(np.int64)
            cnt, t = dc[:4096], dc[4096:8192]
            nz = np.nonzero(cnt)[0]
            print(f"W={words} graph={g}: total {t.sum()/1e6:.1f} ms; per level index: " +
                  " ".join(f"{d}:{t[d]/cnt[d]/1e3:.1f}us(x{cnt[d]})" for d in nz[:40]), flush=True)
            ctx.set_param("bfs_dbg", 0)
