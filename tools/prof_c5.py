"""profiling driver: C5 layer-0 closeness, run twice (2nd launch is the one to capture)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context
from synth import build_config
import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--words", type=int, default=16)
ap.add_argument("--graph", default="0")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
h = build_config(a.config)
with Context(0) as ctx:
    ctx.set_param("bfs_words", a.words)
    ctx.set_param("timing", 1)
    ctx.load_layers(h.V, h.layers)
    g = ctx.and_aggregate(list(h.subsets[0])) if a.graph == "and" else int(a.graph)
    for r in range(a.reps):
        ctx.closeness(g, out={})
    ctx.sync()
    st = ctx.stats()
    print("bfs ms per launch", st["bfs_ms"] / st["bfs_launches"], "levels/launch", st["bfs_levels"] / st["bfs_launches"],
          "batches/launch", st["bfs_batches"] / st["bfs_launches"])
