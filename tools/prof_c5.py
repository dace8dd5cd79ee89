"""dev tool: MS-BFS time per launch on one graph of a config (second launch timed).

    python tools/prof_c5.py --config C5 --graph 0|and --set bfs_words=32 --set bfs_pipe=8
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import time
from paper_2207_11662_b200 import Context
from synth import build_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--graph", default="0")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--set", action="append", default=[], help="name=value library parameter")
a = ap.parse_args()
h = build_config(a.config)
with Context(0) as ctx:
    for kv in a.set:
        k, v = kv.split("=")
        ctx.set_param(k, int(v))
    ctx.set_param("timing", 1)
    ctx.load_layers(h.V, h.layers)
    g = ctx.and_aggregate(list(h.subsets[0])) if a.graph == "and" else int(a.graph)
    ctx.closeness(g, out={})
    ctx.sync()
    ctx.stats(reset=True)
    t0 = time.perf_counter()
    for r in range(a.reps - 1):
        ctx.closeness(g, out={})
    ctx.sync()
    call_ms = (time.perf_counter() - t0) * 1e3 / max(a.reps - 1, 1)
    st = ctx.stats()
    print(f"{a.config} graph {a.graph} {' '.join(a.set)}: {st['bfs_ms'] / st['bfs_launches']:.2f} ms/launch, "
          f"levels/launch {st['bfs_levels'] / st['bfs_launches']:.0f}, batches/launch {st['bfs_batches'] / st['bfs_launches']:.0f}, "
          f"whole closeness call {call_ms:.2f} ms",
          flush=True)
