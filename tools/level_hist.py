"""dev tool: per-level time histogram of the MS-BFS launch (bfs_dbg=2) for one graph of a config."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse
import numpy as np
from paper_2207_11662_b200 import Context
from synth import build_config

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--graph", default="0")
ap.add_argument("--set", action="append", default=[], help="name=value library parameter")
ap.add_argument("--level", type=int, default=0, help="profile only this BFS level (HM_MSBFS_PROF builds)")
a = ap.parse_args()
h = build_config(a.config)
with Context(0) as ctx:
    for kv in a.set:
        k, v = kv.split("=")
        ctx.set_param(k, int(v))
    ctx.set_param("timing", 1)
    ctx.load_layers(h.V, h.layers)
    if a.graph == "layers":                    # the layers' Psi as the step runs it (fused when unpruned)
        gl = list(range(len(h.layers)))
        run = lambda: ctx.closeness_multi(gl)
    else:
        g = ctx.and_aggregate(list(h.subsets[0])) if a.graph == "and" else int(a.graph)
        run = lambda: ctx.closeness(g, out={})
    run()
    ctx.sync(); ctx.stats(reset=True)
    ctx.set_param("bfs_dbg", 2 | (a.level << 8))
    run()
    ctx.sync()
    st = ctx.stats()
    dc = ctx.debug_counts().astype(np.int64)
cnt = dc[:4096]; ns = dc[4096:8192]
L = int(np.nonzero(cnt)[0].max()) + 1
print(f"graph {a.graph} {' '.join(a.set)}: {st['bfs_ms']:.2f} ms (dbg run), levels {int(cnt.sum())}, batches {int(cnt[1])}")
tot = ns.sum()
for d in range(1, L):
    if cnt[d]:
        print(f"  d={d:3d} batches={cnt[d]:4d} mean_us={ns[d]/cnt[d]/1e3:8.1f} share={100*ns[d]/tot:5.1f}%")
ph = dc[8192:8200].astype(np.float64)
if ph.sum() > 0:
    names = ["prologue+stage", "heavy", "claim+meta+publish", "scan", "seg+sort", "rounds", "step end", "grid wait"]
    print("  warp-cycle share by phase (HM_MSBFS_PROF build):")
    for n_, v_ in zip(names, ph):
        print(f"    {n_:<20} {100 * v_ / ph.sum():5.1f}%")
if ph.sum() > 0:
    nwarps = 148 * 32
    rounds, iters = float(dc[8200]), float(dc[8201])
    print(f"  per warp: rounds {rounds / nwarps:.0f}, gather iterations {iters / nwarps:.0f}; "
          f"cycles per round {ph[5] / max(rounds, 1):.0f}, "
          f"per level-step per warp {ph.sum() / nwarps / max(cnt[a.level] if a.level else cnt.sum(), 1):.0f}")
    if dc[8204]:
        print(f"  per CTA-level: first warp leaves the unit loop at {dc[8202] / dc[8204]:.0f} cycles, "
              f"last at {dc[8203] / dc[8204]:.0f} cycles ({dc[8204]} CTA-levels)")
