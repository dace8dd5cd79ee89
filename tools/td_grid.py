"""dev experiment: direction switch (bfs_td) on high-diameter graphs, where a level's frontier is a thin
wave: a 2-D grid (diameter ~2 sqrt V) and a long cycle with chords.  MS-BFS ms per launch per setting."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context


def grid(n):
    idx = np.arange(n * n).reshape(n, n)
    e = np.concatenate([np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1),
                        np.stack([idx[:-1, :].ravel(), idx[1:, :].ravel()], 1)])
    return n * n, e.astype(np.int32)


def ring(V, chords, seed=0):
    rng = np.random.default_rng(seed)
    a = np.arange(V)
    e = [np.stack([a, (a + 1) % V], 1)]
    u = rng.integers(0, V, chords)
    e.append(np.stack([u, (u + rng.integers(2, 64, chords)) % V], 1))
    e = np.sort(np.concatenate(e), axis=1)
    return V, np.unique(e[e[:, 0] != e[:, 1]], axis=0).astype(np.int32)


cases = {"grid256": grid(256), "grid512": grid(512), "ring65k": ring(65536, 4096)}
for name, (V, E) in cases.items():
    for td in (0, 16, 64, 256, 1024):
        with Context(0) as ctx:
            ctx.set_param("bfs_td", td)
            ctx.set_param("timing", 1)
            ctx.load_layers(V, [E])
            r0 = ctx.closeness(0, out={})
            ctx.sync()
            ctx.stats(reset=True)
            ctx.closeness(0, out={})
            ctx.sync()
            st = ctx.stats(reset=True)
            print(f"{name} V={V} bfs_td={td}: {st['bfs_ms']:.2f} ms/launch, levels {st['bfs_levels']}, "
                  f"top-down levels {st['bfs_td_levels']}", flush=True)
