import sys, os, random
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2207_11662_b200 import Context
from oracle import oracle as O
from synth import random_graph
rng = random.Random(2022)
for t in range(40):
    V = rng.choice([5, 33, 64, 65, 200, 513, 1000, 2500])
    m = rng.choice([0, V // 4, V // 2, V, 2 * V, 4 * V])
    kind = rng.choice(["er", "rmat"])
    E = random_graph(V, m, seed=1000 + t, kind=kind)
    Es = set(map(tuple, E.tolist()))
    ref = O.bfs_sums(V, Es)[0].astype(np.int64)
    deg = np.bincount(E.ravel(), minlength=V) if len(E) else np.zeros(V, int)
    out = []
    for words in (8, 16, 32):
        for heavy in (100000, 256, 4):
            with Context(0) as ctx:
                ctx.set_param("bfs_words", words); ctx.set_param("bfs_heavy", heavy)
                ctx.load_layers(V, [E])
                S = ctx.closeness(0)["S"].astype(np.int64)
            bad = np.nonzero(S != ref)[0]
            out.append(f"w{words}h{heavy}:{len(bad)}")
    print(t, V, m, kind, "maxdeg", int(deg.max()) if V else 0, " ".join(out), flush=True)
