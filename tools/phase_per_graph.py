"""dev tool: per-phase time of each closeness call of a config (library timing = 2)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_11662_b200 import Context
from synth import build_config

NAMES = ["cc", "prune", "relabel", "setup", "msbfs", "final"]
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
h = build_config(name)
with Context(0) as ctx:
    ctx.load_layers(h.V, [torch.from_numpy(L).cuda() for L in h.layers])
    gs = [(f"L{i}", i) for i in range(len(h.layers))] + [("AND" + "".join(map(str, T)), ctx.and_aggregate(list(T)))
                                                         for T in h.subsets[:3]]
    for n, g in gs:
        ctx.closeness(g, out={})
    ctx.sync()
    ctx.set_param("timing", 2)
    for n, g in gs:
        ctx.stats(reset=True)
        ctx.closeness(g, out={})
        ctx.sync()
        st = ctx.stats(reset=True)
        print(n, " ".join(f"{k}={v * 1e3:.0f}us" for k, v in zip(NAMES, st["phase_ms"][:6])), flush=True)
