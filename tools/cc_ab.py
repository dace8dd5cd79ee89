"""dev tool: connected-components phase time and results per cc_init (library timing = 2)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_11662_b200 import Context
from synth import build_config

for name in sys.argv[1:]:
    h = build_config(name)
    for cc in (2, 3):
        with Context(0) as ctx:
            ctx.set_param("cc_init", cc)
            ctx.load_layers(h.V, [torch.from_numpy(L).cuda() for L in h.layers])
            for g in range(len(h.layers)):
                for rep in range(2):
                    ctx.set_param("timing", 2)
                    ctx.stats(reset=True)
                    r = ctx.closeness(g)
                    st = ctx.stats(reset=True)
                print(f"{name} L{g} cc_init={cc}: components {st['phase_ms'][0]:.4f} ms, S sum {int(r['S'].sum())}",
                      flush=True)
