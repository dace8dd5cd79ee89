"""dev tool: per-phase time of one bench step (library timing = 2: CUDA events around every phase).

    python tools/phase_profile.py C3 [C4 ...]
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_11662_b200 import Context
from synth import build_config

NAMES = ["components", "prune decision", "relabel", "bfs setup", "msbfs", "finalize", "compose", "topk",
         "aggregate", "other"]
for name in sys.argv[1:] or ["C3"]:
    h = build_config(name)
    with Context(0) as ctx:
        ctx.load_layers(h.V, [torch.from_numpy(L).cuda() for L in h.layers])
        ids = torch.zeros(h.K, dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")

        def step():
            ands = [ctx.and_aggregate(list(T)) for T in h.subsets]
            ctx.closeness_multi(list(range(len(h.layers))) + ands)     # bench's Psi (fused when small)
            for T, g in zip(h.subsets, ands):
                ctx.topk_closeness(g, h.K, out=ids)
                for heur in ("cc2", "cc1" if len(T) == 2 else "cc1_rary", "naive"):
                    ctx.compose(heur, list(T), h.K, out=ids, count_out=cnt)
                ctx.free_graph(g)
        step()
        ctx.sync()
        ctx.set_param("timing", 2)
        ctx.stats(reset=True)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        step()
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        st = ctx.stats(reset=True)
        tot = e0.elapsed_time(e1)
        print(f"{name}: step {tot:.3f} ms (with phase events), host syncs {st['host_syncs']}")
        for n, v in zip(NAMES, st["phase_ms"]):
            if v:
                print(f"  {n:<16} {v:8.3f} ms  {100 * v / tot:5.1f} %")
