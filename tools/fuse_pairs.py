"""dev tool: time hm_closeness_multi over chosen graphs of a config fused (bfs_fuse 1) vs one pass per graph.

    python tools/fuse_pairs.py C3 "2 3" "0 1" ...     # groups of layer ids; 'a' = every AND graph
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2207_11662_b200 import Context
from synth import build_config

name = sys.argv[1]
h = build_config(name)
with Context(0) as ctx:
    ctx.load_layers(h.V, [torch.from_numpy(L).cuda() for L in h.layers])
    ands = [ctx.and_aggregate(list(T)) for T in h.subsets]
    for grp in sys.argv[2:]:
        gids = ands if grp == "a" else [int(x) for x in grp.split()]
        for fuse in (0, 1, 0, 1):
            ctx.set_param("bfs_fuse", fuse)
            ctx.closeness_multi(gids)
            ctx.sync()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            for _ in range(3):
                ctx.closeness_multi(gids)
            e1.record(ctx.stream)
            torch.cuda.synchronize()
            print(f"{name} graphs {grp!r} fuse={fuse}: {e0.elapsed_time(e1) / 3:.3f} ms", flush=True)
