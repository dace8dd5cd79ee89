"""dev tool: where the e2e (host arrays -> public API -> host results) time goes on one HoMLN."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2207_11662_b200 import Context
from synth import build_config

h = build_config(sys.argv[1] if len(sys.argv) > 1 else "C5")
host = [torch.from_numpy(np.ascontiguousarray(L, dtype=np.int32)).pin_memory() for L in h.layers]
with Context(0) as ctx:
    s = torch.cuda.current_stream()
    for it in range(3):
        marks = []
        def mark(name):
            torch.cuda.synchronize()
            marks.append((name, time.perf_counter()))
        mark("start")
        ctx.load_layers(h.V, [t.numpy() for t in host]); mark("load_layers")
        ands = [ctx.and_aggregate(list(T)) for T in h.subsets]; mark("and")
        for g in list(range(len(h.layers))) + ands:
            ctx.closeness(g, out={}); mark(f"closeness{g}")
        for T, g in zip(h.subsets, ands):
            ctx.topk_closeness(g, h.K); mark("topk")
            ctx.compose("cc2", list(T), h.K); mark("cc2")
            ctx.compose("cc1" if len(T) == 2 else "cc1_rary", list(T), h.K); mark("cc1")
            ctx.compose("naive", list(T), h.K); mark("naive")
            ctx.free_graph(g); mark("free")
        print(" ".join(f"{n}={1e3 * (t - marks[i][1]):.1f}" for i, (n, t) in enumerate(marks[1:])),
              f"total={1e3 * (marks[-1][1] - marks[0][1]):.1f} ms", flush=True)
