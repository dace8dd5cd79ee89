# compute-sanitizer (memcheck, then initcheck) over the MS-BFS push phase and the default path on small graphs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np
from paper_2207_11662_b200 import Context
from synth import build_config
from oracle import oracle as O
for name, V, words, push in (("C5", 8192, 64, 8), ("C5", 8192, 128, 8), ("C4", 8192, 0, -1)):
    h = build_config(name, V=V)
    with Context(0) as ctx:
        ctx.set_param("bfs_words", words)
        ctx.set_param("bfs_push", push)
        ctx.load_layers(h.V, h.layers)
        g = ctx.and_aggregate(list(h.subsets[0]))
        for gid, E in ((0, set(map(tuple, h.layers[0].tolist()))),):
            got = ctx.closeness(gid)
            ref = O.analyze(h.V, E)
            assert got["S"].tolist() == ref["S"], (name, words)
        ctx.closeness(g)
        st = ctx.stats()
        print(name, V, words, push, "ok, push levels", st["bfs_td_levels"], flush=True)
PY
for tool in memcheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --kernel-regex kns=msbfs python /tmp/san.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|ok, push" gpurun_out/sanitize_$tool.log | tail -5
done
