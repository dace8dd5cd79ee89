python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
# ncu full capture of the C5 AND launch alone (W = 128 weighted kernel)
cat > /tmp/and_only.py <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2207_11662_b200 import Context
from synth import build_config
h = build_config("C5")
with Context(0) as ctx:
    ctx.load_layers(h.V, h.layers)
    g = ctx.and_aggregate([0, 1, 2])
    ctx.closeness(g, out={})
    ctx.sync()
PY
ncu --set full --clock-control none --import-source on -k regex:msbfs -c 1 -o gpurun_out/msbfs_full_and -f python /tmp/and_only.py > gpurun_out/ncu_and.log 2>&1; echo "ncu and rc=$?"
python tools/ncu_summary.py gpurun_out/msbfs_full_and.ncu-rep 0 > gpurun_out/ncu_summary_and.txt 2>&1
for g in 0 and; do python tools/level_hist.py --graph $g 2>&1; done > gpurun_out/levels_r2.log
for p in 0 2; do AB_CONFIG=C2 AB_CFGS="bfs_prune=$p" bash tools/gpu_r2_ab.sh; done
for p in 0 2; do python bench.py --config C2 --set bfs_prune=$p --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | tail -1 | python3 -c "
import json,sys; l=json.loads(sys.stdin.read()); print('C2 prune', $p, l['ms_per_step'], l['cuda_graph'])" ; done
