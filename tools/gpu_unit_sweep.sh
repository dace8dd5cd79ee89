# MS-BFS work-unit size sweep over the configs (ms per launch, layer 0 and AND graph)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in ${US_CONFIGS:-C1 C2 C3 C4}; do for u in ${US_UNITS:-32 16 8}; do for g in 0 and; do
  timeout 300 python tools/prof_c5.py --config $c --graph $g --set bfs_unit=$u ${US_SETS}; done; done; done > gpurun_out/unit_sweep.log 2>&1
