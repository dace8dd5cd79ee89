# sweep of one MS-BFS knob over the configs (ms per launch, layer 0 and AND graph):
# US_KNOB (default bfs_unit), US_UNITS values, US_CONFIGS, US_SETS extra "--set k=v" options
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in ${US_CONFIGS:-C1 C2 C3 C4}; do for u in ${US_UNITS:-32 16 8}; do for g in 0 and; do
  timeout 300 python tools/prof_c5.py --config $c --graph $g --set ${US_KNOB:-bfs_unit}=$u ${US_SETS}; done; done; done > gpurun_out/unit_sweep.log 2>&1
