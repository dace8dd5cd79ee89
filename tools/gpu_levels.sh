# per-level MS-BFS time histograms (non-profiling build, bfs_dbg=2) for the C5 layer and AND graphs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for g in ${LV_GRAPHS:-0 and}; do timeout 300 python tools/level_hist.py --config ${LV_CONFIG:-C5} --graph $g ${LV_SETS}; done > gpurun_out/levels.log 2>&1
