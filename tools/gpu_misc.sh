# round-1 follow-ups: full GPU tests, W=32 vs W=64 A/B on C5, per-level histograms of the small configs
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
for cfg in "bfs_words=64" "bfs_words=32" "bfs_words=32 bfs_hints=3" "bfs_words=64"; do
  sets=""; for kv in $cfg; do sets="$sets --set $kv"; done
  for g in 0 and; do timeout 300 python tools/prof_c5.py --config C5 --graph $g $sets; done
done > gpurun_out/ab.log 2>&1
for c in C1 C2 C3; do for g in 0 and; do timeout 300 python tools/level_hist.py --config $c --graph $g; done; done > gpurun_out/levels_small.log 2>&1
