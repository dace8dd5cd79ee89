# A/B of MS-BFS variants: AB_CFGS="cfgA;cfgB" with each cfg a space-separated list of name=value params
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q ${AB_K:+-k "$AB_K"} > gpurun_out/gputests_ab.log 2>&1; echo "tests rc=$?"
IFS=';' read -ra CFGS <<< "${AB_CFGS:-bfs_words=32}"
for cfg in "${CFGS[@]}"; do
  sets=""; for kv in $cfg; do sets="$sets --set $kv"; done
  for g in ${AB_GRAPHS:-0 and}; do timeout 300 python tools/prof_c5.py --config ${AB_CONFIG:-C5} --graph $g $sets; done
done > gpurun_out/ab.log 2>&1
