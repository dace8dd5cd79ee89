# A/B: DEFS (compile-time define lists, ',' separated; 'none' = defaults) x AB_CFGS (';'-separated runtime
# param sets) x AB_GRAPHS of AB_CONFIG (default C5: layer 0 and the AND graph)
for D in ${DEFS:-none}; do
  [ "$D" = none ] && D=""
  HM_DEFINES="${D//,/ }" python -m paper_2207_11662_b200.build --force > gpurun_out/build.log 2>&1 || { echo "build failed $D"; continue; }
  IFS=';' read -ra CFGS <<< "${AB_CFGS:-bfs_gd=0}"
  for cfg in "${CFGS[@]}"; do
    sets=""; for kv in $cfg; do sets="$sets --set $kv"; done
    for g in ${AB_GRAPHS:-0 and}; do echo -n "[$D] "; timeout 300 python tools/prof_c5.py --config ${AB_CONFIG:-C5} --graph $g $sets; done
  done 2>&1 | grep -v Warn
done
python -m paper_2207_11662_b200.build --force > /dev/null 2>&1
