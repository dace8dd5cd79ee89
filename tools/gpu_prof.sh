# per-phase profile (HM_MSBFS_PROF build) of MS-BFS variants; AB_CFGS as in gpu_ab.sh
HM_MSBFS_PROF=1 python -m paper_2207_11662_b200.build --force > gpurun_out/build.log 2>&1
IFS=';' read -ra CFGS <<< "${AB_CFGS:-bfs_words=32}"
for cfg in "${CFGS[@]}"; do
  sets=""; for kv in $cfg; do sets="$sets --set $kv"; done
  for g in ${AB_GRAPHS:-0 and}; do timeout 300 python tools/level_hist.py --config ${PROF_CONFIG:-C5} --graph $g $sets; done
done > gpurun_out/prof.log 2>&1
python -m paper_2207_11662_b200.build --force > /dev/null 2>&1
