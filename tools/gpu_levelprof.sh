# per-phase profile of single BFS levels (HM_MSBFS_PROF build): LEVELS="1 2 3 6 10", G=graph, SETS="bfs_x=1 ..."
HM_MSBFS_PROF=1 python -m paper_2207_11662_b200.build --force > gpurun_out/build.log 2>&1
sets=""; for kv in ${SETS:-}; do sets="$sets --set $kv"; done
for L in ${LEVELS:-1 2 3 6 10}; do timeout 300 python tools/level_hist.py --graph ${G:-0} --level $L $sets; done 2>&1 | grep -v "d=" >> gpurun_out/levelprof.log
python -m paper_2207_11662_b200.build --force > /dev/null 2>&1
