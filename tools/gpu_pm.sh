python -m paper_2207_11662_b200.build --force > gpurun_out/build.log 2>&1
timeout 600 ncu --section PmSampling --section PmSampling_WarpStates --section SpeedOfLight --section MemoryWorkloadAnalysis_Tables --clock-control none -k regex:msbfs --launch-skip 1 -c 1 -o gpurun_out/pm_w32 -f python tools/prof_c5.py --words 32 --streams 1 --graph 0 > gpurun_out/pm.log 2>&1
echo rc=$?
