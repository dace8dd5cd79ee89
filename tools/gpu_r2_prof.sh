# round-2 profiling: ncu DRAM bytes + L2 hit of the 4 MS-BFS launches of a C5 step, per-phase level profiles
bash tools/gpu_traffic.sh; tail -3 gpurun_out/ncu_traffic.log
ncu -i gpurun_out/msbfs_traffic.ncu-rep --page raw --csv > gpurun_out/msbfs_traffic.csv 2>&1
rm -f gpurun_out/levelprof.log
G=0 LEVELS="2 5" bash tools/gpu_levelprof.sh
G=and LEVELS="2 10 18" bash tools/gpu_levelprof.sh
cat gpurun_out/levelprof.log
DEFS="HM_BLOCK_WEIGHTED=288 HM_BLOCK_WEIGHTED=320 HM_BLOCK_WEIGHTED=352" AB_GRAPHS=and bash tools/gpu_defines.sh
cat gpurun_out/defines.log
