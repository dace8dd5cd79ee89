# round-2 evidence in one call: tools/gpu_r2_round.sh on C5 (GPU tests, smoke, ncu DRAM traffic of the
# MS-BFS launches, bench + reference arm, ncu launch list, ncu full capture, --shard at N = 1), bench lines
# of C1-C4, per-phase profiles, level histograms of the C5 launches
CFG=C5 bash tools/gpu_r2_round.sh > gpurun_out/round.log 2>&1; echo "round rc=$?"
CFGS="C1 C2 C3 C4" bash tools/gpu_r2_configs.sh > gpurun_out/configs_summary.txt 2>&1; cat gpurun_out/configs_summary.txt
timeout 600 python tools/phase_profile.py C1 C2 C3 C4 C5 > gpurun_out/phases.txt 2>&1
(timeout 300 python tools/level_hist.py --config C5 --graph 0; timeout 300 python tools/level_hist.py --config C5 --graph and) > gpurun_out/level_hist_C5.txt 2>&1
# gpurun copies back at most 64 MiB: the ncu reports are summarised above, only the text goes home
rm -f gpurun_out/*.ncu-rep
