# copy what tools/gpu_r2_evidence.sh brought back in gpurun_out/ into profiles/ (run here, after the gpurun call)
G=gpurun_out P=profiles
tail -1 $G/bench_C5.log > $P/r2_bench_line_C5.json
tail -1 $G/bench_ref_C5.log > $P/r2_reference_arm_line_C5.json
tail -1 $G/bench_shard_C5.log > $P/r2_shard_n1_line_C5.json
{ cat $G/configs.jsonl; tail -1 $G/bench_C5.log; } > $P/r2_all_configs_bench_lines.jsonl
cp $G/launches_C5.csv $P/r2_launches_C5.csv
cp $G/launch_summary_C5.txt $P/r2_launch_list_summary_C5.txt
cp $G/r2_msbfs_traffic_C5.json $P/
{ echo "ncu --set full --clock-control none --import-source on, C5 AND-graph MS-BFS launch alone (msbfs_kernel<128,16,2,2,weighted,lean,TC,PS>, 8192 sources per batch, T-ordered core, top-down push phase on the first levels), round-2 final build"; cat $G/ncu_summary_C5_3.txt; } > $P/r2_ncu_and_C5.txt
{ echo "ncu --set full --clock-control none --import-source on: first MS-BFS launch (C5 layer 0, separate pass) of bench.py's setup pass, round-2 final build (tools/gpu_r2_round.sh)"; cat $G/ncu_summary_C5_0.txt; } > $P/r2_ncu_layer_C5.txt
{ echo "per-level MS-BFS time (bfs_dbg=2, tools/level_hist.py), C5 layer 0 and the AND graph (separate passes; the AND graph's levels 1-4 run the top-down push phase), round-2 final build"; cat $G/level_hist_C5.txt; } > $P/r2_level_histograms_C5.txt
{ echo "tools/phase_profile.py C1..C5: one eager step (bench's Psi through hm_closeness_multi) with library timing = 2 (CUDA events around every phase), round-2 final build"; cat $G/phases.txt; } > $P/r2_phase_profiles.txt
