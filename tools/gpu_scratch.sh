# scratch: A/B of bfs_push on the C5 AND launch (and layer), PU 4 / 8
for D in none HM_PUSH_PU=8; do
DEFS=$D AB_CFGS="bfs_push=0;bfs_push=4;bfs_push=8;bfs_push=12;bfs_push=16;bfs_push=24" AB_GRAPHS="and" bash tools/gpu_r2_ab.sh
done 2>&1 | tee gpurun_out/push_ab2.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/prof_c5.py --config C5 --graph 0 --set bfs_push=8 | tee -a gpurun_out/push_ab2.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "push_phase" > gpurun_out/push_tests.log 2>&1; echo "push tests rc=$?"; tail -3 gpurun_out/push_tests.log
(timeout 300 python tools/level_hist.py --config C5 --graph and --set bfs_push=8) > gpurun_out/push_levels.txt 2>&1
for c in C3 C4; do for p in 0 8; do for g in 0 1 and; do timeout 300 python tools/prof_c5.py --config $c --graph $g --set bfs_push=$p; done; done; done 2>&1 | grep -v Warn | tee -a gpurun_out/push_ab2.txt
