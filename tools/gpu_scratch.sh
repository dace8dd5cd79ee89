# scratch (last ad-hoc GPU experiment): bfs_push A/B on the C5 AND and layer launches, push-phase parity test, level histogram
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "push_phase" > gpurun_out/push_tests.log 2>&1; echo "push tests rc=$?"; tail -3 gpurun_out/push_tests.log
for p in 0 2 8 -1; do for g in 0 and; do timeout 300 python tools/prof_c5.py --config C5 --graph $g --set bfs_push=$p; done; done 2>&1 | grep -v Warn | tee gpurun_out/push_ab.txt
(timeout 300 python tools/level_hist.py --config C5 --graph and; timeout 300 python tools/level_hist.py --config C5 --graph 0 --set bfs_push=2) > gpurun_out/push_levels.txt 2>&1
