# scratch: push level with several lanes per pair on short lists: parity test, AND / layer A/B, level histogram
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "push_phase" > gpurun_out/push_tests.log 2>&1; echo "push tests rc=$?"; tail -3 gpurun_out/push_tests.log
for p in 0 8 -1; do timeout 300 python tools/prof_c5.py --config C5 --graph and --set bfs_push=$p; done 2>&1 | grep -v Warn | tee gpurun_out/push_ab3.txt
timeout 300 python tools/prof_c5.py --config C5 --graph 0 --set bfs_push=8 2>&1 | grep -v Warn | tee -a gpurun_out/push_ab3.txt
timeout 300 python tools/prof_c5.py --config C5 --graph 0 --set bfs_push=2 2>&1 | grep -v Warn | tee -a gpurun_out/push_ab3.txt
(timeout 300 python tools/level_hist.py --config C5 --graph and; timeout 300 python tools/level_hist.py --config C5 --graph 0 --set bfs_push=2) > gpurun_out/push_levels3.txt 2>&1
