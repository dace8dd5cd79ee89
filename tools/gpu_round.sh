# Round artifacts on one B200: GPU tests, smoke, bench (ours + reference arm), ncu launch list, ncu full capture.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
[ -n "$NO_REF" ] || { timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; }
[ -n "$NO_NCU" ] && exit 0
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "ncu list rc=$?"
# full capture of the 4 MS-BFS launches of bench.py's setup pass (3 layers + AND of one HoMLN)
P="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$P > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:msbfs -c 4 -o gpurun_out/msbfs_full -f $P > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
