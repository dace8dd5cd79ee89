# round-2 artifacts on one B200: GPU tests, smoke, ncu traffic of the MS-BFS launches, bench (ours +
# reference arm), ncu launch list of the bench command
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
fi
CFG=${CFG:-C5}
P="python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$P > gpurun_out/plain3.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none \
      -k regex:msbfs -c ${NCU_C:-4} -o gpurun_out/msbfs_traffic -f $P > gpurun_out/ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
# the step's own launches in steady state (second setup step: graphs fused by bfs_fuse)
NG=$(python -c "from synth import build_config as b; h=b('$CFG'); print(len(h.layers)+len(h.subsets))")
$P > /dev/null 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none \
      -k regex:msbfs -s $NG -c 2 -o gpurun_out/msbfs_traffic_step -f $P > gpurun_out/ncu_traffic_step.log 2>&1
python tools/ncu_traffic.py gpurun_out/msbfs_traffic.ncu-rep gpurun_out/r2_msbfs_traffic_$CFG.json $CFG 0 11 \
    gpurun_out/msbfs_traffic_step.ncu-rep && \
  cp gpurun_out/r2_msbfs_traffic_$CFG.json profiles/
timeout 900 python bench.py --config $CFG ${BENCH_ARGS} > gpurun_out/bench_$CFG.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_$CFG.log | cut -c1-600
[ -n "$NO_REF" ] || { timeout 900 python bench.py --config $CFG --impl reference > gpurun_out/bench_ref_$CFG.log 2>&1; echo "ref rc=$?"; }
[ -n "$NO_NCU" ] && exit 0
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_list.log 2>&1
echo "ncu list rc=$?"
# full ncu capture of the 4 MS-BFS launches of bench.py's setup pass (3 layers + AND of one HoMLN)
[ -n "$NO_FULL" ] && exit 0
P="python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph"
$P > gpurun_out/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:msbfs -c ${NCU_C:-4} -o gpurun_out/msbfs_full_$CFG -f $P > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
python tools/ncu_summary.py gpurun_out/msbfs_full_$CFG.ncu-rep 0 > gpurun_out/ncu_summary_${CFG}_0.txt 2>&1
# the AND launch alone (its replay inside the 4-launch capture reports no metrics)
cat > /tmp/and_only.py <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2207_11662_b200 import Context
from synth import build_config
h = build_config(sys.argv[1])
with Context(0) as ctx:
    ctx.load_layers(h.V, h.layers)
    g = ctx.and_aggregate(list(h.subsets[0]))
    ctx.closeness(g, out={})
    ctx.sync()
PY
python /tmp/and_only.py $CFG && ncu --set full --clock-control none --import-source on -k regex:msbfs -c 1 \
  -o gpurun_out/msbfs_full_and_$CFG -f python /tmp/and_only.py $CFG > gpurun_out/ncu_and.log 2>&1
python tools/ncu_summary.py gpurun_out/msbfs_full_and_$CFG.ncu-rep 0 > gpurun_out/ncu_summary_${CFG}_3.txt 2>&1
python tools/launch_summary.py gpurun_out/launches_$CFG.csv > gpurun_out/launch_summary_$CFG.txt 2>&1
# source-batch sharding at N = 1 (the partial/combine split's own cost)
timeout 900 python bench.py --config $CFG --shard --no-cpu-baseline --no-e2e > gpurun_out/bench_shard_$CFG.log 2>&1; echo "shard rc=$?"
