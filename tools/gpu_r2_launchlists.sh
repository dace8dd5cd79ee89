python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for c in C1 C2 C3; do
CMD="python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-graph"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv $CMD > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_$c.csv > gpurun_out/launch_summary_$c.txt 2>&1
echo "== $c"; head -22 gpurun_out/launch_summary_$c.txt
done
