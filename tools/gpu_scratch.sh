python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.log
for c in C1 C2 C3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_$c.log 2>&1
  echo "$c rc=$?"; tail -1 gpurun_out/b_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('cuda_graph'), d['roofline']['frac'], d['roofline'].get('fused_graphs'))"
done
python -c "import __graft_entry__ as g; g.smoke()"
