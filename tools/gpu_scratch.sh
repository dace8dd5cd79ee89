python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in C5 C3 C1; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/b_$c.log 2>&1
  echo "$c rc=$?"; tail -1 gpurun_out/b_$c.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['ms_per_step'], d['e2e']['ms_per_step'], d['cuda_graph'], r['kernel'], round(r['frac'],3), r['ms_per_launch'], json.dumps(r['l2_row_traffic'])[:200])
for k,v in r['step_launches'].items(): print(' ', k, v)"
done
