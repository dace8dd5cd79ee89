# round-2 iteration: build, GPU parity (fast subset unless FULL=1), C5 bench, per-level histograms
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
if [ -n "$FULL" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
else
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
fi
tail -4 gpurun_out/gputests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
l=json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
r=l["roofline"]; print("ms/step", round(l["ms_per_step"],2), "TEPS %.3e"%l["value"], "bfs ms/launch", round(r["ms_per_launch"],2), "frac", round(r["frac"],3), "clk", l["clocks"]["sm_mhz"])
print({k:v for k,v in (l.get("breakdown_ms") or {}).items() if k.startswith(("psi","gt_clo","and_","theta"))})
PY
for g in 0 and; do timeout 300 python tools/level_hist.py --config C5 --graph $g; done > gpurun_out/levels.log 2>&1
cat gpurun_out/levels.log
