# bench every BASELINE config (ours), one line each into gpurun_out/configs.jsonl
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
rm -f gpurun_out/configs.jsonl
for c in ${CFGS:-C1 C2 C3 C4 C5}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline ${BENCH_ARGS} 2> gpurun_out/bench_err_$c.log | tail -1 >> gpurun_out/configs.jsonl
done
python - <<'PY'
import json
for ln in open("gpurun_out/configs.jsonl"):
    try:
        l = json.loads(ln)
    except Exception:
        print("bad line", ln[:200]); continue
    print(l["config"]["workload"], "ms/step %.3f" % l["ms_per_step"], "TEPS %.3e" % l["value"],
          "e2e ms %.3f" % (l["e2e"] or {}).get("ms_per_step", float("nan")), "graph", l.get("cuda_graph"),
          "launches", l["gpu_launches"], "clk", l["clocks"].get("sm_mhz"), l["clocks"].get("samples"), l["clocks"].get("reasons"))
PY
