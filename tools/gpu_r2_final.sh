# round-2 final evidence: GPU tests, smoke, bench on every config (lines to gpurun_out/final_configs.jsonl),
# reference arm on C5, phase profile
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
rm -f gpurun_out/final_configs.jsonl
for c in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --config $c > gpurun_out/final_bench_$c.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/final_bench_$c.log >> gpurun_out/final_configs.jsonl
done
timeout 900 python bench.py --config C5 --impl reference > gpurun_out/final_ref_C5.log 2>&1; echo "ref rc=$?"
python tools/phase_profile.py C1 C2 C3 C4 C5 > gpurun_out/final_phases.txt 2>&1
