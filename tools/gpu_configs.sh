# bench.py on every BASELINE config (device-timed step; no e2e / cpu baseline)
python -m paper_2207_11662_b200.build > gpurun_out/build.log 2>&1
for c in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1
  echo "$c rc=$?"
done
