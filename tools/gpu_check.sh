set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_w32.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --words 64 --no-cpu-baseline > gpurun_out/bench_w64.log 2>&1; echo "bench64 rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --fused --no-cpu-baseline > gpurun_out/bench_fused.log 2>&1; echo "benchf rc=$?"
