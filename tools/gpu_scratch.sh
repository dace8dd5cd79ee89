python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for t in 1 4096 2048 1024 0; do
  timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --set topk_tiles=$t > gpurun_out/b_C3.log 2>&1
  echo "C3 topk_tiles=$t rc=$?"; tail -1 gpurun_out/b_C3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"
done
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "topk" > gpurun_out/t.log 2>&1; echo "topk tests rc=$?"; tail -1 gpurun_out/t.log
