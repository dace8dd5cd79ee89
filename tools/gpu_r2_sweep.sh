python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "not (test_fullsize_config and C5)" > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputests.log
DEFS="none HM_BLOCK_PLAIN=512,HM_BLOCK_WEIGHTED=448 HM_BLOCK_PLAIN=384,HM_BLOCK_WEIGHTED=320 HM_CAP=448 HM_BLOCK_PLAIN=480,HM_BLOCK_WEIGHTED=416" REPS=1 bash tools/gpu_defines.sh
cat gpurun_out/defines.log
