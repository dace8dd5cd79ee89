# level-1 push step (HM_TD1=1; the kernel with it is tools/experiments/msbfs_level1_push.cu.txt -- copy it over
# csrc/msbfs.cu first): parity tests on that build, then a same-call A/B against the default build
HM_DEFINES="HM_TD1=1" python -m paper_2207_11662_b200.build --force > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests_td1.log 2>&1; echo "td1 tests rc=$?"
REPS=2 DEF_CONFIGS="${TD_CONFIGS:-C5 C4 C3}" DEFS="none HM_TD1=1" bash tools/gpu_defines.sh
