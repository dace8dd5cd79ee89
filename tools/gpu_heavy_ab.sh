# A/B: previous heavy path (tools/experiments/msbfs_prev_heavy.cu.txt) vs chunked heavy items with HM_HEAVY_GD in flight
CU=paper_2207_11662_b200/csrc/msbfs.cu
cp $CU /tmp/msbfs_new.cu
run() { for c in ${HA_CONFIGS:-C5 C4}; do for g in 0 and; do timeout 300 python tools/prof_c5.py --config $c --graph $g; done; done; }
{
for rep in 1 2; do
  cp tools/experiments/msbfs_prev_heavy.cu.txt $CU; python -m paper_2207_11662_b200.build --force > gpurun_out/build.log 2>&1 || echo "build failed prev"
  echo "== prev"; run
  cp /tmp/msbfs_new.cu $CU
  for gd in ${HA_GDS:-1 4}; do for gu in ${HA_GUARDS:-0}; do
    HM_DEFINES="HM_HEAVY_GD=$gd HM_HV_NOINLINE=$gu" python -m paper_2207_11662_b200.build --force > gpurun_out/build.log 2>&1 || echo "build failed $gd"
    echo "== items gd=$gd noinline=$gu"; run
  done; done
done
} > gpurun_out/heavy_ab.log 2>&1
cp /tmp/msbfs_new.cu $CU
python -m paper_2207_11662_b200.build --force > /dev/null 2>&1
