# A/B of compile-time variants: DEFS="'' 'HM_X=1' ..." (each a space-free define list joined by ,);
# DEF_CONFIGS (default C5) x AB_GRAPHS (default "0 and"); REPS repetitions of the whole list
for rep in $(seq ${REPS:-1}); do
for D in ${DEFS:-none}; do
  [ "$D" = none ] && D=""
  HM_DEFINES="${D//,/ }" python -m paper_2207_11662_b200.build --force > gpurun_out/build.log 2>&1 || { echo "build failed $D"; continue; }
  echo "== defines: $D"
  for c in ${DEF_CONFIGS:-C5}; do for g in ${AB_GRAPHS:-0 and}; do timeout 300 python tools/prof_c5.py --config $c --graph $g; done; done
done
done > gpurun_out/defines.log 2>&1
python -m paper_2207_11662_b200.build --force > /dev/null 2>&1
