# DRAM bytes of every MS-BFS launch of bench.py's setup pass (3 layers + AND): metrics-only ncu capture
python -m paper_2207_11662_b200.build > gpurun_out/build.log 2>&1
P="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
$P > gpurun_out/plain3.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none \
      -k regex:msbfs -c ${NCU_C:-4} -o gpurun_out/msbfs_traffic -f $P > gpurun_out/ncu_traffic.log 2>&1
echo "ncu traffic rc=$?"
