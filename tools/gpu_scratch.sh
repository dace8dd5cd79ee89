# scratch: __grid_constant__ kernel parameter A/B on the C4 / C3 layer launches (and the C5 layer), same box
for D in none HM_NO_GRID_CONSTANT=1 none HM_NO_GRID_CONSTANT=1; do
DEFS=$D AB_CONFIG=C4 AB_CFGS="bfs_gd=0" AB_GRAPHS="0 1" bash tools/gpu_r2_ab.sh
DEFS=$D AB_CONFIG=C3 AB_CFGS="bfs_gd=0" AB_GRAPHS="0 2" bash tools/gpu_r2_ab.sh
done 2>&1 | tee gpurun_out/gc_ab.txt
