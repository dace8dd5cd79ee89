# A/B: skip the gathers of full chunks (HM_FULL_SKIP 0 / 1 / 2), C5 layer 0 + AND, C4 layer 0 + AND, control repeat
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
DEFS="HM_FULL_SKIP=0 HM_FULL_SKIP=1 HM_FULL_SKIP=2 HM_FULL_SKIP=0" AB_CFGS="bfs_gd=0" bash tools/gpu_r2_ab.sh
DEFS="HM_FULL_SKIP=0 HM_FULL_SKIP=1 HM_FULL_SKIP=2" AB_CONFIG=C4 AB_CFGS="bfs_gd=0" bash tools/gpu_r2_ab.sh
