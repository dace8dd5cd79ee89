python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for w in 32 64; do for g in 0 and; do timeout 300 python tools/level_hist.py --words $w --graph $g; done; done > gpurun_out/hist.log 2>&1
