for cap in 0 4 100; do
HM_DEFINES="HM_PLANE_CAP=$cap" python -m paper_2207_11662_b200.build --force > gpurun_out/build.log 2>&1 || exit 1
python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2207_11662_b200 import Context
from synth import build_config
h = build_config("C5")
with Context(0) as ctx:
    ctx.set_param("timing", 1)
    ctx.load_layers(h.V, h.layers)
    g = ctx.and_aggregate([0, 1, 2])
    ctx.closeness(g); ctx.sync(); ctx.stats(reset=True)
    ctx.closeness(g); ctx.sync(); st = ctx.stats(reset=True)
    print("AND", {k: st[k] for k in ("bfs_ms", "bfs_levels")})
PY
done
python -m paper_2207_11662_b200.build --force > /dev/null 2>&1
