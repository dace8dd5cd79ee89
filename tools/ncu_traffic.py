"""Per-launch DRAM traffic of the MS-BFS kernel from an ncu capture of bench.py's setup pass.

    python tools/ncu_traffic.py gpurun_out/msbfs_traffic.ncu-rep profiles/r2_msbfs_traffic.json C5 64 11

The setup pass runs one MS-BFS launch per graph in this order: the layers L0..L{l-1}, then the AND
graph of every subset; the captured launches are named accordingly (per_graph).  Writes
dram__bytes_read.sum + dram__bytes_write.sum, duration and L2 hit rate per launch, plus the
src_sha of the MS-BFS sources (bench.py uses the file only for the same build, config, batch
width and L2 policy)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

rep, out, cfg, words, hints = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, units = rows[hi], rows[hi + 1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
tscale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
per = []
for r in rows[hi + 2:]:
    d = dict(zip(hdr, r))
    if "msbfs" not in d.get("Kernel Name", ""):
        continue
    b = sum(float(d[k]) * scale[units[hdr.index(k)]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    t = float(d["gpu__time_duration.sum"]) * tscale.get(units[hdr.index("gpu__time_duration.sum")], 1e-3)
    e = {"kernel": d["Kernel Name"], "dram_bytes": b, "duration_s": t, "dram_GBps": b / t / 1e9}
    if "lts__t_sector_hit_rate.pct" in d:
        e["l2_hit_pct"] = float(d["lts__t_sector_hit_rate.pct"])
    per.append(e)
from synth import build_config  # noqa: E402
from bench import src_digest  # noqa: E402
h = build_config(cfg)
names = [f"L{i}" for i in range(len(h.layers))] + ["AND" + "".join(map(str, T)) for T in h.subsets]
res = {"config": cfg, "bfs_words": words, "bfs_hints": hints, "src_sha": src_digest(), "launches": len(per),
       "dram_bytes_per_launch": sum(p["dram_bytes"] for p in per) / max(1, len(per)),
       "per_launch": per, "per_graph": dict(zip(names, per)),
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                 "lts__t_sector_hit_rate.pct --clock-control none (tools/gpu_traffic.sh), the MS-BFS launches of "
                 "bench.py's setup pass (layers, then AND graphs); ncu replays are serialised and cold-cache"}
# optional: a second capture of the step's own launches in steady state (graphs fused by bfs_fuse), e.g.
# `-s <graphs> -c 2` on bench.py: the longest launch is the layers' (C5: the three layers fused)
if len(sys.argv) > 6 and os.path.exists(sys.argv[6]):
    raw2 = subprocess.run(["ncu", "-i", sys.argv[6], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows2 = list(csv.reader(io.StringIO(raw2)))
    h2 = next(i for i, r in enumerate(rows2) if "Kernel Name" in r)
    hdr2, units2 = rows2[h2], rows2[h2 + 1]
    step = []
    for r in rows2[h2 + 2:]:
        d = dict(zip(hdr2, r))
        if "msbfs" not in d.get("Kernel Name", ""):
            continue
        b = sum(float(d[k]) * scale[units2[hdr2.index(k)]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        t = float(d["gpu__time_duration.sum"]) * tscale.get(units2[hdr2.index("gpu__time_duration.sum")], 1e-3)
        e = {"kernel": d["Kernel Name"], "dram_bytes": b, "duration_s": t, "dram_GBps": b / t / 1e9}
        if "lts__t_sector_hit_rate.pct" in d:
            e["l2_hit_pct"] = float(d["lts__t_sector_hit_rate.pct"])
        step.append(e)
    if step:
        res["step_launches"] = {"layers": max(step, key=lambda e: e["duration_s"]), "all": step}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k not in ("per_launch", "per_graph")}))
for n, p in zip(names, per):
    print(f"  {n:8s} {p['dram_bytes'] / 1e9:8.1f} GB  {p['duration_s'] * 1e3:8.2f} ms  {p['dram_GBps']:8.0f} GB/s"
          f"  L2 hit {p.get('l2_hit_pct', float('nan')):.1f} %")
