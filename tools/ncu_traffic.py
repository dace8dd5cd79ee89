"""Per-launch DRAM traffic of the MS-BFS kernel from an ncu --set full capture of a bench step.

    python tools/ncu_traffic.py gpurun_out/msbfs_step.ncu-rep profiles/r1_msbfs_traffic.json C5 64 11

Writes the mean dram__bytes_read.sum + dram__bytes_write.sum over the captured msbfs
launches (bench.py's roofline.traffic reads this file when config/words/hints match)."""
import csv
import io
import json
import subprocess
import sys

rep, out, cfg, words, hints = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
per = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if "msbfs" not in d.get("Kernel Name", ""):
        continue
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        b += float(d[k]) * scale[units[hdr.index(k)]]
    t = float(d["gpu__time_duration.sum"]) * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3,
                                              "nsecond": 1e-9}.get(units[hdr.index("gpu__time_duration.sum")], 1e-3)
    per.append({"kernel": d["Kernel Name"], "dram_bytes": b, "duration_s": t, "dram_GBps": b / t / 1e9})
res = {"config": cfg, "bfs_words": words, "bfs_hints": hints, "launches": len(per),
       "dram_bytes_per_launch": sum(p["dram_bytes"] for p in per) / max(1, len(per)),
       "per_launch": per,
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none (tools/gpu_traffic.sh), the MS-BFS launches of bench.py's setup pass "
                 "(3 layers + AND graph of one HoMLN); ncu replays are serialised and cold-cache"}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "per_launch"}))
for p in per:
    print(f"  {p['dram_bytes'] / 1e9:8.1f} GB  {p['duration_s'] * 1e3:8.2f} ms  {p['dram_GBps']:8.0f} GB/s")
