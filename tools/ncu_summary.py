"""summarise an ncu report: key SOL metrics + top stall lines (sass)"""
import csv, subprocess, sys, io
rep = sys.argv[1]
k_launch = int(sys.argv[2]) if len(sys.argv) > 2 else 0      # which captured launch (0 = first)
sel = ["--launch-skip", str(k_launch), "--launch-count", "1"] if k_launch else []
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(det)))
hdr = r[0]
want = ["Duration", "DRAM Throughput", "L2 Cache Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "L1/TEX Hit Rate", "L2 Hit Rate", "Memory Throughput", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Avg. Active Threads Per Warp", "Registers Per Thread", "Achieved Occupancy",
        "Eligible Warps Per Scheduler", "No Eligible"]
ids = []
for row in r[1:]:
    i = dict(zip(hdr, row)).get("ID")
    if i not in ids:
        ids.append(i)
first = ids[k_launch] if len(ids) > k_launch else None
for row in r[1:]:
    d = dict(zip(hdr, row))
    if d.get("ID") != first:          # the selected captured launch only
        continue
    if d.get("Metric Name") in want:
        print(f"  {d['Metric Name']:<40} {d['Metric Value']:>16} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h2 = rr[0]
vals = dict(zip(h2, rr[2 + k_launch])) if len(rr) > 2 + k_launch else {}
units = dict(zip(h2, rr[1])) if len(rr) > 1 else {}
for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "gpu__time_duration.sum"]:
    if k in vals:
        print(f"  {k:<40} {vals[k]:>16} {units.get(k,'')}")
sass = subprocess.run(["ncu", "-i", rep, *sel, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                      text=True).stdout
rows = list(csv.reader(io.StringIO(sass)))
hdr = rows[1]
data = []
for x in rows[2:]:                    # first kernel's section only
    if x and x[0] == "Kernel Name":
        break
    if len(x) == len(hdr) and x[0] != hdr[0]:
        data.append(dict(zip(hdr, x)))
f = lambda x: float(x) if x not in ("", None) else 0.0
tot = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data) or 1
stalls = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(f(d[c]) for d in data) for c in stalls}
print("  stalls:", ", ".join(f"{c[6:]}={100*v/tot:.1f}%" for c, v in sorted(agg.items(), key=lambda x: -x[1])[:7]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
for d in sorted(data, key=lambda d: -f(d["Warp Stall Sampling (All Samples)"]))[:n]:
    st = sorted(((c[6:], f(d[c])) for c in stalls), key=lambda x: -x[1])[:2]
    print(f"  {d['Address'][-5:]} {d['Source'][:58]:<58} {100*f(d['Warp Stall Sampling (All Samples)'])/tot:5.1f}% {st[0][0]}")
