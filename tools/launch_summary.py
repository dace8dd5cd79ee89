"""summarise an ncu launch list (gpu__time_duration per launch) by kernel name"""
import csv, sys, collections, re
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
hdr = rows[0]
data = [dict(zip(hdr, r)) for r in rows[1:] if r[hdr.index("Metric Name")] == "gpu__time_duration.sum"]
tot = collections.defaultdict(float)
cnt = collections.Counter()
for d in data:
    name = d["Kernel Name"]
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    name = name.replace("hm::<unnamed>::", "hm::").replace("hm::(anonymous namespace)::", "hm::")
    name = name[:70]
    tot[name] += float(d["Metric Value"]) / 1e6
    cnt[name] += 1
T = sum(tot.values())
print(f"{len(data)} launches, {T:.1f} ms total (ncu serialised, cold caches)")
for n, t in sorted(tot.items(), key=lambda x: -x[1])[:25]:
    print(f"  {100*t/T:5.1f}%  {t:9.3f} ms  x{cnt[n]:<5d} {n}")
