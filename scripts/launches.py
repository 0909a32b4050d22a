"""Print an ncu --metrics gpu__time_duration.sum launch list (csv) as name / us / grid."""
import csv, re, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(list)
for d in data:
    m = re.search(r"(k_[a-z0-9_]+)", d["Kernel Name"])
    name = m.group(1) if m else d["Kernel Name"][:30]
    us = float(d["Metric Value"].replace(",", "")) / (1e3 if d["Metric Unit"] == "ns" else 1.0)
    agg[name].append(us)
    if "-v" in sys.argv:
        print(f"{name:26s} {us:8.1f} us grid {d['Grid Size']:>14s} block {d['Block Size']}")
tot = sum(sum(v) for v in agg.values())
for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{n:26s} n={len(v):4d} total={sum(v)/1e3:8.3f} ms mean={sum(v)/len(v):8.1f} us share={100*sum(v)/tot:5.1f}%")
print(f"total {tot/1e3:.3f} ms over {sum(len(v) for v in agg.values())} launches")
