"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
data = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[key] or 0) for d in data)
for i, d in enumerate(sorted(data, key=lambda d: -float(d[key] or 0))[:n]):
    print(f"{float(d[key]):8.0f} {100*float(d[key])/tot:5.1f}%  {d['Address'][-5:]}  {d['Source'][:90]}")
