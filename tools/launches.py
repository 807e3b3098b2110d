"""Summarise an ncu launch-list CSV (gpu__time_duration per launch) by kernel for the last timed step."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; data = []
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr and len(r) == len(hdr): data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    n = d["Kernel Name"].split("(")[0][:44]
    a = agg.setdefault(n, [0, 0.0]); a[0] += 1; a[1] += float(d["Metric Value"])
tot = sum(v[1] for v in agg.values())
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:46s} {c:4d} launches {v/1e3/c:10.1f} us/launch  {100*v/tot:5.1f}%")
