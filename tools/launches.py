"""Summarise an ncu --metrics gpu__time_duration.sum launch list (last view pass)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
idx = [i for i, d in enumerate(data) if "k_project" in d["Kernel Name"]][-1]
agg = collections.OrderedDict()
tot = 0.0
for d in [d for d in data[idx:] if d.get("Metric Name", "gpu__time_duration.sum") == "gpu__time_duration.sum"]:
    v = float(d["Metric Value"].replace(",", "")) / 1000.0
    k = d["Kernel Name"].split("(")[0].replace("void ", "")
    agg.setdefault(k, [0.0, 0])
    agg[k][0] += v
    agg[k][1] += 1
    tot += v
for k, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{v:9.1f} us  {100 * v / tot:5.1f}%  x{c:<3d} {k}")
print(f"{tot:9.1f} us  total (one view, serialised, cold caches)")
