"""Stall reasons of an ncu capture per SASS instruction class and region.
    ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv
    python tools/sass_stalls.py s.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
rows = rows[2:]
reasons = [(i, x) for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
ninst = 0
for r in rows:
    s = r[1].strip()
    op = (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0]
    ninst += int(r[5])
    for i, name in reasons:
        v = int(r[i] or 0)
        tot[name] += v
        byop[op][name] += v
T = sum(tot.values())
print("warp instructions %.2fM, stall samples %d" % (ninst / 1e6, T))
for name, v in tot.most_common():
    if v:
        top = sorted(((byop[o][name], o) for o in byop), reverse=True)[:5]
        print("%-24s %5.1f%%   %s" % (name, 100 * v / T, ", ".join("%s %.1f%%" % (o, 100 * c / T) for c, o in top)))
