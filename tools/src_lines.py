"""Instructions executed and stall samples per CUDA source line of an ncu
--set full capture (needs -lineinfo and --import-source):
    python tools/src_lines.py X.ncu-rep [top]"""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
h, data = rows[hi], rows[hi + 1:]
ie, st = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


agg, stall, src = collections.Counter(), collections.Counter(), {}
for r in data:
    if len(r) < len(h):
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    agg[ln] += f(r[ie])
    stall[ln] += f(r[st])
    src[ln] = r[1]
tot, tots = sum(agg.values()) or 1, sum(stall.values()) or 1
print("total warp instructions %.2fM" % (tot / 1e6))
for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print("%5.1f%% inst %5.1f%% stall  L%-4d %s" % (100 * v / tot, 100 * stall[ln] / tots, ln, src[ln].strip()[:90]))
