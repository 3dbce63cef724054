"""Kernel durations of a command under ncu (cold, serialised; for ranking only).

    python tools/ncu_times.py "<kernel regex>" python tools/profile_view.py --reps 2
"""
import csv
import io
import subprocess
import sys

regex, cmd = sys.argv[1], sys.argv[2:]
out = subprocess.run(["ncu", "--metrics", "gpu__time_duration.sum", "--clock-control", "none", "--csv",
                      "-k", "regex:" + regex] + cmd, capture_output=True, text=True).stdout
rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 10]
rows = rows[next(i for i, r in enumerate(rows) if "Kernel Name" in r):]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
for r in rows[1:]:
    print(f"{float(r[vi].replace(',', '')) / 1000:9.2f} us  {r[ki].split('(')[0]}")
