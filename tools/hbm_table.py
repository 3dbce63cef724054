"""DRAM traffic and achieved HBM bandwidth per captured kernel (ncu --set full
reports), against MEASURED_PEAKS.json's copy bandwidth.
    python tools/hbm_table.py gpurun_out/prof_*.ncu-rep"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6528.4)
print("%-28s %10s %10s %10s %9s %7s %7s" % ("kernel", "us", "read MB", "write MB", "GB/s", "of HBM", "issue%"))
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        g = lambda k: float(v[h.index(k)].replace(",", ""))
        scale = lambda k: {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u[h.index(k)], 1.0)
        t = g("gpu__time_duration.sum") * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(
            u[h.index("gpu__time_duration.sum")], 1.0)
        rd = g("dram__bytes_read.sum") * scale("dram__bytes_read.sum")
        wr = g("dram__bytes_write.sum") * scale("dram__bytes_write.sum")
        gbs = (rd + wr) * 1e6 / (t * 1e-6) / 1e9
        name = v[h.index("Kernel Name")].split("(")[0].replace("void ", "")[:28]
        print("%-28s %10.1f %10.2f %10.2f %9.0f %6.1f%% %6.1f" % (name, t, rd, wr, gbs, 100 * gbs / peak,
                                                                g("smsp__issue_active.avg.pct_of_peak_sustained_active")))
