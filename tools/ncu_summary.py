"""Print the key counters and the top stall lines of an ncu --set full report."""
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
pat = (r"^(gpu__time_duration.sum|sm__cycles_active.avg|sm__cycles_elapsed.avg|sm__warps_active.avg.pct_of_peak_sustained_active|"
       r"smsp__issue_active.avg.pct_of_peak_sustained_active|smsp__inst_executed.sum|launch__registers_per_thread|"
       r"launch__occupancy_limit_registers|sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active|"
       r"sm__inst_executed_pipe_(alu|fma|lsu|xu).avg.pct_of_peak_sustained_active|dram__bytes_(read|write).sum|"
       r"smsp__sass_thread_inst_executed_op_(ffma|fadd|fmul)_pred_on.sum|smsp__average_warps_issue_stalled_.*_per_issue_active.ratio)$")
for i, n in enumerate(h):
    if re.search(pat, n):
        try:
            if "stalled" in n and float(v[i]) < 0.1:
                continue
        except ValueError:
            pass
        print(f"  {n:78s} {v[i]:>16s} {u[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hh, data = rows[1], rows[2:]
i_s, i_src, i_ex = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Source"), hh.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in data)
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:top]:
    print(f"  {float(r[i_s]) / tot * 100:5.1f}%  ex={r[i_ex]:>9s}  {r[0][-5:]} {r[i_src][:90]}")
