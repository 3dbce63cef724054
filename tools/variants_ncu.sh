#!/bin/bash
# Like variants.sh, but prints per-kernel duration / warp instructions /
# active cycles of one steady-state view (ncu, cold-cache, serialised).
#   tools/variants_ncu.sh "<flags>" ...      (KREGEX overrides the kernel regex)
mkdir -p gpurun_out
KR=${KREGEX:-"k_bwd_pixels|k_render_fwd|k_tile_sort|k_emit|k_tile_counts|k_bin_prep|k_project|k_bwd_gauss|k_loss"}
for v in "$@"; do
  GS_EXTRA_NVCC="$v" python -m paper_2312_10070_b200._build --force > /dev/null 2>&1 || { echo "$v: build failed"; continue; }
  echo "== $v"
  ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_active.avg --clock-control none --csv \
      -k "regex:$KR" python tools/profile_view.py --reps 2 2> /dev/null | python -c '
import csv, sys, collections
rows = [r for r in csv.reader(sys.stdin) if len(r) > 10]
rows = rows[next(i for i, r in enumerate(rows) if "Kernel Name" in r):]
h = rows[0]; ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = collections.OrderedDict()
for r in rows[1:]:
    d.setdefault((r[ii], r[ki].split("(")[0]), {})[r[mi]] = float(r[vi].replace(",", ""))
seen = {}
for (i, k), m in d.items(): seen[k] = m   # last launch of each kernel
for k, m in seen.items():
    print("%-40s %8.1f us  %8.2f M inst  %9.0f cyc" % (k[:40], m["gpu__time_duration.sum"] / 1e3, m["smsp__inst_executed.sum"] / 1e6, m["sm__cycles_active.avg"]))
'
done
