#!/bin/bash
# Compile-time variant sweep on the GPU box: for each quoted flag set, rebuild
# libgs.so with GS_EXTRA_NVCC=<flags> and print the short bench summary.
#   tools/variants.sh "-DBWD_MINB=9" "-DBWD_MINB=10" ...
mkdir -p gpurun_out
for v in "$@"; do
  GS_EXTRA_NVCC="$v" python -m paper_2312_10070_b200._build --force > /dev/null 2>&1 || { echo "$v: build failed"; continue; }
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/v.json 2> /dev/null
  python - "$v" <<'PY'
import json, sys
d = json.load(open("gpurun_out/v.json"))
ro = d["roofline_other"]
print("%-28s MP/s %7.1f  ms %.3f  fwd %.1f us  bwd %.1f us  track %.0f it/s" % (
    sys.argv[1], d["value"], d["ms_per_step"], ro["render_fwd_isolated"]["ms_per_launch"] * 1e3,
    d["roofline"]["ms_per_launch"] * 1e3, d.get("tracking", {}).get("value", 0)))
PY
done
