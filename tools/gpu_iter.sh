#!/bin/bash
# Quick GPU iteration (on the box): parity tests, then a short bench with the
# kernel-level numbers.   tools/gpu_iter.sh [pytest -k expr]
mkdir -p gpurun_out
if [ -n "$1" ]; then K="-k $1"; else K=""; fi
timeout 900 python -m pytest tests -m gpu -x -q $K > gpurun_out/gpu_tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?"; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print("MP/s %.1f  ms/step %.3f  e2e %s" % (d["value"], d["ms_per_step"], d.get("e2e", {}).get("value")))
ro = d["roofline_other"]
for k, v in (("render_fwd_isolated", ro["render_fwd_isolated"]), ("render_bwd_pixels_isolated", d["roofline"])):
    print("%-28s %.1f us  frac %.3f" % (k, v["ms_per_launch"] * 1e3, v["frac"]))
ins = ro["render_bwd_pixels_in_step"]
print("bwd in-step frac %.3f  %.1f us active of %.1f per step; p10/50/90 %s" % (ins["frac"], ins.get("ms_active_per_step", 0) * 1e3, d["ms_per_step"] * 1e3, d.get("ms_per_step_p10_p50_p90")))
if "single_view" in d: print("single view (config1) MP/s %.1f" % d["single_view"]["value"])
if "scaling_budget" in d: print("scaling budget " + "  ".join("k=%s share %.3f ms + AR %.3f -> %.2fx" % (k[1:], v["ms_share"], v["ms_allreduce_model"], v["projected_speedup"]) for k, v in d["scaling_budget"].items() if k.startswith("k")))
if "tracking" in d: print("tracking it/s %.1f" % d["tracking"]["value"])
if "mapping_ssim" in d: print("mapping+SSIM MP/s %.1f" % d["mapping_ssim"]["value"])
if "optimizer" in d: print("optimizer %.1f us  %.0f GB/s" % (d["optimizer"]["ms"] * 1e3, d["optimizer"]["achieved_gbs"]))
if "seeding" in d: print("seeding %.1f us  accepted %d" % (d["seeding"]["ms"] * 1e3, d["seeding"]["accepted"]))
PY
