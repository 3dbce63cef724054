#!/bin/bash
# On the GPU box: bench line, ncu launch list of the bench command, full ncu
# captures of the two compositing kernels and the top binning kernel.
#   tools/make_profiles.sh <round-tag>
set -u
tag=${1:-r01}
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-tracking --no-e2e"
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
timeout 300 $B > gpurun_out/${tag}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv $B > gpurun_out/${tag}_ncu_list.log 2>&1
echo "launch list rc=$?"
for k in k_bwd_pixels k_render_fwd; do
  timeout 400 tools/ncu_full.sh ${tag}_$k $k --reps 6; echo "$k rc=$?"
done
SKIP=8 timeout 400 tools/ncu_full.sh ${tag}_k_rs_downsweep k_rs_downsweep --reps 3; echo "rs rc=$?"
