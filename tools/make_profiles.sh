#!/bin/bash
# On the GPU box: bench line, ncu launch lists of the bench command and of a
# tracking iteration, full ncu captures of the compositing kernels and of the
# HBM / latency-bound stages, and the per-kernel HBM table.
#   tools/make_profiles.sh <round-tag>
set -u
tag=${1:-r02}
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --profile"
timeout 900 python bench.py --steps 30 --warmup 10 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"
timeout 300 $B > gpurun_out/${tag}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches.csv $B > gpurun_out/${tag}_ncu_list.log 2>&1
echo "launch list rc=$?"
python tools/launches.py gpurun_out/${tag}_launches.csv > gpurun_out/${tag}_launches_one_view.txt 2>&1
timeout 300 python tools/profile_track.py 2 > /dev/null 2>&1 && \
  timeout 300 python tools/ncu_times.py "." python tools/profile_track.py 2 > gpurun_out/${tag}_tracking_launches.txt 2>&1
echo "tracking list rc=$?"
for k in "k_bwd_pixels" "k_render_fwd" "^k_tile_sort_p$" "^k_emit$" "^k_project$" "k_bwd_gauss" "^k_bin_prep$" "^k_tile_counts$"; do
  n=$(echo $k | tr -d '^$')
  SKIP=${SKIP:-2} timeout 400 tools/ncu_full.sh ${tag}_$n "$k" --reps 3; echo "$n rc=$?"
  python tools/ncu_summary.py gpurun_out/prof_${tag}_$n.ncu-rep 30 > gpurun_out/sum_${tag}_$n.txt 2>&1
done
python tools/hbm_table.py gpurun_out/prof_${tag}_*.ncu-rep > gpurun_out/${tag}_hbm_table.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_debug_build.py -q > gpurun_out/${tag}_debug_build.log 2>&1
echo "debug build rc=$?"
