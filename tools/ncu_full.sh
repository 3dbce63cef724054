#!/bin/bash
# Usage (on the GPU box): tools/ncu_full.sh <tag> <kernel-regex> [profile_view args]
# One `ncu --set full` capture of one steady-state launch of each matching kernel.
set -e
tag=$1; shift; pat=$1; shift
mkdir -p gpurun_out
python tools/profile_view.py "$@" > gpurun_out/plain_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:$pat" -s ${SKIP:-3} -c 1 -o gpurun_out/prof_$tag \
    python tools/profile_view.py "$@" > gpurun_out/ncu_$tag.log 2>&1
