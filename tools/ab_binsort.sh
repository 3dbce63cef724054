#!/bin/bash
# A/B of two binsort.cu versions on the GPU box: tools/ab_binsort.sh <old.cu> "<bench args>"
# builds libgs.so with each version and prints the bench summary line of each.
set -u
old=$1; shift
args="$*"
cp paper_2312_10070_b200/csrc/binsort.cu /tmp/binsort_new.cu
for v in new old; do
  if [ $v = old ]; then cp "$old" paper_2312_10070_b200/csrc/binsort.cu; else cp /tmp/binsort_new.cu paper_2312_10070_b200/csrc/binsort.cu; fi
  python -m paper_2312_10070_b200._build --force > /dev/null 2>&1 || { echo "$v build failed"; continue; }
  timeout 900 python bench.py $args > gpurun_out/ab_$v.json 2> /dev/null
  python -c "import json,sys; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', 'MP/s %.1f ms %.3f' % (d['value'], d['ms_per_step']), 'track', d.get('tracking', {}).get('value'))"
done
cp /tmp/binsort_new.cu paper_2312_10070_b200/csrc/binsort.cu
