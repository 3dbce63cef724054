#!/bin/bash
# A/B of two versions of one source file on the GPU box:
#   tools/ab_file.sh <repo-relative source path> <old copy> <bench args...>
# builds libgs.so with the current file ("new") and with <old copy> ("old"),
# runs bench.py <bench args> for each and prints its summary line.
set -u
src=$1; old=$2; shift 2
args="$*"
cp "$src" /tmp/ab_new_src
for v in new old; do
  if [ $v = old ]; then cp "$old" "$src"; else cp /tmp/ab_new_src "$src"; fi
  python -m paper_2312_10070_b200._build --force > /dev/null 2>&1 || { echo "$v build failed"; continue; }
  timeout 900 python bench.py $args > gpurun_out/ab_$v.json 2> /dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); ro=d['roofline_other']; print('$v', 'MP/s %.1f ms %.3f fwd %.1f bwd %.1f' % (d['value'], d['ms_per_step'], ro['render_fwd_isolated']['ms_per_launch']*1e3, d['roofline']['ms_per_launch']*1e3), 'track', d.get('tracking', {}).get('value'))"
done
cp /tmp/ab_new_src "$src"
python -m paper_2312_10070_b200._build --force > /dev/null 2>&1
