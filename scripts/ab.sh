#!/bin/bash
# A/B bench lines: ab.sh <tag> "<bench args>" ...  (each line: ms per call, launch us)
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1; shift
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
i=0
for spec in "$@"; do
  i=$((i+1))
  timeout 900 python bench.py $spec --no-cpu-baseline --no-e2e > $OUT/ab_$i.json 2> $OUT/ab_$i.err
  python -c "
import json,sys
d=json.loads(open('$OUT/ab_$i.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$spec', '|', round(d['ms_per_step'],3), 'ms', round(r['avg_launch_ms']*1000,2), 'us/launch', r['launches_per_step'], 'l/step', 'design', round(r['design_gbs']), 'sm', d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $OUT/summary.txt 2>&1
done
cat $OUT/summary.txt
