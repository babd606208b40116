#!/bin/bash
# A/B of library builds: ab_libs.sh <tag> "<bench args>" lib1.so lib2.so ... (each copied over the in-tree
# libkpm.so in turn, the in-tree build restored at the end); prints ms per call of each run.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1; ARGS=$2; shift 2
mkdir -p $OUT
cp paper_1105_5481_b200/libkpm.so $OUT/libkpm_orig.so
for rep in 1 2; do
  for lib in "$@"; do
    cp $lib paper_1105_5481_b200/libkpm.so
    timeout 900 python bench.py $ARGS --no-cpu-baseline --no-e2e > $OUT/run.json 2> $OUT/run.err
    python -c "
import json,sys; d=json.loads(open('$OUT/run.json').read().strip().splitlines()[-1])
print('$lib', 'rep $rep', round(d['ms_per_step'],3), 'ms', d['clocks']['sm_mhz'], d['roofline']['kernel'][:24])" >> $OUT/summary.txt 2>&1
  done
done
cp $OUT/libkpm_orig.so paper_1105_5481_b200/libkpm.so
cat $OUT/summary.txt
