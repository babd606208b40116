#!/bin/bash
# ncu --set full of one four-step and one three-step launch on c4 (A/B of the kernels' limiters)
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/quadncu; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --config c4"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpm_step_quad -s 3 -c 1 -o $OUT/quad $B > $OUT/quad.log 2>&1
[ "${KS:-quad tri}" = quad ] || timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpm_step_tri -s 3 -c 1 -o $OUT/tri $B > $OUT/tri.log 2>&1
ls -la $OUT
for k in ${KS:-quad tri}; do
  ncu -i $OUT/$k.ncu-rep --page raw --csv > $OUT/${k}_raw.csv 2>/dev/null
  ncu -i $OUT/$k.ncu-rep --page details --csv > $OUT/${k}_details.csv 2>/dev/null
  ncu -i $OUT/$k.ncu-rep --page source --csv --print-source sass > $OUT/${k}_sass.csv 2>/dev/null
  rm -f $OUT/$k.ncu-rep
done
ls -la $OUT
