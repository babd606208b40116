#!/bin/bash
# ncu --set full of one four-step launch on c4 for the in-tree library (A) and scratch/libkpm_B.so (B)
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/varncu; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e ${CFG:---config c4}"
K=${KREGEX:-kpm_step_quad}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $OUT/A $B > $OUT/A.log 2>&1
cp paper_1105_5481_b200/libkpm.so scratch/libkpm_A.so
cp scratch/libkpm_B.so paper_1105_5481_b200/libkpm.so
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $OUT/B $B > $OUT/B.log 2>&1
cp scratch/libkpm_A.so paper_1105_5481_b200/libkpm.so
for k in A B; do
  ncu -i $OUT/$k.ncu-rep --page raw --csv > $OUT/${k}_raw.csv 2>/dev/null
  ncu -i $OUT/$k.ncu-rep --page details --csv > $OUT/${k}_details.csv 2>/dev/null
  ncu -i $OUT/$k.ncu-rep --page source --csv --print-source sass > $OUT/${k}_sass.csv 2>/dev/null
  rm -f $OUT/$k.ncu-rep
done
