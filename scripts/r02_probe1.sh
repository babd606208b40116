#!/bin/bash
# Round-2 probe: ncu of the ELL step kernel (c2/c3 via CSR), small-R c2 timing + launch list.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/probe1
mkdir -p $OUT
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
for c in c2 c3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpm_ell_step -s 3 -c 1 \
    -o $OUT/ell_$c $B --config $c --format csr > $OUT/ell_$c.log 2>&1
  ncu -i $OUT/ell_$c.ncu-rep --page raw --csv > $OUT/ell_${c}_raw.csv 2>/dev/null
  ncu -i $OUT/ell_$c.ncu-rep --page details --csv > $OUT/ell_${c}_details.csv 2>/dev/null
done
timeout 300 python bench.py --config c2 --r-per-gpu 8 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c2_r8.json 2> $OUT/bench_c2_r8.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches_c2_r8.csv \
   $B --config c2 --r-per-gpu 8 > /dev/null 2>&1
nvidia-smi -q | head -40 > $OUT/smi.txt
ls -la $OUT
