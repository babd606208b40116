#!/bin/bash
# Profiling pass for profiles/: per config (1) the launch list of one bench step
# (gpu__time_duration, clock-control none), (2) steady-state DRAM bytes per step launch,
# (3) one `ncu --set full` capture of the step kernel.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1; shift
CONFIGS=${*:-c2 c3 c4 c5 pd}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
# the recursion-step kernels (2D two-step, 3D dense-box / generic march, dense DMMA GEMM)
K="kpm_step2_tma|kpm_step3_tma|kpm_step_tma|kpm_dense_step"
for c in $CONFIGS; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $OUT/launchlist_$c.csv $B --config $c > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"$K" -s 4 -c 8 --csv --log-file $OUT/dram_$c.csv $B --config $c > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 5 -c 1 \
    -o $OUT/full_$c $B --config $c > $OUT/full_$c.log 2>&1
done
# summaries on the box (the .ncu-rep files are too large to bring back, except one)
mkdir -p $OUT/profiles
cp profiles/traffic.json $OUT/profiles/ 2>/dev/null
python scripts/ncu_summary.py $OUT ${ROUND:-r01} $OUT/profiles
for c in $CONFIGS; do [ "$c" = "${KEEP_REP:-c3}" ] || rm -f $OUT/full_$c.ncu-rep; done
ls -la $OUT $OUT/profiles
