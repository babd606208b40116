#!/bin/bash
# One GPU pass: bench every config, ncu launch metrics of the step kernels, full ncu of c3's step.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
for c in c1 c2 c3 c4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
for c in c2 c3 c4 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:kpm_step -s 4 -c 12 --csv --log-file $OUT/launches_$c.csv \
    python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpm_step_tma -s 10 -c 1 -o $OUT/prof_c3 \
  python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $OUT/ncu_c3.log 2>&1
ls -la $OUT
