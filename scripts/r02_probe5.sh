#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/probe5
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpm_step_tri -s 3 -c 1 -o $OUT/tri_c4 $B --config c4 > $OUT/tri_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpm_step_tri -s 3 -c 1 -o $OUT/tri_c2 $B --config c2 > $OUT/tri_c2.log 2>&1
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c5.json 2>$OUT/bench_c5.err
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --plan no_zorder=1 > $OUT/bench_c5_rowmajor.json 2>$OUT/bench_c5_rowmajor.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c3.json 2>$OUT/bench_c3.err
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --plan no_zorder=1 > $OUT/bench_c3_rowmajor.json 2>$OUT/bench_c3_rowmajor.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:kpm_step3_tma -s 4 -c 4 --csv --log-file $OUT/dram_c3.csv $B --config c3 > /dev/null 2>&1
ls -la $OUT
