#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/probe4
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dos_green.py tests/test_gpu_parity.py -q -x -k "dos or green or first or local or two_step or tma" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py > $OUT/sanitize_$tool.log 2>&1
  echo "exit $?" >> $OUT/sanitize_$tool.log
done
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
for c in c5 c3 c4 c2; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:first -c 1 --csv --log-file $OUT/first_$c.csv $B --config $c > /dev/null 2>&1
done
timeout 300 python bench.py --config c2 --r-per-gpu 8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --plan no_two_step=1 > $OUT/bench_c2r8_single.json 2>&1
timeout 300 python bench.py --config c2 --r-per-gpu 8 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/bench_c2r8.json 2>&1
ls -la $OUT
