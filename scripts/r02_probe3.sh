#!/bin/bash
# tests of the expansions + first-step kernel; ncu of the first-step tile kernel (c5, c3); sanitizers
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/probe3
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dos_green.py tests/test_gpu_parity.py -q -x -k "dos or green or first or local" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpm_first_tile -c 1 \
    -o $OUT/first_c5 $B --config c5 > $OUT/first_c5.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:first -c 1 --csv --log-file $OUT/first_c3.csv $B --config c3 > /dev/null 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py > $OUT/sanitize_$tool.log 2>&1
  echo "exit $?" >> $OUT/sanitize_$tool.log
done
ls -la $OUT
