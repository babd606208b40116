#!/bin/bash
# ncu captures of the small-R two-step kernel (c2, R=8 per GPU) and the ELL step kernel (c2 via CSR)
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/probe2
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_dos_green.py -q -x > $OUT/pytest_dos.log 2>&1; echo "exit $?" >> $OUT/pytest_dos.log
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpm_step2_tma -s 20 -c 1 \
    -o $OUT/small_c2 $B --config c2 --r-per-gpu 8 > $OUT/small_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpm_ell_step -s 5 -c 1 \
    -o $OUT/ell_c2 $B --config c2 --format csr > $OUT/ell_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/launches_small_c2.csv \
    $B --config c2 --r-per-gpu 8 > /dev/null 2>&1
ls -la $OUT
