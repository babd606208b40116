#!/bin/bash
# Round-2 closing pass: GPU tests, smoke, bench lines for every config (incl. CSR, small R, rows/IPC, the
# reference arm), then the profiling pass for the kernels changed late in the round.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
b() { name=$1; shift; timeout 1200 python bench.py "$@" > $OUT/bench_$name.json 2> $OUT/bench_$name.err; }
b c4 --config c4 --steps 3 --warmup 3
b c2 --config c2 --steps 10 --warmup 3
b c1 --config c1 --steps 10 --warmup 3
b c3 --config c3 --steps 3 --warmup 3
b c5 --config c5 --steps 2 --warmup 3
b pd --config pd --steps 5 --warmup 3
b c2_csr --config c2 --format csr --steps 5 --warmup 3 --no-cpu-baseline
b c3_csr --config c3 --format csr --steps 2 --warmup 3 --no-cpu-baseline
b c2_R8 --config c2 --r-per-gpu 8 --steps 10 --warmup 3 --no-cpu-baseline
b c5_rows_ipc --config c5 --partition rows --steps 2 --warmup 3 --no-cpu-baseline
b reference_c4 --impl reference --config c4 --steps 2 --warmup 1
[ "${PROFILE:-1}" = 1 ] && KEEP_REP=none bash scripts/profile_r02.sh $1/prof ${PROFILE_CONFIGS:-c2_R8 c3 c5 c2_csr c3_csr}
ls -la $OUT
