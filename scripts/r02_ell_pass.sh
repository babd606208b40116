#!/bin/bash
# ELL (CSR input) bench lines and profiles after the row-major layout / evict-last changes
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "csr or ell or Ell or ELL" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
timeout 900 python bench.py --config c2 --format csr --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_c2_csr.json 2> $OUT/c2.err
timeout 900 python bench.py --config c3 --format csr --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_csr.json 2> $OUT/c3.err
KEEP_REP=none bash scripts/profile_r02.sh $1/prof c2_csr c3_csr
