#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tma_march or box_kernel or two_step" > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
for tl in 0 64; do
  env KPM_TMA_TL=$tl timeout 600 python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/c4_tl${tl}.json 2> $OUT/c4_tl${tl}.err
done
timeout 900 python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/c5.json 2> $OUT/c5.err
ls $OUT
