#!/bin/bash
# Parity of the KS-step kernel, then c2/c4 timings for its variants (device time only).
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "multi_step or tma_march or two_step" > $OUT/pytest.log 2>&1
tail -3 $OUT/pytest.log
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
for c in c2 c4; do
  for v in ${VARIANTS:-"KPM_NO_TMAK=1" "KPM_TMAK_KS=3"}; do
    env $v timeout 300 $B --config $c > $OUT/b_${c}_${v}.json 2> $OUT/b_${c}_${v}.err
    python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[1], d['ms_per_step'], round(d['roofline']['achieved']), d['roofline']['kernel'][:22])" $OUT/b_${c}_${v}.json 2>&1 | tail -1
  done
done
