#!/bin/bash
# One GPU pass: GPU tests, bench lines for every config, then the profiling pass.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
for c in c2 c1 c3 c4 pd; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 python bench.py --config c5 --steps 2 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err
[ "${PROFILE:-1}" = 1 ] && bash scripts/profile_round.sh $1/prof ${PROFILE_CONFIGS:-c2 c3 c4 c5 pd}
ls -la $OUT
