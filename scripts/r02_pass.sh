#!/bin/bash
# Round-2 GPU pass: build, GPU tests, smoke, bench lines.  usage: r02_pass.sh <tag> [bench configs...]
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1; shift
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ "${TESTS:-1}" = 1 ]; then
  timeout 2400 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
fi
for spec in "$@"; do
  name=$(echo "$spec" | tr ' =,' '__-' | tr -d '-' )
  timeout 900 python bench.py $spec > $OUT/bench_$name.json 2> $OUT/bench_$name.err
done
ls -la $OUT
