#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on the small parity cases of scripts/sanitize.py
# (produced profiles/r02_sanitize_*.log; compute-sanitizer was closed on the GPU pool later in round 2)
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/${1:-sanitize}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py > $OUT/r02_sanitize_$tool.log 2>&1
  echo "exit $?" >> $OUT/r02_sanitize_$tool.log
done
