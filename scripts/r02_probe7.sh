#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/probe7
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py > $OUT/r02_sanitize_$tool.log 2>&1
  echo "exit $?" >> $OUT/r02_sanitize_$tool.log
done
bash scripts/ab.sh probe7/ab "--config c2 --r-per-gpu 8 --steps 10 --warmup 3" "--config c2 --r-per-gpu 8 --steps 10 --warmup 3 --plan halo_warp=1"
