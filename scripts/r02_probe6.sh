#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/probe6
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kpm_step_tri -s 3 -c 1 -o $OUT/tri_c4 $B --config c4 > $OUT/tri_c4.log 2>&1
bash scripts/ab.sh probe6/ab "--steps 3 --warmup 3 --plan tma_lanes=16" "--steps 3 --warmup 3 --plan tma_lanes=8"
