#!/bin/bash
# c3 step-kernel time vs lanes per tile site (DRAM locality experiment).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tl in 8 16 32 64; do
  for box in 0 1; do
    env KPM_TMA_TL=$tl KPM_NO_TMA3=$box timeout 600 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $OUT/c3_tl${tl}_nobox${box}.json 2> $OUT/c3_tl${tl}_nobox${box}.err
  done
done
ls $OUT
