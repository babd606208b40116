#!/bin/bash
# four-step kernel: parity, then A/B against the three-step default (c4, c2)
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/quad
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/quad/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "four_step or three_step or two_step or tma" > gpurun_out/quad/pytest.log 2>&1
tail -5 gpurun_out/quad/pytest.log
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "four_step and peierls_anderson and 41" > gpurun_out/quad/memcheck.log 2>&1
tail -3 gpurun_out/quad/memcheck.log
bash scripts/ab.sh quad_ab "--config c4 --steps 3 --warmup 3" "--config c4 --steps 3 --warmup 3 --plan no_four_step=1" "--config c2 --steps 10 --warmup 3" "--config c2 --steps 10 --warmup 3 --plan no_four_step=1"
