#!/bin/bash
# KPM_COMM_IPC pass: IPC tests, the bench row-partition test, c5 rows at world 1 (IPC vs NCCL halo) and 2 ranks
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ipc.py tests/test_gpu_multirank.py -x -q > $OUT/pytest.log 2>&1; echo "rc $?" >> $OUT/pytest.log
timeout 600 python bench.py --config c5 --partition rows --halo ipc --steps 2 --warmup 3 --no-cpu-baseline > $OUT/c5_rows1_ipc.json 2> $OUT/c5_rows1_ipc.err
timeout 600 python bench.py --config c5 --partition rows --halo nccl --steps 2 --warmup 3 --no-cpu-baseline > $OUT/c5_rows1_nccl.json 2> $OUT/c5_rows1_nccl.err
timeout 900 python bench.py --gpus 2 --config c5 --partition rows --halo ipc --steps 2 --warmup 3 --no-cpu-baseline > $OUT/c5_rows2_ipc.json 2> $OUT/c5_rows2_ipc.err
ls -la $OUT
