#!/bin/bash
# A/B of the in-tree library against a variant build in scratch/libkpm_B.so: var.sh "<bench args>" ...
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash scripts/ab.sh var_A "$@" > /dev/null 2>&1
cp paper_1105_5481_b200/libkpm.so scratch/libkpm_A.so
cp scratch/libkpm_B.so paper_1105_5481_b200/libkpm.so
bash scripts/ab.sh var_B "$@" > /dev/null 2>&1
cp scratch/libkpm_A.so paper_1105_5481_b200/libkpm.so
bash scripts/ab.sh var_A2 "$@" > /dev/null 2>&1
echo A; cat gpurun_out/var_A/summary.txt; echo B; cat gpurun_out/var_B/summary.txt; echo A2; cat gpurun_out/var_A2/summary.txt
