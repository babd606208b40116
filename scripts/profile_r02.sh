#!/bin/bash
# Round-2 profiling pass for profiles/: per spec (1) the launch list of one bench step (gpu__time_duration,
# clock-control none), (2) DRAM bytes of steady-state step launches, (3) one `ncu --set full` capture of the
# step kernel; summaries via scripts/ncu_summary.py.  usage: profile_r02.sh <tag> [spec names]
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out/$1; shift
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
declare -A ARGS=( [c2]="--config c2" [c3]="--config c3" [c4]="--config c4" [c5]="--config c5" [pd]="--config pd"
                  [c2_csr]="--config c2 --format csr" [c3_csr]="--config c3 --format csr" [c2_R8]="--config c2 --r-per-gpu 8" )
declare -A RLOC=( [c2]=64 [c3]=128 [c4]=256 [c5]=32 [pd]=1792 [c2_csr]=64 [c3_csr]=128 [c2_R8]=8 )
NAMES=${*:-c2 c3 c4 c5 c2_csr c3_csr c2_R8}
python - "$OUT" $NAMES <<'PY'
import json, sys
R = {"c2": 64, "c3": 128, "c4": 256, "c5": 32, "pd": 1792, "c2_csr": 64, "c3_csr": 128, "c2_R8": 8}
json.dump({n: {"R_loc": R[n]} for n in sys.argv[2:]}, open(sys.argv[1] + "/specs.json", "w"))
PY
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e"
K="kpm_step_quad|kpm_step_tri|kpm_step2_tma|kpm_step3_tma|kpm_step_tma|kpm_ell_step|kpm_dense_step"
for c in $NAMES; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
    --log-file $OUT/launchlist_$c.csv $B ${ARGS[$c]} > /dev/null 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"$K" -s 4 -c 4 --csv --log-file $OUT/dram_$c.csv $B ${ARGS[$c]} > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 5 -c 1 \
    -o $OUT/full_$c $B ${ARGS[$c]} > $OUT/full_$c.log 2>&1
done
mkdir -p $OUT/profiles
cp profiles/traffic.json $OUT/profiles/ 2>/dev/null
python scripts/ncu_summary.py $OUT ${ROUND:-r02} $OUT/profiles
for c in $NAMES; do [ "$c" = "${KEEP_REP:-c4}" ] || rm -f $OUT/full_$c.ncu-rep; done
ls -la $OUT $OUT/profiles
