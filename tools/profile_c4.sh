#!/bin/bash
# C4 (the bench headline) evidence: ncu --set full of the dense SpMM sweeps
# (batch 1, sweeps 3 and 4) and one PageRank SpMV sweep, plus the launch list
# of one bench step.  Outputs in gpurun_out/ (summaries go to profiles/).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFG=${1:-c4}
timeout 600 python tools/profile_step.py --config $CFG --batches 1 > gpurun_out/ps_$CFG.log 2>&1; echo "plain rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_mm_fused" -s 1 -c 2 \
    -o gpurun_out/prof_${CFG}_spmm -f python tools/profile_step.py --config $CFG --batches 1 > gpurun_out/ncu_${CFG}_spmm.log 2>&1
echo "spmm full rc $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_step_spmv2" -s 40 -c 1 \
    -o gpurun_out/prof_${CFG}_spmv -f python tools/profile_step.py --config $CFG --batches 1 > gpurun_out/ncu_${CFG}_spmv.log 2>&1
echo "spmv full rc $?"
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu --no-e2e"
timeout 900 env TPA_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ll_$CFG.log 2>&1; echo "launch list rc $?"
