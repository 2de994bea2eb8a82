#!/bin/bash
# ncu --set full of one PageRank sweep (K2) at C4
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFG=${1:-c4}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_step_spmv2" -s 40 -c 1 \
    -o gpurun_out/prof_${CFG}_spmv -f python tools/profile_step.py --config $CFG --batches 1 > gpurun_out/ncu_${CFG}_spmv.log 2>&1
echo "spmv full rc $?"
python tools/ncu_summary.py gpurun_out/prof_${CFG}_spmv.ncu-rep | tee gpurun_out/prof_${CFG}_spmv.txt
