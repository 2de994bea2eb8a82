#!/bin/bash
# ncu --set full of the last (dense, fused-combine) B = 32 sweep of one C4 query batch
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFG=${1:-c4}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_mm_fused" -s 2 -c 1 \
    -o gpurun_out/prof_${CFG}_sweep4 -f python tools/profile_step.py --config $CFG --batches 1 > gpurun_out/ncu_${CFG}_sweep4.log 2>&1
echo "sweep4 full rc $?"
python tools/ncu_summary.py gpurun_out/prof_${CFG}_sweep4.ncu-rep | tee gpurun_out/prof_${CFG}_sweep4.txt
