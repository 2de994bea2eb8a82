#!/bin/bash
# One GPU call: bench line, launch list of one bench step, full captures of
# the two sweep kernels.  Outputs land in gpurun_out/ (copy summaries to profiles/).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/ll_plain.json 2> gpurun_out/ll_plain.err && \
  TPA_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ll_ncu.log 2>&1; echo "launch list rc $?"
python tools/profile_step.py > gpurun_out/ps_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_step_spmv2|k_mm_fused" -s 116 -c 5 \
      -o gpurun_out/prof_full python tools/profile_step.py > gpurun_out/ps_ncu.log 2>&1; echo "full rc $?"
