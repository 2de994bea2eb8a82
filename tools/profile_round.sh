#!/bin/bash
# One GPU call: bench line, launch list of one bench step, full captures of
# an active PageRank sweep and the B = 32 family sweeps.  Outputs land in
# gpurun_out/ (copy summaries to profiles/).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
CMD="python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/ll_plain.json 2> gpurun_out/ll_plain.err && \
  TPA_PROFILE_RANGE=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $CMD > gpurun_out/ll_ncu.log 2>&1; echo "launch list rc $?"
python tools/profile_step.py > gpurun_out/ps_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_step_spmv2" -s 30 -c 1 \
      -o gpurun_out/prof_spmv python tools/profile_step.py > gpurun_out/ps_ncu1.log 2>&1; echo "spmv full rc $?"
python tools/profile_step.py > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_mm_fused" -s 0 -c 4 \
      -o gpurun_out/prof_spmm python tools/profile_step.py > gpurun_out/ps_ncu2.log 2>&1; echo "spmm full rc $?"
