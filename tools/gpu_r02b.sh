#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in c4 c2; do
  for v in base S SG SGL; do
    PYTHONPATH=tools/bin/$v timeout 300 python tools/ab_sweeps.py --config $cfg --tag $v >> gpurun_out/ab_$cfg.jsonl 2>> gpurun_out/ab.err
  done
done
echo "ab done"; cat gpurun_out/ab_c4.jsonl gpurun_out/ab_c2.jsonl
timeout 1500 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider > gpurun_out/pytest_b.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_b.log; grep -E "FAILED|Error" gpurun_out/pytest_b.log | head -20
bash tools/profile_c4.sh c4
