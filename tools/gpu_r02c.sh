#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_partition_ipc.py -q -p no:cacheprovider > gpurun_out/pytest_ipc.log 2>&1; echo "ipc rc $?"; tail -3 gpurun_out/pytest_ipc.log
timeout 300 tools/bin/gather_micro > gpurun_out/gather_micro.txt 2>&1; echo "micro rc $?"
timeout 300 tools/bin/gather8_micro > gpurun_out/gather8_l2.txt 2>&1; echo "micro8 rc $?"
timeout 300 tools/bin/gather8_micro 16777216 > gpurun_out/gather8_c4.txt 2>&1; echo "micro8c4 rc $?"
cat gpurun_out/gather_micro.txt gpurun_out/gather8_l2.txt gpurun_out/gather8_c4.txt
for cfg in c4; do
  for v in base S SG SGL; do
    PYTHONPATH=tools/bin/$v timeout 300 python tools/ab_sweeps.py --config $cfg --tag $v >> gpurun_out/ab2_$cfg.jsonl 2>> gpurun_out/ab2.err
  done
done
cat gpurun_out/ab2_c4.jsonl
