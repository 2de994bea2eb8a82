#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in c4 c2; do
  for v in nohot hot nohot hot; do
    PYTHONPATH=tools/bin/$v timeout 300 python tools/ab_sweeps.py --config $cfg --tag $v >> gpurun_out/ab3.jsonl 2>> gpurun_out/ab3.err
  done
done
cat gpurun_out/ab3.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_d.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_d.log
