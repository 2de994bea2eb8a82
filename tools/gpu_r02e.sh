#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in norank rank norank rank; do
  PYTHONPATH=tools/bin/$v timeout 300 python tools/ab_sweeps.py --config c4 --batches 2 --tag $v >> gpurun_out/ab4.jsonl 2>> gpurun_out/ab4.err
done
cat gpurun_out/ab4.jsonl
timeout 900 python -m pytest tests/test_large_configs.py tests/test_gpu_parity.py tests/test_edge_cases.py tests/test_partition.py -q -x -p no:cacheprovider > gpurun_out/pytest_e.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_e.log
