#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_edge_cases.py -q -x -p no:cacheprovider > gpurun_out/pytest_f.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_f.log; grep -E "Error|assert" gpurun_out/pytest_f.log | head -10
for cfg in c2 c4; do for v in nopush push nopush push; do
  PYTHONPATH=tools/bin/$v timeout 300 python tools/ab_sweeps.py --config $cfg --batches 4 --tag $v 2>&1 | grep tag
done; done
