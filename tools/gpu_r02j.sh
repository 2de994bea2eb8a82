#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in c2 c4; do for v in u16b8 u32b6 u32b5 u16b6 u16b8; do
  PYTHONPATH=tools/bin/$v timeout -s KILL 300 python tools/ab_sweeps.py --config $cfg --batches 4 --tag $v 2>&1 | grep tag
done; done
