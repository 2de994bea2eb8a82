#!/bin/bash
# K2h (hub shares in shared memory): parity tests, then per-sweep A/B at C2 / C4
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_edge_cases.py -m gpu -x -q 2>&1 | tail -5
for cfg in c2 c4; do for v in k2 product g8 g5 g4 k2 product; do
  if [ $v = product ]; then pp=""; else pp=tools/bin/$v; fi
  PYTHONPATH=$pp timeout -s KILL 400 python tools/ab_sweeps.py --config $cfg --no-queries --reps 2 --tag $v 2>&1 | grep tag
done; done | tee gpurun_out/r02m_ab.log
