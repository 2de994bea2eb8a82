#!/bin/bash
# ranked [n][B] share layout (+ persisting-L2 window) for the fused B >= 16 sweeps: per-sweep A/B
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in c4 c2 c3; do for v in base r0 product base r0 product; do
  if [ $v = product ]; then pp=""; else pp=tools/bin/$v; fi
  PYTHONPATH=$pp timeout -s KILL 600 python tools/ab_sweeps.py --config $cfg --batches 6 --reps 2 --tag $v 2>&1 | grep tag | python -c "import sys,json; [print(d['config'], d['tag'], *(round(d[k],4) for k in ('spmv_ms','sweep1_ms','sweep2_ms','sweep3_ms','sweep4_ms'))) for d in map(json.loads, sys.stdin)]"
done; done | tee gpurun_out/r02r_ab.log
