#!/bin/bash
# K3 gather variants: per-sweep A/B at C4 / C2 (variants given as arguments; default base zr)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
VARS=${@:-base zr base zr}
for cfg in c4 c2; do for v in $VARS; do
  PYTHONPATH=tools/bin/$v timeout -s KILL 600 python tools/ab_sweeps.py --config $cfg --batches 6 --reps 2 --tag $v 2>&1 | grep tag | python -c "import sys,json; [print(d['config'], d['tag'], *(round(d[k],4) for k in ('spmv_ms','sweep1_ms','sweep2_ms','sweep3_ms','sweep4_ms'))) for d in map(json.loads, sys.stdin)]"
done; done | tee gpurun_out/r02q_ab.log
