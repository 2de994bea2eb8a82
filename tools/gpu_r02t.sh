#!/bin/bash
# interleaved hot slots of the ranked share vector (L2 slice balance): SpMV A/B at C4 (and C5 with arg c5)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in ${@:-c4}; do for v in sp0 product sp12 sp20 sp0 product; do
  if [ $v = product ]; then pp=""; else pp=tools/bin/$v; fi
  PYTHONPATH=$pp timeout -s KILL 900 python tools/ab_sweeps.py --config $cfg --no-queries --reps 2 --tag $v 2>&1 | grep tag | python -c "import sys,json; [print(d['config'], d['tag'], round(d['spmv_ms'],4)) for d in map(json.loads, sys.stdin)]"
done; done | tee gpurun_out/r02t_ab.log
