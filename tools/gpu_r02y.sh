#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in ${@:-c2 c4}; do for v in base product q3 q6 q8 q16 d32 d64 d128q8 product; do
  if [ $v = product ]; then pp=""; else pp=tools/bin/$v; fi
  PYTHONPATH=$pp timeout -s KILL 900 python tools/ab_sweeps.py --config $cfg --no-queries --reps 2 --tag $v 2>&1 | grep tag | python -c "import sys,json; [print(d['config'], d['tag'], round(d['spmv_ms'],4)) for d in map(json.loads, sys.stdin)]"
done; done | tee gpurun_out/r02y_ab.log
