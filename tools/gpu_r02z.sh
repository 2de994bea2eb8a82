#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
( timeout -s KILL 1500 python -m pytest tests -m gpu -x -q ) 2>&1 | tail -4
for cfg in c5 c3 c1; do for v in base product base product; do
  if [ $v = product ]; then pp=""; else pp=tools/bin/$v; fi
  PYTHONPATH=$pp timeout -s KILL 900 python tools/ab_sweeps.py --config $cfg --no-queries --reps 1 --tag $v 2>&1 | grep tag | python -c "import sys,json; [print(d['config'], d['tag'], round(d['spmv_ms'],4)) for d in map(json.loads, sys.stdin)]"
done; done | tee gpurun_out/r02z_ab.log
