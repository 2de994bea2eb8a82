#!/bin/bash
# K2h shape sweep: groups x hub size (shared-memory carve-out vs L1), C2 / C4
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in c2 c4; do for v in k2 a b c d e f g h0 na k2; do
  PYTHONPATH=tools/bin/$v timeout -s KILL 400 python tools/ab_sweeps.py --config $cfg --no-queries --reps 2 --tag $v 2>&1 | grep tag | python -c "import sys,json; [print(d['config'], d['tag'], round(d['spmv_ms'],4)) for d in map(json.loads, sys.stdin)]"
done; done | tee gpurun_out/r02n_ab.log
