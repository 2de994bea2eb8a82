#!/bin/bash
# K3: rows without a live source skip their row-sum store: parity tests, per-sweep A/B
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_edge_cases.py tests/test_partition_queries.py tests/test_topk.py -m gpu -x -q 2>&1 | tail -4
for cfg in c4 c2 c3; do for v in base product base product; do
  if [ $v = product ]; then pp=""; else pp=tools/bin/$v; fi
  PYTHONPATH=$pp timeout -s KILL 600 python tools/ab_sweeps.py --config $cfg --batches 6 --reps 2 --tag $v 2>&1 | grep tag | python -c "import sys,json; [print(d['config'], d['tag'], *(round(d[k],4) for k in ('spmv_ms','sweep1_ms','sweep2_ms','sweep3_ms','sweep4_ms'))) for d in map(json.loads, sys.stdin)]"
done; done | tee gpurun_out/r02aa_ab.log
