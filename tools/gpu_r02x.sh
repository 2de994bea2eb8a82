#!/bin/bash
# K2 with several strided items per CTA: parity tests, then SpMV A/B
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_edge_cases.py tests/test_partition.py tests/test_partition_ipc.py -m gpu -x -q 2>&1 | tail -4
for cfg in ${@:-c2 c4}; do for v in base product p1 p4r p2 p8r base product; do
  if [ $v = product ]; then pp=""; else pp=tools/bin/$v; fi
  PYTHONPATH=$pp timeout -s KILL 900 python tools/ab_sweeps.py --config $cfg --no-queries --reps 2 --tag $v 2>&1 | grep tag | python -c "import sys,json; [print(d['config'], d['tag'], round(d['spmv_ms'],4)) for d in map(json.loads, sys.stdin)]"
done; done | tee gpurun_out/r02x_ab.log
