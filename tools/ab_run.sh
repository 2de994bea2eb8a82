#!/bin/bash
# Per-sweep A/B on the GPU box: ab_sweeps.py for every (config, variant) pair.
#   tools/ab_run.sh "c4 c2" "base product v1" [extra ab_sweeps.py flags, e.g. --no-queries]
# A variant is a build made by tools/ab_variants.py (tools/bin/<name>); "product" is the
# in-tree library.  Run under gpurun; prints one line per run and appends to gpurun_out/ab_run.log.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CFGS=${1:-c4}; VARS=${2:-product}; shift 2 || true
for cfg in $CFGS; do for v in $VARS; do
  if [ "$v" = product ]; then pp=""; else pp=tools/bin/$v; fi
  PYTHONPATH=$pp timeout -s KILL 900 python tools/ab_sweeps.py --config "$cfg" --reps 2 --tag "$v" "$@" 2>&1 | grep tag | \
    python -c "import sys,json; [print(d['config'], d['tag'], *(None if d[k] is None else round(d[k],4) for k in ('spmv_ms','sweep1_ms','sweep2_ms','sweep3_ms','sweep4_ms'))) for d in map(json.loads, sys.stdin)]"
done; done | tee -a gpurun_out/ab_run.log
