#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for cfg in c4 c5; do for v in nopers pers nopers pers; do
  PYTHONPATH=tools/bin/$v timeout -s KILL 400 python tools/ab_sweeps.py --config $cfg --no-queries --reps 1 --tag $v 2>&1 | grep tag
done; done
