#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for v in notma tma; do PYTHONPATH=tools/bin/$v timeout -s KILL 200 python tools/save_q.py gpurun_out/q_$v.npz; done
python -c "
import numpy as np
a=np.load('gpurun_out/q_notma.npz'); b=np.load('gpurun_out/q_tma.npz')
for k in a: print(k, 'bitwise', np.array_equal(a[k], b[k]), 'maxdiff', float(np.abs(a[k]-b[k]).max()))"
for cfg in c2 c4; do for v in notma tma notma tma; do
  PYTHONPATH=tools/bin/$v timeout -s KILL 300 python tools/ab_sweeps.py --config $cfg --batches 4 --tag $v 2>&1 | grep tag
done; done
