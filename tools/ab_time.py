"""Times the four sweeps of one C2 query batch (CUDA events via the library's
profile hooks) for A/B kernel experiments: TPA_LIB=... python tools/ab_time.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02574_b200 as P  # noqa: E402
from paper_1708_02574_b200 import _native as N  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 32
g = bench.build_graph(cfg)
art = P.preprocess(g, 0.15, 1e-9, 10)
seeds = P.sample_seeds(g, batch * 8, 1)
out = torch.empty((batch, g.node_count()), dtype=torch.float64, device="cuda")
dg = g.device()
for k in range(2):
    P.query_batch(g, art, seeds[k * batch:(k + 1) * batch], 5, out=out)
torch.cuda.synchronize()
dg.profile(True)
P.preprocess(g, 0.15, 1e-9, 10)
c1, ms1 = dg.profile_read(1)
print("  spmv sweeps", c1, "avg ms", round(ms1 / max(c1, 1), 4), "preprocess sweeps total ms", round(ms1, 2))
for k in range(2, 8):
    P.query_batch(g, art, seeds[k * batch:(k + 1) * batch], 5, out=out)
cnt, ms = dg.profile_read(batch)
for i in range(1, 5):
    c_i, ms_i = dg.profile_read(batch, i)
    print("  sweep", i, "avg ms", round(ms_i / max(c_i, 1), 4))
dg.profile(False)
print(os.environ.get("TPA_LIB", "default"), cfg, "B", batch, "sweeps", cnt, "avg ms/sweep", round(ms / cnt, 4),
      "ms/batch", round(ms / 6, 3))
