"""Per-sweep kernel times of one config (experiments): PageRank preprocess +
query batches, per-kernel CUDA events (the library's profile mode).

    PYTHONPATH=tools/bin/VARIANT python tools/ab_sweeps.py --config c4 [--batches 4] [--reps 2]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.append(ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1708_02574_b200 as P  # noqa: E402  (the variant on PYTHONPATH, before bench adds ROOT)
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--batches", type=int, default=4)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--tag", default=os.environ.get("PYTHONPATH", "product"))
ap.add_argument("--no-queries", action="store_true", help="PageRank sweeps only (C5: no [B][n] output)")
a = ap.parse_args()
_, _, nq, B, seed = bench.CONFIGS[a.config]
g = bench.build_graph(a.config)
dg = g.device(0)
art = P.preprocess(g, 0.15, 1e-9, 10)
if a.no_queries:
    a.batches = 0
seeds = P.sample_seeds(g, B * max(a.batches, 1), 1)
out = torch.empty((B, g.node_count()), dtype=torch.float64, device="cuda") if a.batches else None
for k in range(a.batches):  # warm
    P.query_batch(g, art, seeds[k * B:(k + 1) * B], 5, out=out)
torch.cuda.synchronize()
dg.profile(True)
for _ in range(a.reps):
    P.preprocess(g, 0.15, 1e-9, 10)
    for k in range(a.batches):
        P.query_batch(g, art, seeds[k * B:(k + 1) * B], 5, out=out)
torch.cuda.synchronize()
res = {"tag": a.tag, "config": a.config, "lib": P._native.LIB_PATH}
c, ms = dg.profile_read(1)
res["spmv_ms"] = ms / max(c, 1)
for i in range(1, 5):
    c, ms = dg.profile_read(B, i)
    res[f"sweep{i}_ms"] = ms / max(c, 1) if c else None
dg.profile(False)
print(json.dumps(res), flush=True)
