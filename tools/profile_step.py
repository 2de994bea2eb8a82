"""Small fixed workload for ncu: C2 graph, one preprocess + two query batches.

    python tools/profile_step.py [--config c2] [--batch 32]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_1708_02574_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--batches", type=int, default=2)
a = ap.parse_args()
g = bench.build_graph(a.config)
art = P.preprocess(g, 0.15, 1e-9, 10)
seeds = P.sample_seeds(g, a.batch * a.batches, 1)
import torch  # noqa: E402
if g.node_count() * a.batch * 8 > (8 << 30):  # C5: scores in the idle iterate buffer (bench.py)
    tot = 0.0
    for k in range(a.batches):
        _, vals = P.query_batch_topk(g, art, seeds[k * a.batch:(k + 1) * a.batch], 5, 10)
        tot += float(vals.sum())
    print("ok", g.node_count(), g.edge_count(), tot)
else:
    out = torch.empty((a.batch, g.node_count()), dtype=torch.float64, device="cuda")
    for k in range(a.batches):
        P.query_batch(g, art, seeds[k * a.batch:(k + 1) * a.batch], 5, out=out)
    torch.cuda.synchronize()
    print("ok", g.node_count(), g.edge_count(), float(out.sum()))
