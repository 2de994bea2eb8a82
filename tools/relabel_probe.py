"""Does relabelling nodes by out-degree (hubs first) speed up the sweeps?
Times PageRank SpMV sweeps and a query batch on C2 and on its isomorphic
relabelled copy (same work, different gather locality)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_1708_02574_b200 as P

def timing(g, label):
    art = P.preprocess(g, 0.15, 1e-9, 10)
    dg = g.device()
    seeds = P.sample_seeds(g, 32 * 8, 1)
    out = torch.empty((32, g.node_count()), dtype=torch.float64, device="cuda")
    for k in range(2):
        P.query_batch(g, art, seeds[k * 32:(k + 1) * 32], 5, out=out)
    torch.cuda.synchronize()
    dg.profile(True)
    P.preprocess(g, 0.15, 1e-9, 10)
    c1, ms1 = dg.profile_read(1)
    for k in range(2, 8):
        P.query_batch(g, art, seeds[k * 32:(k + 1) * 32], 5, out=out)
    torch.cuda.synchronize()
    per = [dg.profile_read(32, i) for i in range(1, 5)]
    dg.profile(False)
    print(label, "spmv ms", round(ms1 / c1, 4), "sweeps", [round(ms / max(c, 1), 4) for c, ms in per])

g = bench.build_graph("c2")
timing(g, "original")
n = g.node_count()
off = g.out_offsets().astype(np.int64)
deg = np.diff(off)
src = np.repeat(np.arange(n, dtype=np.uint32), deg)
dst = g.out_targets()
for name, key in (("outdeg", -deg), ("indeg", -np.bincount(dst, minlength=n))):
    order = np.argsort(key, kind="stable")       # new id -> old id
    perm = np.empty(n, np.uint32)
    perm[order] = np.arange(n, dtype=np.uint32)  # old id -> new id
    g2 = P.Graph(n, (perm[src], perm[dst]), "selfloop")
    timing(g2, "relabel-" + name)
