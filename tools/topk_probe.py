"""Times the device top-k on one C2 query batch (tools/ launch-list probe)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import bench
import paper_1708_02574_b200 as P
g = bench.build_graph("c2")
art = P.preprocess(g, 0.15, 1e-9, 10)
seeds = P.sample_seeds(g, 64, 1)
out = torch.empty((32, g.node_count()), dtype=torch.float64, device="cuda")
P.query_batch(g, art, seeds[:32], 5, out=out)
torch.cuda.synchronize()
for k in (10, 100):
    for _ in range(2):
        ids, vals = P.top_k(g, out, k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        ids, vals = P.top_k(g, out, k)
    torch.cuda.synchronize()
    print("k", k, "top_k ms", (time.perf_counter() - t0) / 10 * 1e3)
t0 = time.perf_counter()
for _ in range(5):
    P.query_batch_topk(g, art, seeds[:32], 5, 10)
print("query_batch_topk ms", (time.perf_counter() - t0) / 5 * 1e3)
t0 = time.perf_counter()
for _ in range(5):
    P.query_batch(g, art, seeds[:32], 5, out=out)
torch.cuda.synchronize()
print("query_batch ms", (time.perf_counter() - t0) / 5 * 1e3)

seeds = P.sample_seeds(g, 1024, 1)
times = []
for i in range(32):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P.query_batch_topk(g, art, seeds[i * 32:(i + 1) * 32], 5, 10)
    times.append((time.perf_counter() - t0) * 1e3)
print("per-batch query_batch_topk ms", [round(t, 2) for t in times])
