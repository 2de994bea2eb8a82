"""Smoke check of the B = 32 sweep kernels (dense sweeps on k_mm_tma) against
the oracle and, bitwise, against the B = 16 / 64 kernels (experiments)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1708_02574_b200 as P
from oracle import Oracle
o = Oracle()
for scale, policy in ((10, "selfloop"), (12, "drop"), (13, "selfloop"), (12, "uniform")):
    g = P.generate_rmat(scale, 16, rng_seed=5, policy=policy)
    art = P.preprocess(g, 0.15, 1e-9, 10)
    seeds = P.sample_seeds(g, 64, 3)
    q32 = P.query_batch(g, art, seeds[:32], 5)
    q64 = P.query_batch(g, art, seeds, 5)
    q16 = np.concatenate([P.query_batch(g, art, seeds[:16], 5), P.query_batch(g, art, seeds[16:32], 5)])
    same = np.array_equal(q32, q64[:32]) and np.array_equal(q32, q16)
    worst = 0.0
    for k in (0, 7, 31):
        w = o.query(g, art.stranger_scores, 0.15, 1e-9, 10, int(seeds[k]), 5)
        worst = max(worst, float(np.abs(q32[k] - w).max()))
    print(f"scale {scale} {policy}: bitwise vs B=16/64 {same}, max-abs vs oracle {worst:.2e}", flush=True)
    assert same and worst <= 1e-12
print("ok")
