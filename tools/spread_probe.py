import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import numpy as np
import paper_1708_02574_b200 as P
from oracle import Oracle
o = Oracle()
bad = 0
for scale, seed in ((16, 3), (15, 5)):
    g = P.generate_rmat(scale, 16, rng_seed=seed, policy="uniform")
    art = P.preprocess(g, 0.15, 1e-9, 10)
    want = o.preprocess(g, 0.15, 1e-9, 10)
    seeds = P.sample_seeds(g, 64, 1)
    out = P.query_batch(g, art, seeds, 5)
    for k in range(0, 64, 7):
        ref = o.query(g, want, 0.15, 1e-9, 10, int(seeds[k]), 5)
        d = np.abs(out[k] - ref)
        print(scale, k, d.max(), d.sum())
        bad += d.max() > 1e-12
print("BAD" if bad else "ok")
