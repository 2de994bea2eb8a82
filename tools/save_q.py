"""Save a batch's scores (B = 32) for cross-variant bitwise comparison (experiments)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1708_02574_b200 as P
out = {}
for scale, policy in ((12, "uniform"), (13, "selfloop"), (14, "drop")):
    g = P.generate_rmat(scale, 16, rng_seed=9, policy=policy)
    art = P.preprocess(g, 0.15, 1e-9, 10)
    seeds = P.sample_seeds(g, 32, 4)
    out[f"{scale}{policy}"] = P.query_batch(g, art, seeds, 5)
np.savez(sys.argv[1], **out)
