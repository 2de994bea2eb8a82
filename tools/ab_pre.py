"""Times the PageRank preprocess sweeps (SpMV, B = 1) of a config for A/B
experiments, without the query batches: python tools/ab_pre.py c5"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1708_02574_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
g = bench.build_graph(cfg)
dg = g.device()
t0 = time.perf_counter()
P.preprocess(g, 0.15, 1e-9, 10)  # first call: builds the relabelled twin when it is on
t1 = time.perf_counter()
dg.profile(True)
for _ in range(2):
    art = P.preprocess(g, 0.15, 1e-9, 10)
c1, ms1 = dg.profile_read(1)
dg.profile(False)
print(f"{cfg} RELABEL={os.environ.get('TPA_RELABEL', 'auto')} first preprocess {t1 - t0:.2f}s; "
      f"spmv sweeps {c1} avg ms {ms1 / max(c1, 1):.4f}; device bytes {dg.device_bytes() / 1e9:.1f} GB; "
      f"stranger sum {art.stranger_scores.sum():.15f}")
