"""Golden fixtures for the full-size parity tests (C3, C4) -- TEST INFRASTRUCTURE.

    python oracle/make_large_fixtures.py c3 c4     # minutes per config (threads = 1)

Runs the UNMODIFIED reference library (oracle/_ref/librwrank_ref.so, compiled
from /root/reference/proj/src by oracle/Makefile) on the BASELINE.json config's
graph -- built by the reference's own Graph constructor (graph.cpp:53-91) from
the benchmark generator's edges (ref_capi.cpp ref_graph_rmat) or by the
reference's generate_random_graph (graph.cpp:166-205) for ER -- and records,
at threads = 1 (the reference's deterministic output):

* the graph identity (n, m, #dangling, FNV fingerprint);
* the stranger vector, pagerank(start_iter = T) == preprocess() (tpa.cpp:19-37):
  iterations_run, converged, residual, its L1 norm, its values at a fixed
  sample of node ids (seeded; plus the max-in-degree node and the query
  seeds), and its top-1000 (score desc, id asc -- metrics.cpp:25-36 order);
* four reference query() results (tpa.cpp:61-76; S = 5, T = 10): two seeds of
  the config's sample_seeds draw, one in-neighbour of the max-in-degree node
  (so the first sweep already reaches the longest CSR(A^T) row) and the last
  seed of the draw -- each as its L1 norm, its values at the sampled ids and
  its top-100.

The full vectors are 34-134 MB each, so only these samples are committed
(tests/golden/large/<config>.npz); the GPU tests compare the device results
element-wise against the C oracle at run time as well.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402

C, EPS, S, T = 0.15, 1e-9, 5, 10
CONFIGS = {
    "c3": ("er", dict(n=4194304, m=67108864), 4096, 1),
    "c4": ("rmat", dict(scale=24, edge_factor=32), 1024, 1),
}
N_SAMPLE = 20000


def topk(x, k):
    order = np.lexsort((np.arange(len(x)), -x))[:k]
    return order.astype(np.uint32), x[order]


def make(cfg: str, out_dir: str) -> str:
    kind, p, nq, seed = CONFIGS[cfg]
    ref = Reference()
    t0 = time.time()
    if kind == "rmat":
        g = ref.graph_rmat(p["scale"], p["edge_factor"], 0.57, 0.19, 0.19, seed=seed, threads=0)
    else:
        g = ref.graph_random(p["n"], p["m"], seed)
    print(f"[{cfg}] graph n={g.n} m={g.m} fp={g.fingerprint:#x} in {time.time() - t0:.1f}s", flush=True)
    draw = g.sample_seeds(nq, 1)
    hub, hub_deg = g.max_indeg()
    # an in-neighbour u != hub of the max-in-degree node (u -> hub is a real edge)
    src = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.out_offsets.astype(np.int64)))
    into = src[(g.out_targets == hub) & (src != hub)]
    hub_seed = int(into[len(into) // 2])
    qseeds = np.array([draw[0], draw[1], hub_seed, draw[-1]], np.uint32)
    rng = np.random.default_rng(12345)
    ids = np.unique(np.concatenate([rng.choice(g.n, N_SAMPLE, replace=False).astype(np.uint32),
                                    np.array([hub, 0, g.n - 1], np.uint32), qseeds]))
    t0 = time.time()
    stranger, iters, conv, res = g.cpi_run(None, C, EPS, start=T, threads=1)
    print(f"[{cfg}] pagerank start={T}: {iters} iterations, residual {res:.3e} in {time.time() - t0:.1f}s",
          flush=True)
    st_top_ids, st_top_vals = topk(stranger, 1000)
    rec = dict(n=g.n, m=g.m, fingerprint=np.uint64(g.fingerprint), n_dangling=len(g.dangling),
               hub=hub, hub_indeg=hub_deg, draw_seed=1, draw_count=nq, query_seeds=qseeds, ids=ids,
               pr_iterations=iters, pr_converged=conv, pr_residual=res, stranger_l1=np.abs(stranger).sum(),
               stranger_at=stranger[ids], stranger_top_ids=st_top_ids, stranger_top_vals=st_top_vals)
    fp = g.fingerprint
    q_at, q_l1, q_top_ids, q_top_vals = [], [], [], []
    for s in qseeds:
        t0 = time.time()
        q = g.query(stranger, C, EPS, T, int(s), S, fingerprint=fp, threads=1)
        print(f"[{cfg}] query seed {s}: {time.time() - t0:.1f}s", flush=True)
        q_at.append(q[ids])
        q_l1.append(np.abs(q).sum())
        i_, v_ = topk(q, 100)
        q_top_ids.append(i_)
        q_top_vals.append(v_)
    rec.update(query_at=np.array(q_at), query_l1=np.array(q_l1), query_top_ids=np.array(q_top_ids),
               query_top_vals=np.array(q_top_vals))
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, f"{cfg}.npz")
    np.savez_compressed(path, **rec)
    print(f"[{cfg}] wrote {path}", flush=True)
    return path


if __name__ == "__main__":
    out = os.path.join(ROOT, "tests", "golden", "large")
    for name in sys.argv[1:] or ["c3", "c4"]:
        make(name, out)
