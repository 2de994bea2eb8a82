"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

    make -C oracle && python oracle/make_golden.py

Each fixture stores a graph (the reference Graph's out-CSR and fingerprint)
together with outputs of the reference's own public API on it:
propagation_sweep, cpi_run (three windows), pagerank, preprocess, query,
query_na, exact_rwr, cpi_partition.  The graphs come from the reference's
generate_random_graph (graph.cpp:166-205) for all three dangling policies plus
an R-MAT scale-10 graph built by the reference Graph constructor from an edge
list drawn here with numpy (seeded).  Run only in the build container, where
/root/reference exists; the fixtures are committed and travel with the repo.
"""
from __future__ import annotations

import os
import zlib
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
C, EPS, S, T = 0.15, 1e-9, 5, 10


def rmat_edges(scale, ef, seed, a=0.57, b=0.19, c=0.19):
    rng = np.random.default_rng(seed)
    m = ef << scale
    u = np.zeros(m, np.int64)
    v = np.zeros(m, np.int64)
    for lvl in range(scale):
        r = rng.random(m)
        bit = 1 << (scale - 1 - lvl)
        right = (r >= a) & (r < a + b) | (r >= a + b + c)
        down = r >= a + b
        u |= np.where(down, bit, 0)
        v |= np.where(right, bit, 0)
    keep = u != v
    return u[keep].astype(np.uint32), v[keep].astype(np.uint32)


def emit(name, g, policy, ref_seed_list):
    n = g.n
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    x = rng.random(n)
    seeds = np.asarray(ref_seed_list, np.uint32)
    rec = dict(n=np.uint32(n), policy=np.int32(policy), fingerprint=np.uint64(g.fingerprint),
               out_offsets=g.out_offsets, out_targets=g.out_targets, dangling=g.dangling,
               c=C, eps=EPS, S=np.uint32(S), T=np.uint32(T), seeds=seeds)
    rec["sweep_x"] = x
    rec["sweep_y"] = g.sweep(x, C)
    pr, it, conv, res = g.cpi_run(None, C, EPS)
    rec["pagerank"], rec["pagerank_iters"], rec["pagerank_conv"], rec["pagerank_res"] = pr, it, conv, res
    st = g.preprocess(C, EPS, T)
    rec["stranger"] = st
    rec["query"] = np.stack([g.query(st, C, EPS, T, int(s), S) for s in seeds])
    rec["query_na"] = np.stack([g.query_na(int(s), S, T, C, EPS) for s in seeds])
    rec["exact_rwr"] = np.stack([g.exact_rwr(int(s), C, EPS) for s in seeds])
    rec["partition"] = g.cpi_partition([int(seeds[0])], C, EPS, [S, T])
    win = []
    for (lo, hi) in [(0, 0), (2, 7), (3, None)]:
        sc, it, conv, res = g.cpi_run([int(seeds[1])], C, EPS, lo, hi)
        win.append((sc, it, conv, res))
    rec["win_scores"] = np.stack([w[0] for w in win])
    rec["win_iters"] = np.array([w[1] for w in win], np.uint32)
    rec["win_conv"] = np.array([w[2] for w in win], np.int32)
    rec["win_res"] = np.array([w[3] for w in win], np.float64)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **rec)
    print(name, "n", n, "m", g.m, "pagerank iters", rec["pagerank_iters"])


def main():
    os.makedirs(OUT, exist_ok=True)
    ref = Reference()
    for pol, pname in enumerate(["selfloop", "uniform", "drop"]):
        g = ref.graph_random(200, 1200, 88, pname)
        emit(f"random200_{pname}", g, pol, [0, 7, 31, 199])
    u, v = rmat_edges(10, 16, 2024)
    for pol, pname in enumerate(["selfloop", "uniform", "drop"]):
        g = ref.graph_from_edges(1 << 10, u, v, pname)
        nd = set(int(d) for d in g.dangling)
        seeds = [s for s in range(0, 1024, 37) if s not in nd][:6]
        emit(f"rmat10_{pname}", g, pol, seeds)


if __name__ == "__main__":
    main()
