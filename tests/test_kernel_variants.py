"""The A/B kernel generations kept in the library (selected per process by
environment variables, read once at load) stay parity-correct: each runs a
small preprocess + query batch against the oracle in a fresh interpreter."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1708_02574_b200 as P
from oracle import Oracle
o = Oracle()
for policy in ("selfloop", "uniform"):
    g = P.generate_rmat(12, 16, rng_seed=7, policy=policy)
    art = P.preprocess(g, 0.15, 1e-9, 10)
    want = o.preprocess(g, 0.15, 1e-9, 10)
    assert np.abs(art.stranger_scores - want).max() <= 1e-12
    seeds = P.sample_seeds(g, 40, 3)
    for B in (1, 16, 32, 40):
        out = P.query_batch(g, art, seeds[:B], 5)
        for k in range(0, B, 13):
            ref = o.query(g, want, 0.15, 1e-9, 10, int(seeds[k]), 5)
            d = np.abs(out[k] - ref)
            assert d.max() <= 1e-12 and d.sum() <= 1e-9, (policy, B, k, d.max())
print("ok")
'''


@pytest.mark.gpu
@pytest.mark.parametrize("env", ["TPA_SPMM=2", "TPA_SPMM=3", "TPA_SPMM=4", "TPA_SPMV=1", "TPA_SPMV=3",
                                 "TPA_NO_SPARSE=1", "TPA_NO_WINDOW_LIST=1", "TPA_MM5_RB=16", "TPA_SPARSE_DIV=4",
                                 "TPA_NO_SEED_PUSH=1", "TPA_RELABEL=1", "TPA_MM5_RB=8", "TPA_MV_SHAPE=L", "TPA_MV_SHAPE=W"])
def test_variant_parity(env):
    k, v = env.split("=")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env={**os.environ, k: v},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


RELABEL_SCRIPT = r'''
import os, sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1708_02574_b200 as P
out = {{}}
for policy in ("selfloop", "drop", "uniform"):
    g = P.generate_rmat(13, 16, rng_seed=5, policy=policy)
    r = P.preprocess(g, 0.15, 1e-9, 10).stranger_scores
    pr = P.pagerank(g, P.CpiParams(0.15, 1e-9))
    np.save(os.path.join({tmp!r}, policy + "_" + os.environ.get("TPA_RELABEL", "0") + ".npy"), r)
    np.save(os.path.join({tmp!r}, policy + "_pr_" + os.environ.get("TPA_RELABEL", "0") + ".npy"),
            np.append(pr.scores, pr.iterations_run))
print("ok")
'''


@pytest.mark.gpu
def test_relabelled_twin_is_bitwise(tmp_path):
    """TPA_RELABEL=1 sweeps PageRank over the out-degree-relabelled twin of
    CSR(A^T) (tpa_relabel.cuh): each row keeps its old nonzero order, so the
    scores are bitwise the original's (SelfLoop, Drop); under Uniform the
    dangling-mass spread comes from differently grouped exact sums (last bits)."""
    for v in ("0", "1"):
        r = subprocess.run([sys.executable, "-c", RELABEL_SCRIPT.format(root=ROOT, tmp=str(tmp_path))],
                           env={**os.environ, "TPA_RELABEL": v}, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
    import numpy as np
    for policy in ("selfloop", "drop", "uniform"):
        for kind in ("", "pr_"):
            a = np.load(tmp_path / f"{policy}_{kind}0.npy")
            b = np.load(tmp_path / f"{policy}_{kind}1.npy")
            if policy == "uniform":
                assert a[-1] == b[-1] if kind else True
                assert np.abs(a - b).max() <= 1e-17
            else:
                assert np.array_equal(a, b), (policy, kind, np.abs(a - b).max())
