"""Batched queries on a row-partitioned graph (graphs beyond one GPU):
tpa_group_query_batch runs K3 on every partition's rows of the padded share
layout, exchanging spans, frontier words and exact residual limbs per sweep.
Against the whole-graph query_batch: bit for bit under SelfLoop / Drop, within
the parity bar under Uniform (its spread comes from per-block dangling sums,
grouped differently by a partition); query_na; host and device outputs; the
reference's error behaviour (tpa.cpp:61-86)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import assert_close

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1708_02574_b200")
C, EPS, S, T = 0.15, 1e-9, 5, 10


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("G", [2, 3])
@pytest.mark.parametrize("policy", ["selfloop", "drop", "uniform"])
def test_partitioned_query_batch_equals_whole_graph(G, policy):
    g = P.generate_rmat(13, 16, rng_seed=12, policy=policy)  # rows up to ~2k in-degree: segments
    art = P.preprocess(g, C, EPS, T)
    grp = P.PartitionGroup(g, [0] * G)
    try:
        for B in (10, 32, 40):  # batch widths 16 / 32 / 64
            seeds = P.sample_seeds(g, B, B)
            want = P.query_batch(g, art, seeds, S)
            got = grp.query_batch(art, seeds, S)
            if policy == "uniform":
                assert_close(got, want, what=f"G={G} B={B}")
            else:
                assert np.array_equal(got, want), (G, B, float(np.abs(got - want).max()))
        prm = P.TpaParams(S, T, C, EPS)
        seeds = P.sample_seeds(g, 24, 7)
        want_na = np.stack([P.query_na(g, int(s), prm) for s in seeds])
        assert_close(grp.query_batch(None, seeds, S, na=True, params=prm), want_na, what="query_na")
    finally:
        grp.close()


def test_partitioned_query_batch_device_output_and_errors():
    import torch
    g = P.generate_rmat(12, 16, rng_seed=3)
    art = P.preprocess(g, C, EPS, T)
    grp = P.PartitionGroup(g, [0, 0])
    try:
        seeds = P.sample_seeds(g, 32, 1)
        out = torch.empty((32, g.node_count()), dtype=torch.float64, device="cuda")
        grp.query_batch(art, seeds, S, out=out)
        assert np.array_equal(out.cpu().numpy(), P.query_batch(g, art, seeds, S))
        stale = P.StrangerArtifact(art.stranger_scores, art.graph_fingerprint ^ 1, C, EPS, T)
        with pytest.raises(RuntimeError, match="fingerprint"):
            grp.query_batch(stale, seeds, S)
        with pytest.raises(ValueError):
            grp.query_batch(art, seeds, T)  # S must be < T
        with pytest.raises(IndexError):
            grp.query_batch(art, np.array([g.node_count()], np.uint32), S)
    finally:
        grp.close()
