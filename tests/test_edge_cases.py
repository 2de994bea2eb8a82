"""Degenerate and extreme graphs through the GPU path, against the oracle:
single node, no edges at all, every node dangling, a hub row longer than the
SpMV tile (2,048 nnz) and the SpMM segment (512 nnz), a hub with a huge
out-degree (the sweep-1 push and push-marking), duplicate seeds in a batch,
seeds at the id extremes -- under all three dangling policies."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1708_02574_b200 as P
from conftest import assert_close

C, EPS, S, T = 0.15, 1e-9, 5, 10
POLICIES = ["selfloop", "uniform", "drop"]


def _check(oracle, g, seeds):
    art = P.preprocess(g, C, EPS, T)
    want = oracle.preprocess(g, C, EPS, T)
    assert_close(art.stranger_scores, want, what="stranger")
    q = P.query_batch(g, art, seeds, S)
    for k, s in enumerate(seeds):
        assert_close(q[k], oracle.query(g, want, C, EPS, T, int(s), S), what=f"seed {s}")
        assert_close(P.query(g, art, int(s), S), q[k], what=f"single {s}")
    pr = P.pagerank(g, P.CpiParams(C, EPS))
    opr = oracle.pagerank(g, C, EPS)
    assert_close(pr.scores, opr[0], what="pagerank")


@pytest.mark.gpu
@pytest.mark.parametrize("policy", POLICIES)
def test_single_node(oracle, policy):
    g = P.Graph(1, (np.zeros(0, np.uint32), np.zeros(0, np.uint32)), policy)
    _check(oracle, g, np.array([0], np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("policy", POLICIES)
def test_no_edges(oracle, policy):
    g = P.Graph(7, (np.zeros(0, np.uint32), np.zeros(0, np.uint32)), policy)
    _check(oracle, g, np.arange(7, dtype=np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("policy", POLICIES)
def test_hub_rows_beyond_tile_and_segment(oracle, policy):
    # node 0 receives 5,000 in-edges (a row longer than the SpMV tile and ten
    # SpMM segments) and sends 3,000 out-edges (the sweep-1 push / marking of
    # a hub seed); the rest is a sparse random graph with dangling nodes
    rng = np.random.default_rng(3)
    n = 6000
    src = [np.arange(1, 5001, dtype=np.uint32), np.zeros(3000, np.uint32)]
    dst = [np.zeros(5000, np.uint32), rng.choice(np.arange(1, n, dtype=np.uint32), 3000, replace=False)]
    r_src = rng.integers(1, n, 20000, dtype=np.uint32)
    r_dst = rng.integers(1, n, 20000, dtype=np.uint32)
    keep = r_src % 7 != 0  # sources = 0 mod 7 stay dangling unless hit above
    src.append(r_src[keep])
    dst.append(r_dst[keep])
    g = P.Graph(n, (np.concatenate(src), np.concatenate(dst)), policy)
    seeds = np.array([0, 1, 7, n - 1, 0, 4999, 5000, 5001] * 4, np.uint32)  # duplicates, extremes
    _check(oracle, g, seeds)


@pytest.mark.gpu
def test_every_node_dangling_but_one(oracle):
    # a single edge; every other node is dangling (Uniform spreads each sweep)
    for policy in POLICIES:
        g = P.Graph(50, [(3, 4)], policy)
        _check(oracle, g, np.array([3, 4, 0, 49], np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("policy", POLICIES)
def test_sweep_of_caller_vectors(oracle, policy):
    """propagation_sweep (graph.cpp:230-270) of arbitrary caller vectors: a
    dangling entry far above any CPI mass, x = ones over hundreds of dangling
    nodes (dangling mass >= 256), and signed entries -- the Uniform spread is a
    signed sum of the dangling entries (a clamped fixed-point total
    got these wrong)."""
    g = P.Graph(3, [(0, 1)], policy)  # nodes 1 and 2 dangling
    x = np.array([0.0, 100.0, 0.0])
    assert_close(P.propagation_sweep(g, x, C), oracle.sweep(g, x, C), max_abs=1e-13, what="x = 100 e_1")
    rng = np.random.default_rng(5)
    n = 2000
    src = rng.integers(0, n // 2, 6000, dtype=np.uint32)  # nodes >= n/2 dangling
    dst = rng.integers(0, n, 6000, dtype=np.uint32)
    g = P.Graph(n, (src, dst), policy)
    for x, what in ((np.ones(n), "ones"), (rng.normal(0.0, 50.0, n), "signed"),
                    (np.where(np.arange(n) % 2 == 0, 1e3, -1e3), "alternating")):
        want = oracle.sweep(g, x, C)
        # entries are O(1e3) here: the bar scales with them (relative 1e-15)
        bar = 1e-15 * max(1.0, np.abs(x).sum())
        assert_close(P.propagation_sweep(g, x, C), want, max_abs=bar, l1=bar * n, what=what)
