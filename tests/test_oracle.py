"""Pins the CPU oracle (oracle/cpi_oracle.c) before anything is checked against it.

1. Bitwise against the committed golden fixtures (made by the unmodified
   reference, oracle/make_golden.py).
2. Bitwise against the reference library itself on fresh random graphs
   (skipped where oracle/_ref was not built).
3. The reference's own known-answer tests for the path (proj/tests/
   graph_test.cpp, cpi_test.cpp, tpa_test.cpp), restated against the oracle.
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

from conftest import GOLDEN, CsrGraph, golden_files, load_golden


@pytest.mark.parametrize("path", golden_files(), ids=lambda p: p.rsplit("/", 1)[-1])
def test_oracle_matches_golden_bitwise(oracle, path):
    rec = load_golden(path)
    g = CsrGraph(rec)
    c, eps, S, T = float(rec["c"]), float(rec["eps"]), int(rec["S"]), int(rec["T"])
    assert np.array_equal(oracle.sweep(g, rec["sweep_x"], c), rec["sweep_y"])
    pr, it, conv, res = oracle.pagerank(g, c, eps)
    assert np.array_equal(pr, rec["pagerank"])
    assert (it, conv, res) == (int(rec["pagerank_iters"]), bool(rec["pagerank_conv"]), float(rec["pagerank_res"]))
    st = oracle.preprocess(g, c, eps, T)
    assert np.array_equal(st, rec["stranger"])
    for k, s in enumerate(rec["seeds"]):
        assert np.array_equal(oracle.query(g, st, c, eps, T, int(s), S), rec["query"][k])
        assert np.array_equal(oracle.query(g, None, c, eps, T, int(s), S, na=True), rec["query_na"][k])
        assert np.array_equal(oracle.exact_rwr(g, int(s), c, eps), rec["exact_rwr"][k])
    assert np.array_equal(oracle.cpi_partition(g, [int(rec["seeds"][0])], c, eps, [S, T]), rec["partition"])
    for k, (lo, hi) in enumerate([(0, 0), (2, 7), (3, None)]):
        sc, it, conv, res = oracle.cpi_run(g, [int(rec["seeds"][1])], c, eps, lo, hi)
        assert np.array_equal(sc, rec["win_scores"][k])
        assert it == int(rec["win_iters"][k]) and conv == bool(rec["win_conv"][k]) and res == float(rec["win_res"][k])


@pytest.mark.parametrize("policy", ["selfloop", "uniform", "drop"])
def test_oracle_matches_reference_bitwise(oracle, reference, policy):
    for seed in range(3):
        g = reference.graph_random(150 + 50 * seed, 900, seed, policy)
        g._policy = policy
        x = np.random.default_rng(seed).random(g.n)
        assert np.array_equal(oracle.sweep(g, x, 0.15), g.sweep(x, 0.15))
        st = g.preprocess(0.15, 1e-9, 10)
        assert np.array_equal(oracle.preprocess(g, 0.15, 1e-9, 10), st)
        a = g.cpi_run([3, 9], 0.2, 1e-10, 1, 40)
        b = oracle.cpi_run(g, [3, 9], 0.2, 1e-10, 1, 40)
        assert np.array_equal(a[0], b[0]) and a[1:] == b[1:]
        for s in (0, 5, 17):
            assert np.array_equal(oracle.query(g, st, 0.15, 1e-9, 10, s, 5), g.query(st, 0.15, 1e-9, 10, s, 5))
        assert np.array_equal(oracle.cpi_partition(g, [4], 0.15, 1e-9, [2, 6, 11]),
                              g.cpi_partition([4], 0.15, 1e-9, [2, 6, 11]))


# --- the reference's known answers (proj/tests/*.cpp) ------------------------
class Tiny:
    def __init__(self, n, edges, policy):
        self.n = n
        edges = sorted(set(edges))
        has = {u for u, _ in edges}
        if policy == 0:
            edges = sorted(edges + [(u, u) for u in range(n) if u not in has])
        off = np.zeros(n + 1, np.uint64)
        for u, _ in edges:
            off[u + 1] += 1
        self.out_offsets = np.cumsum(off).astype(np.uint64)
        self.out_targets = np.array([v for _, v in edges], np.uint32)
        self.policy = policy


def test_two_cycle_sweep(oracle):
    # graph_test.cpp:131-137
    g = Tiny(2, [(0, 1), (1, 0)], 0)
    y = oracle.sweep(g, [0.15, 0.0], 0.15)
    assert y[0] == 0.0 and abs(y[1] - 0.1275) < 1e-15 * (1 + 0.1275)


def test_uniform_and_drop_spread(oracle):
    # graph_test.cpp:204-215
    y = oracle.sweep(Tiny(3, [(0, 1)], 1), [0.0, 0.9, 0.0], 0.15)
    assert np.allclose(y, 0.85 * 0.9 / 3.0, rtol=0, atol=1e-15)
    z = oracle.sweep(Tiny(3, [(0, 1)], 2), [0.0, 0.9, 0.0], 0.15)
    assert np.all(z == 0.0)


def test_convergence_iteration_count(oracle):
    # cpi_test.cpp:50-61
    expected = math.ceil(math.log(1e-9 / 0.15) / math.log(0.85))
    assert expected == 116
    _, it, conv, res = oracle.cpi_run(Tiny(2, [(0, 1), (1, 0)], 0), [0], 0.15, 1e-9)
    assert conv and it == 116 and res < 1e-9


def test_two_cycle_exact(oracle):
    # cpi_test.cpp:63-69
    r = oracle.exact_rwr(Tiny(2, [(0, 1), (1, 0)], 0), 0, 0.15, 1e-9)
    assert abs(r[0] - 1 / 1.85) < 1e-8 and abs(r[1] - 0.85 / 1.85) < 1e-8


def test_terminal_zero(oracle):
    # cpi_test.cpp:168-178
    sc, it, conv, res = oracle.cpi_run(Tiny(2, [(0, 1), (1, 0)], 0), [0], 0.15, 1e-9, 0, 0)
    assert it == 0 and not conv and sc[0] == 0.15 and sc[1] == 0.0 and res == 0.15


def test_neighbor_scale_factor_rationals(oracle):
    # tpa_test.cpp:40-50
    assert abs(oracle.neighbor_scale_factor(0.15, 5, 10) - 1419857 / 3200000) < 1e-12
    assert abs(oracle.neighbor_scale_factor(0.15, 5, 100000) - 1419857 / 1780143) < 1e-12
    assert oracle.neighbor_scale_factor(0.15, 5, 5) == 0.0
    assert oracle.neighbor_scale_factor(0.15, 5, 10) == 0.44370531249999995


def test_self_loop_query_is_unit(oracle):
    # tpa_test.cpp:76-81
    g = Tiny(1, [(0, 0)], 0)
    st = oracle.preprocess(g, 0.15, 1e-9, 10)
    r = oracle.query(g, st, 0.15, 1e-9, 10, 0, 5)
    assert abs(r[0] - 1.0) < 1e-6 * 2


def test_reference_side_generator_matches_the_product(reference):
    """The reference arm and the large fixtures build the benchmark graph with
    the reference's own Graph constructor from oracle/ref_capi.cpp's R-MAT
    restatement (no product code): same graph, fingerprint and seed draw as the
    product's generator (csrc/host_graph.cpp)."""
    import paper_1708_02574_b200 as P
    for scale, ef, policy in ((10, 16, "selfloop"), (13, 8, "uniform"), (12, 4, "drop")):
        g = P.generate_rmat(scale, ef, 0.57, 0.19, 0.19, rng_seed=3, policy=policy)
        rg = reference.graph_rmat(scale, ef, 0.57, 0.19, 0.19, seed=3, policy=policy)
        assert rg.fingerprint == g.fingerprint()
        assert np.array_equal(rg.out_offsets, g.out_offsets()) and np.array_equal(rg.out_targets, g.out_targets())
        assert np.array_equal(rg.sample_seeds(40, 9), P.sample_seeds(g, 40, 9))


def test_large_fixtures_are_consistent():
    """tests/golden/large/*.npz (oracle/make_large_fixtures.py): the reference's
    stranger vector and queries obey the SelfLoop closed forms."""
    import glob
    paths = sorted(glob.glob(os.path.join(GOLDEN, "large", "*.npz")))
    assert paths
    for p in paths:
        fx = dict(np.load(p))
        assert int(fx["pr_iterations"]) == 116 and bool(fx["pr_converged"])
        assert abs(float(fx["stranger_l1"]) - 0.85 ** 10) <= 1e-9 / 0.15
        nsf = (0.85 ** 5 - 0.85 ** 10) / (1 - 0.85 ** 5)
        mass = (1 + nsf) * (1 - 0.85 ** 5) + float(fx["stranger_l1"])
        assert np.all(np.abs(fx["query_l1"] - mass) <= 1e-9 / 0.15)
        assert np.all(np.diff(fx["stranger_top_vals"]) <= 0)
