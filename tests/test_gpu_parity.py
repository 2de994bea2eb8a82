"""GPU parity: the sm_100a CPI path (through the C-ABI) against the oracle.

Bar (BASELINE.json north_star): fp64, per RWR vector max-abs <= 1e-12 and
L1 <= 1e-9; iteration counts equal.  Most cases are in fact bitwise (the
kernels keep the reference's rounding; see cpi_kernels.cuh) and the tests
record how many entries are bit-identical where that is asserted.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import CsrGraph, assert_close, golden_files, load_golden

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1708_02574_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def graph_from_golden(rec):
    n = int(rec["n"])
    off = rec["out_offsets"].astype(np.int64)
    src = np.repeat(np.arange(n, dtype=np.uint32), np.diff(off))
    g = P.Graph(n, (src, rec["out_targets"].astype(np.uint32)), int(rec["policy"]))
    assert g.fingerprint() == int(rec["fingerprint"])
    return g


# --- golden fixtures (reference outputs) ------------------------------------
@pytest.mark.parametrize("path", golden_files(), ids=lambda p: p.rsplit("/", 1)[-1])
def test_golden(path):
    rec = load_golden(path)
    g = graph_from_golden(rec)
    c, eps, S, T = float(rec["c"]), float(rec["eps"]), int(rec["S"]), int(rec["T"])
    assert_close(P.propagation_sweep(g, rec["sweep_x"], c), rec["sweep_y"], what="sweep")
    pr = P.pagerank(g, P.CpiParams(c, eps))
    assert_close(pr.scores, rec["pagerank"], what="pagerank")
    assert pr.iterations_run == int(rec["pagerank_iters"]) and pr.converged == bool(rec["pagerank_conv"])
    assert abs(pr.residual_l1 - float(rec["pagerank_res"])) <= 1e-15
    art = P.preprocess(g, c, eps, T)
    assert_close(art.stranger_scores, rec["stranger"], what="stranger")
    seeds = rec["seeds"].astype(np.uint32)
    for k, s in enumerate(seeds):
        assert_close(P.query(g, art, int(s), S), rec["query"][k], what=f"query {s}")
        assert_close(P.query_na(g, int(s), P.TpaParams(S, T, c, eps)), rec["query_na"][k], what="query_na")
        assert_close(P.exact_rwr(g, int(s), c, eps), rec["exact_rwr"][k], what="exact_rwr")
    assert_close(P.query_batch(g, art, seeds, S), rec["query"], what="query_batch")
    assert_close(P.exact_rwr_batch(g, seeds, c, eps), rec["exact_rwr"], what="exact_rwr_batch")
    parts = P.cpi_partition(g, P.SeedSet.single(int(seeds[0])), c, eps, [S, T])
    assert_close(np.stack(parts), rec["partition"], what="partition")
    for k, (lo, hi) in enumerate([(0, 0), (2, 7), (3, None)]):
        r = P.cpi_run(g, P.SeedSet.single(int(seeds[1])), P.CpiParams(c, eps, lo, hi))
        assert_close(r.scores, rec["win_scores"][k], what=f"window {lo}-{hi}")
        assert r.iterations_run == int(rec["win_iters"][k])
        assert r.converged == bool(rec["win_conv"][k])
        assert abs(r.residual_l1 - float(rec["win_res"][k])) <= 1e-15


# --- oracle on fresh graphs -------------------------------------------------
@pytest.mark.parametrize("policy", ["selfloop", "uniform", "drop"])
@pytest.mark.parametrize("scale", [8, 12, 14])
def test_preprocess_and_queries_rmat(oracle, policy, scale):
    g = P.generate_rmat(scale, 16, rng_seed=scale, policy=policy)
    c, eps, S, T = 0.15, 1e-9, 5, 10
    art = P.preprocess(g, c, eps, T)
    want = oracle.preprocess(g, c, eps, T)
    assert_close(art.stranger_scores, want, what="stranger")
    seeds = P.sample_seeds(g, 40, 7)
    qs = P.query_batch(g, art, seeds, S)
    for k, s in enumerate(seeds):
        w = oracle.query(g, want, c, eps, T, int(s), S)
        assert_close(qs[k], w, what=f"batch query {s}")
        if k < 3:
            assert_close(P.query(g, art, int(s), S), w, what=f"query {s}")
    # property checks (tpa_test.cpp:92-99, cpi_test.cpp:127-134)
    if policy != "drop":
        assert abs(art.stranger_scores.sum() - 0.85 ** T) < eps / c
        assert np.all(np.abs(qs.sum(axis=1) - 1.0) < eps / c)


@pytest.mark.parametrize("B", [1, 2, 5, 8, 13, 16, 31, 32, 33, 64, 100])
def test_query_batch_widths(oracle, B):
    g = P.generate_rmat(11, 16, rng_seed=99, policy="uniform")
    art = P.preprocess(g, 0.15, 1e-9, 10)
    seeds = P.sample_seeds(g, B, B)
    qs = P.query_batch(g, art, seeds, 5)
    for k, s in enumerate(seeds):
        assert_close(qs[k], oracle.query(g, art.stranger_scores, 0.15, 1e-9, 10, int(s), 5), what=f"{B}:{s}")


def test_spmm_is_bitwise_the_reference_order_and_slot_independent(oracle):
    # SpMM rows with in-degree <= 512 are summed sequentially in ascending
    # source order, exactly the reference's scatter order: those entries equal
    # the oracle bit for bit; longer rows (fixed 512-nnz segments) are within
    # tolerance.  Neither depends on the batch width or the slot.
    for scale in (10, 12):
        g = P.generate_rmat(scale, 16, rng_seed=5)
        art = P.preprocess(g, 0.15, 1e-9, 10)
        seeds = P.sample_seeds(g, 64, 3)
        full = P.query_batch(g, art, seeds, 5)
        for B in (8, 16, 32):
            sub = P.query_batch(g, art, seeds[:B][::-1].copy(), 5)[::-1]
            assert np.array_equal(sub, full[:B])
        st = oracle.preprocess(g, 0.15, 1e-9, 10)
        art2 = P.StrangerArtifact(st, g.fingerprint(), 0.15, 1e-9, 10)
        q = P.query_batch(g, art2, seeds[:32], 5)
        indeg = np.bincount(g.out_targets(), minlength=g.node_count())
        all_short = indeg.max() <= 512  # scale 10: max in-degree 332
        for k in range(32):
            want = oracle.query(g, st, 0.15, 1e-9, 10, int(seeds[k]), 5)
            if all_short:
                assert np.array_equal(q[k], want)
            assert_close(q[k], want)
        if scale == 10:
            assert all_short


def test_determinism_repeat_bitwise():
    g = P.generate_rmat(13, 16, rng_seed=11)
    a1 = P.preprocess(g, 0.15, 1e-9, 10)
    a2 = P.preprocess(g, 0.15, 1e-9, 10)
    assert np.array_equal(a1.stranger_scores, a2.stranger_scores)
    seeds = P.sample_seeds(g, 32, 1)
    assert np.array_equal(P.query_batch(g, a1, seeds, 5), P.query_batch(g, a1, seeds, 5))
    q = [P.query(g, a1, int(s), 5) for s in seeds[:4]]
    assert all(np.array_equal(q[k], P.query(g, a1, int(seeds[k]), 5)) for k in range(4))


def test_concurrent_queries_bitwise_equal_serial():
    # tpa_test.cpp:148-161
    import threading
    g = P.generate_random_graph(200, 1200, 88)
    art = P.preprocess(g, 0.15, 1e-9, 12)
    serial = [P.query(g, art, s, 5) for s in range(8)]
    par = [None] * 8

    def work(s):
        par[s] = P.query(g, art, s, 5)
    ts = [threading.Thread(target=work, args=(s,)) for s in range(8)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert all(np.array_equal(par[s], serial[s]) for s in range(8))


# --- the reference's own unit tests, restated on the GPU path ------------------
def test_sweep_cases():
    g = P.Graph(2, [(0, 1), (1, 0)], "selfloop")  # graph_test.cpp:131-137
    y = P.propagation_sweep(g, np.array([0.15, 0.0]), 0.15)
    assert y[0] == 0.0 and abs(y[1] - 0.1275) <= 1e-15 * 1.1275
    g = P.Graph(3, [(0, 1)], "uniform")  # graph_test.cpp:204-215
    y = P.propagation_sweep(g, np.array([0.0, 0.9, 0.0]), 0.15)
    assert np.all(np.abs(y - 0.85 * 0.9 / 3.0) <= 1e-15)
    d = P.Graph(3, [(0, 1)], "drop")
    assert np.all(P.propagation_sweep(d, np.array([0.0, 0.9, 0.0]), 0.15) == 0.0)
    with pytest.raises(ValueError):  # graph_test.cpp:173-180
        P.propagation_sweep(g, np.array([1.0, 2.0]), 0.15)
    with pytest.raises(ValueError):
        P.propagation_sweep(g, np.zeros(3), 1.0)
    with pytest.raises(ValueError):
        P.propagation_sweep(g, np.zeros(3), -0.1)


@pytest.mark.parametrize("policy", ["selfloop", "uniform", "drop"])
def test_sweep_matches_oracle(oracle, policy):
    for seed in range(4):
        g = P.generate_random_graph(50 + 100 * seed, 400 * (seed + 1), seed, policy)
        x = np.random.default_rng(seed).random(g.node_count())
        for c in (0.0, 0.15, 0.5):
            assert_close(P.propagation_sweep(g, x, c), oracle.sweep(g, x, c), what=f"c={c}")
            # mass preservation (graph_test.cpp:139-157)
            if policy != "drop":
                y = P.propagation_sweep(g, x, c)
                assert abs(y.sum() - (1 - c) * x.sum()) <= 1e-12 * (1 + x.sum())


def test_cpi_cases():
    loop = P.Graph(1, [(0, 0)], "selfloop")
    r = P.cpi_run(loop, P.SeedSet.single(0), P.CpiParams())  # cpi_test.cpp:43-48
    assert r.converged and abs(1.0 - r.scores[0]) < 1e-9 / 0.15
    cyc = P.Graph(2, [(0, 1), (1, 0)], "selfloop")
    for g in (cyc, P.generate_random_graph(30, 120, 9)):  # cpi_test.cpp:50-61
        r = P.cpi_run(g, P.SeedSet.single(0), P.CpiParams(0.15, 1e-9))
        assert r.converged and r.iterations_run == 116 and r.residual_l1 < 1e-9
    e = P.exact_rwr(cyc, 0, 0.15, 1e-9)  # cpi_test.cpp:63-69
    assert abs(e[0] - 1 / 1.85) < 1e-8 and abs(e[1] - 0.85 / 1.85) < 1e-8
    r = P.cpi_run(cyc, P.SeedSet.single(0), P.CpiParams(terminal_iter=0))  # cpi_test.cpp:168-178
    assert r.iterations_run == 0 and not r.converged and r.scores[0] == 0.15 and r.scores[1] == 0.0
    assert r.residual_l1 == 0.15
    with pytest.raises(IndexError):  # cpi_test.cpp:180-183
        P.cpi_run(cyc, P.SeedSet.single(5), P.CpiParams())
    k3 = P.generate_random_graph(3, 6, 7)  # cpi_test.cpp:116-125
    res = P.pagerank(k3, P.CpiParams(tolerance=1e-12))
    assert np.all(np.abs(res.scores - 1 / 3) < 1e-9 * (1 + 1 / 3))
    g = P.generate_random_graph(50, 200, 21)  # cpi_test.cpp:127-134
    res = P.pagerank(g, P.CpiParams(tolerance=1e-12, start_iter=15))
    assert abs(res.scores.sum() - 0.85 ** 15) < 1e-9 * (1 + 0.85 ** 15)
    with pytest.raises(ValueError):  # cpi_test.cpp:219-227
        P.cpi_partition(cyc, P.SeedSet.single(0), 0.15, 1e-9, [0])
    with pytest.raises(ValueError):
        P.cpi_partition(cyc, P.SeedSet.single(0), 0.15, 1e-9, [5, 5])


def test_interim_norms_follow_closed_form():
    # cpi_test.cpp:99-114
    rng = np.random.default_rng(77)
    for trial in range(6):
        pol = "selfloop" if trial % 2 == 0 else "uniform"
        n = 10 + int(rng.integers(0, 30))
        g = P.generate_random_graph(n, 4 * n, int(rng.integers(0, 1 << 30)), pol)
        x = np.zeros(n)
        x[trial % n] = 0.15
        for i in range(1, 51):
            x = P.propagation_sweep(g, x, 0.15)
            want = 0.15 * 0.85 ** i
            assert abs(x.sum() - want) < 1e-12 * (1 + want)


def test_windows_additivity_and_monotone(oracle):
    # cpi_test.cpp:136-166
    rng = np.random.default_rng(31)
    for trial in range(6):
        n = 8 + int(rng.integers(0, 20))
        g = P.generate_random_graph(n, 3 * n, int(rng.integers(0, 1 << 30)))
        s = P.SeedSet.single(int(rng.integers(0, n)))
        a = int(rng.integers(0, 3))
        b = a + 1 + int(rng.integers(0, 5))
        d = b + 1 + int(rng.integers(0, 5))

        def win(lo, hi):
            return P.cpi_run(g, s, P.CpiParams(tolerance=1e-300, start_iter=lo, terminal_iter=hi)).scores
        left, right, whole = win(a, b), win(b + 1, d), win(a, d)
        assert np.all(np.abs(left + right - whole) < 1e-12 * (1 + np.abs(whole)))
        ow = oracle.cpi_run(g, list(s.ids()), 0.15, 1e-300, a, d)[0]
        assert_close(whole, ow)


def test_partition_matches_windows(oracle):
    # cpi_test.cpp:185-217
    rng = np.random.default_rng(55)
    for trial in range(6):
        n = 10 + int(rng.integers(0, 25))
        pol = "uniform" if trial % 2 else "selfloop"
        g = P.generate_random_graph(n, 4 * n, int(rng.integers(0, 1 << 30)), pol)
        seed = int(rng.integers(0, n))
        s = 1 + int(rng.integers(0, 5))
        t = s + 1 + int(rng.integers(0, 8))
        parts = P.cpi_partition(g, P.SeedSet.single(seed), 0.15, 1e-9, [s, t])
        want = oracle.cpi_partition(g, [seed], 0.15, 1e-9, [s, t])
        for k in range(3):
            assert_close(parts[k], want[k], what=f"part {k}")


def test_multi_seed_set(oracle):
    g = P.generate_rmat(10, 16, rng_seed=4, policy="uniform")
    seeds = [3, 77, 500, 1000]
    r = P.cpi_run(g, P.SeedSet(seeds), P.CpiParams(0.2, 1e-10, 1, 30))
    sc, it, conv, res = oracle.cpi_run(g, seeds, 0.2, 1e-10, 1, 30)
    assert_close(r.scores, sc)
    assert r.iterations_run == it and r.converged == conv and abs(r.residual_l1 - res) < 1e-15


def test_tpa_cases():
    g = P.generate_random_graph(3, 6, 7)  # tpa_test.cpp:52-60
    art = P.preprocess(g, 0.15, 1e-9, 2)
    assert np.all(np.abs(art.stranger_scores - 0.85 * 0.85 / 3) < 1e-8)
    assert art.stranger_start == 2 and art.graph_fingerprint == g.fingerprint()
    g = P.generate_random_graph(20, 60, 2)  # tpa_test.cpp:70-74
    art = P.preprocess(g, 0.15, 1e-9, 116)
    assert art.stranger_scores.sum() < 1e-9 / 0.15
    loop = P.Graph(1, [(0, 0)], "selfloop")  # tpa_test.cpp:76-81
    a1 = P.preprocess(loop, 0.15, 1e-9, 10)
    assert abs(P.query(loop, a1, 0, 5)[0] - 1.0) < 1e-6 * 2
    g = P.generate_random_graph(20, 60, 2)  # tpa_test.cpp:83-91
    other = P.generate_random_graph(20, 60, 3)
    art = P.preprocess(g, 0.15, 1e-9, 10)
    with pytest.raises(RuntimeError, match="fingerprint"):
        P.query(other, art, 0, 5)
    with pytest.raises(ValueError):
        P.query(g, art, 0, 10)
    with pytest.raises(ValueError):
        P.query(g, art, 0, 0)
    P.query(g, art, 0, 9)
    with pytest.raises(IndexError):
        P.query(g, art, 20, 5)
    with pytest.raises(IndexError):
        P.query_batch(g, art, np.array([1, 2, 25], np.uint32), 5)
    p = P.TpaParams(3, 8)  # tpa_test.cpp:101-119
    r = P.query_na(loop, 0, p)
    assert abs(r[0] - (1 - 0.85 ** 8)) < 1e-9 * 2
    h = P.generate_random_graph(40, 160, 5)
    art = P.preprocess(h, 0.15, 1e-9, 8)
    with_t = P.query(h, art, 3, 3)
    without = P.query_na(h, 3, P.TpaParams(3, 8))
    assert abs(np.abs(with_t - without).sum() - 0.85 ** 8) < 1e-8 * (1 + 0.85 ** 8)


def test_error_bounds_random_trials(oracle):
    # tpa_test.cpp:163-196 (subset of the 120 trials)
    rng = np.random.default_rng(990)
    for trial in range(30):
        n = 5 + int(rng.integers(0, 50))
        m = min(n + int(rng.integers(0, 4 * n)), n * (n - 1))
        pol = ["selfloop", "uniform", "drop"][int(rng.integers(0, 3))]
        g = P.generate_random_graph(n, m, int(rng.integers(0, 1 << 30)), pol)
        s = 1 + int(rng.integers(0, 7))
        t = s + 1 + int(rng.integers(0, 11))
        c = 0.05 + 0.85 * int(rng.integers(0, 1000)) / 1000.0
        seed = int(rng.integers(0, n))
        parts = P.cpi_partition(g, P.SeedSet.single(seed), c, 1e-12, [s, t])
        want = oracle.cpi_partition(g, [seed], c, 1e-12, [s, t])
        for k in range(3):
            assert_close(parts[k], want[k])
        art = P.preprocess(g, c, 1e-12, t)
        assert_close(art.stranger_scores, oracle.preprocess(g, c, 1e-12, t))
        q = P.query(g, art, seed, s)
        assert_close(q, oracle.query(g, art.stranger_scores, c, 1e-12, t, seed, s))


def test_device_resident_batch_matches_host():
    import torch
    g = P.generate_rmat(12, 16, rng_seed=8)
    art = P.preprocess(g, 0.15, 1e-9, 10)
    seeds = P.sample_seeds(g, 32, 2)
    host = P.query_batch(g, art, seeds, 5)
    dev_out = torch.empty((32, g.node_count()), dtype=torch.float64, device="cuda")
    P.query_batch(g, art, torch.as_tensor(seeds.astype(np.int32)).cuda(), 5, out=dev_out)
    assert np.array_equal(dev_out.cpu().numpy(), host)
    nm = torch.empty((g.node_count(), 32), dtype=torch.float64, device="cuda")
    P.query_batch(g, art, torch.as_tensor(seeds.astype(np.int32)).cuda(), 5, out=nm, node_major=True)
    assert np.array_equal(nm.cpu().numpy().T, host)


def test_transpose_ingest_is_exact():
    g = P.generate_rmat(12, 16, rng_seed=21, policy="drop")
    rp, col = g.device().transpose()
    off = g.out_offsets().astype(np.int64)
    src = np.repeat(np.arange(g.node_count(), dtype=np.int64), np.diff(off))
    dst = g.out_targets().astype(np.int64)
    order = np.lexsort((src, dst))
    assert np.array_equal(col, src[order].astype(np.uint32))
    assert np.array_equal(rp, np.concatenate([[0], np.cumsum(np.bincount(dst, minlength=g.node_count()))]))


@pytest.mark.slow
def test_c1_config_full(oracle):
    # BASELINE configs[0]: R-MAT 16, ef 16; preprocess + 1 query (and 64 more).
    g = P.generate_rmat(16, 16, rng_seed=1)
    art = P.preprocess(g, 0.15, 1e-9, 10)
    want = oracle.preprocess(g, 0.15, 1e-9, 10)
    assert_close(art.stranger_scores, want, what="C1 stranger")
    seeds = P.sample_seeds(g, 65, 1)
    assert_close(P.query(g, art, int(seeds[0]), 5), oracle.query(g, want, 0.15, 1e-9, 10, int(seeds[0]), 5))
    qs = P.query_batch(g, art, seeds[1:], 5)
    for k in range(0, 64, 9):
        assert_close(qs[k], oracle.query(g, want, 0.15, 1e-9, 10, int(seeds[1 + k]), 5))


@pytest.mark.gpu
@pytest.mark.slow
def test_c2_config_full(oracle):
    """BASELINE configs[1] at full size: R-MAT 20, ef 16 (16.6 M edges).  The
    stranger vector and sampled queries against the oracle; all 1,024 queries of
    the bench job through the closed-form mass identity (SelfLoop conserves mass:
    ||family||_1 = 1 - (1-c)^S, ||stranger||_1 = (1-c)^T within eps/c)."""
    import torch
    c, eps, S, T = 0.15, 1e-9, 5, 10
    g = P.generate_rmat(20, 16, rng_seed=1)
    art = P.preprocess(g, c, eps, T)
    want = oracle.preprocess(g, c, eps, T)
    assert_close(art.stranger_scores, want, what="C2 stranger")
    seeds = P.sample_seeds(g, 1024, 1)
    out = torch.empty((32, g.node_count()), dtype=torch.float64, device="cuda")
    nsf = P.neighbor_scale_factor(c, S, T)
    mass = (1 + nsf) * (1 - (1 - c) ** S) + (1 - c) ** T
    for b0 in range(0, 1024, 32):
        P.query_batch(g, art, seeds[b0:b0 + 32], S, out=out)
        sums = out.sum(dim=1).cpu().numpy()
        assert np.all(np.abs(sums - mass) <= eps / c), (b0, sums.min(), sums.max())
        if b0 % 256 == 0:
            host = out.cpu().numpy()
            for k in (0, 31):
                assert_close(host[k], oracle.query(g, want, c, eps, T, int(seeds[b0 + k]), S),
                             what=f"C2 query {b0 + k}")
        if b0 == 512:
            # one whole batch element-wise (32 oracle queries on the host cores)
            from concurrent.futures import ThreadPoolExecutor
            host = out.cpu().numpy()
            with ThreadPoolExecutor(8) as ex:
                ws = list(ex.map(lambda k: oracle.query(g, want, c, eps, T, int(seeds[b0 + k]), S), range(32)))
            for k in range(32):
                assert_close(host[k], ws[k], what=f"C2 query {b0 + k}")


@pytest.mark.gpu
def test_uniform_spread_disables_sparse_pull(oracle):
    """A small frontier that reaches dangling nodes (Uniform policy): the next
    sweep carries a spread onto every row, so it must not take the sparse
    (frontier-reachable rows only) pull."""
    rng = np.random.default_rng(11)
    n, live, k = 200_000, 150_000, 8
    src = np.repeat(np.arange(live, dtype=np.uint32), k)
    dst = rng.integers(0, n, src.size, dtype=np.uint32)  # ~25% of targets are dangling sinks
    g = P.Graph(n, (src, dst), "uniform")
    art = P.preprocess(g, 0.15, 1e-9, 10)
    want = oracle.preprocess(g, 0.15, 1e-9, 10)
    assert_close(art.stranger_scores, want, what="stranger")
    seeds = np.arange(0, 32 * 997, 997, dtype=np.uint32)
    out = P.query_batch(g, art, seeds, 5)
    for j in (0, 13, 31):
        assert_close(out[j], oracle.query(g, want, 0.15, 1e-9, 10, int(seeds[j]), 5), what=f"seed {seeds[j]}")
