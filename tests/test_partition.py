"""Row-partitioned CPI (multi-GPU layout, csrc/tpa_part.cuh).

CPU: the nnz-balanced row split, and the partitioned algorithm itself run by
world_size-2 gloo ranks (tests/part_emul.py: all-gather of share slices +
all-reduce of exact fixed-point totals) against the oracle and against the
same algorithm on one rank (bitwise).
GPU: partitions driven in-process (peer copies) and through NCCL (one rank)
against the whole-graph GPU run (bitwise) and the oracle (tolerance)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import assert_close

import paper_1708_02574_b200 as P
from paper_1708_02574_b200.partition import in_degrees, partition_rows

C, EPS, T = 0.15, 1e-9, 10


def test_partition_rows_balanced_and_covering():
    from paper_1708_02574_b200.partition import TILE_NNZ, item_starts
    g = P.generate_rmat(12, 16, rng_seed=3)
    indeg = in_degrees(g)
    m = int(indeg.sum())
    prefix = np.concatenate([[0], np.cumsum(indeg)]).astype(np.int64)
    cuts = set(item_starts(prefix, g.node_count())) | {g.node_count()}
    for G in (1, 2, 3, 4, 8, 64):
        b = partition_rows(indeg, G)
        assert b[0] == 0 and b[-1] == g.node_count() and np.all(np.diff(b) >= 0)
        for k in range(1, G):
            assert int(b[k]) in cuts  # cut at a tile start only
            assert prefix[b[k]] >= (m * k) // G
        nnz = np.diff(prefix[b])
        assert nnz.max() <= m / G + TILE_NNZ + indeg.max()


def test_partition_rows_degenerate():
    assert list(partition_rows([0, 0, 0], 2)) == [0, 0, 3]
    assert list(partition_rows([5], 4)) == [0, 1, 1, 1, 1]
    # one 2048-nnz tile holds all six rows: no interior cut
    assert list(partition_rows([1, 2, 3, 0, 4, 5], 3)) == [0, 6, 6, 6]
    assert list(partition_rows([3000, 1, 3000, 1], 2)) == [0, 2, 4]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, G, port, args, q):
    import torch.distributed as dist
    import part_emul
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=G)
    try:
        res = part_emul.run(*args, G=G, rank=rank, dist=dist)
        q.put((rank, res[0].tolist(), res[1], res[2], res[3]))
    finally:
        dist.destroy_process_group()


def _run_gloo(G, args):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, G, port, args, q)) for r in range(G)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(G)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out)


@pytest.mark.parametrize("policy", ["selfloop", "uniform", "drop"])
def test_gloo_two_rank_partitioned_pagerank_matches_oracle(oracle, policy):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    import part_emul
    g = P.generate_rmat(9, 8, rng_seed=17, policy=policy)
    n = g.node_count()
    off, tgt = g.out_offsets(), g.out_targets()
    pol = int(g.dangling_policy())
    args = (off, tgt, n, pol, C, EPS, T, -1, None)
    outs = _run_gloo(2, args)
    one = part_emul.run(*args, G=1, rank=0)
    want, it, conv, _ = oracle.pagerank(g, C, EPS, start=T)
    for rank, scores, iters, converged, residual in outs:
        scores = np.array(scores)
        # every rank holds the whole vector; identical to the one-rank run bit for bit
        assert np.array_equal(scores, one[0]) and iters == one[1] and residual == one[3]
        assert iters == it and converged == conv
        assert_close(scores, want, what=f"{policy} rank {rank}")


def test_gloo_two_rank_partitioned_seed_window(oracle):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    g = P.generate_rmat(9, 8, rng_seed=23, policy="uniform")
    n = g.node_count()
    seeds = [3, 100, 257]
    args = (g.out_offsets(), g.out_targets(), n, int(g.dangling_policy()), C, EPS, 2, 7, seeds)
    outs = _run_gloo(2, args)
    want, it, conv, _ = oracle.cpi_run(g, seeds, C, EPS, start=2, terminal=7)
    for rank, scores, iters, converged, residual in outs:
        assert iters == it == 7 and converged == conv
        assert_close(np.array(scores), want, what=f"rank {rank}")


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["selfloop", "uniform", "drop"])
@pytest.mark.parametrize("G", [1, 2, 3, 4])
def test_group_preprocess_bitwise_whole_graph(oracle, policy, G):
    g = P.generate_rmat(12, 16, rng_seed=31, policy=policy)
    whole = P.preprocess(g, C, EPS, T).stranger_scores
    grp = P.PartitionGroup(g, [0] * G)
    try:
        b = grp.bounds()
        assert list(b) == list(partition_rows(in_degrees(g), G))
        got = grp.preprocess(C, EPS, T)
    finally:
        grp.close()
    assert np.array_equal(got, whole), f"max diff {np.abs(got - whole).max():.3e}"
    assert_close(got, oracle.preprocess(g, C, EPS, T), what=f"{policy} G={G}")


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 5])
def test_group_cpi_run_windows_and_seeds(oracle, G):
    g = P.generate_rmat(11, 16, rng_seed=7, policy="uniform")
    grp = P.PartitionGroup(g, [0] * G)
    try:
        for seeds, start, term in [(None, 0, None), ([5], 0, None), ([1, 9, 2000], 3, 9), (None, 10, None)]:
            ss = P.SeedSet.all_nodes(g.node_count()) if seeds is None else P.SeedSet(seeds)
            prm = P.CpiParams(restart_prob=C, tolerance=EPS, start_iter=start, terminal_iter=term)
            got = grp.cpi_run(ss, prm)
            ref = P.cpi_run(g, ss, prm)
            assert np.array_equal(got.scores, ref.scores)
            assert (got.iterations_run, got.converged, got.residual_l1) == \
                (ref.iterations_run, ref.converged, ref.residual_l1)
            want, it, conv, _ = oracle.cpi_run(g, seeds, C, EPS, start, term)
            assert got.iterations_run == it
            assert_close(got.scores, want, what=f"seeds={seeds} window=[{start},{term}]")
    finally:
        grp.close()


@pytest.mark.gpu
def test_nccl_single_rank_partition():
    g = P.generate_rmat(12, 16, rng_seed=5)
    whole = P.pagerank(g, P.CpiParams(restart_prob=C, tolerance=EPS))
    pg = P.PartitionedGraph(g, 1, 0, comm_id=P.partition.comm_unique_id())
    try:
        assert pg.info() == (1, 0, 0, g.node_count(), g.node_count())
        got = pg.pagerank(P.CpiParams(restart_prob=C, tolerance=EPS))
        assert np.array_equal(got.scores, whole.scores) and got.iterations_run == whole.iterations_run
        st = pg.preprocess(C, EPS, T)
        assert np.array_equal(st, P.preprocess(g, C, EPS, T).stranger_scores)
    finally:
        pg.close()


@pytest.mark.gpu
def test_partition_refuses_queries_and_bad_ranks():
    from paper_1708_02574_b200 import _native as N
    import ctypes as Cc
    g = P.generate_rmat(10, 8, rng_seed=1)
    pg = P.PartitionedGraph(g, 1, 0)
    try:
        out = np.empty(g.node_count())
        rc = N.lib.tpa_query(pg.h, None, 0, 5, out.ctypes.data, 0)
        assert rc == N.TPA_ERR_INVALID_ARGUMENT and b"row-partitioned" in N.lib.tpa_last_error()
    finally:
        pg.close()
    with pytest.raises(ValueError):
        P.PartitionedGraph(g, 2, 0)  # nranks > 1 needs a communicator id
    with pytest.raises(ValueError):
        P.PartitionedGraph(g, 2, 2, comm_id=b"\0" * 128)
    h = Cc.c_void_p()
    grp = P.PartitionGroup(g, [0, 0])
    try:
        p0 = Cc.c_void_p()
        N.check(N.lib.tpa_group_part(grp.h, 0, Cc.byref(p0)))
        it = Cc.c_uint32()
        rc = N.lib.tpa_cpi_run(p0, None, 0, C, EPS, 0, -1, out.ctypes.data, Cc.byref(it), None, None, 0)
        assert rc == N.TPA_ERR_INVALID_ARGUMENT  # a group member runs through tpa_group_*
    finally:
        grp.close()
    del h
