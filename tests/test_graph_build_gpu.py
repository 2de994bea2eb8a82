"""GPU graph construction: tpa_host_graph_build_gpu must give
the reference Graph constructor's out-CSR, dangling list and fingerprint
(graph.cpp:53-91) -- checked against the host builder, which
tests/test_host_abi.py pins to the reference itself."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1708_02574_b200 as P


def _same(a: P.Graph, b: P.Graph):
    assert a.node_count() == b.node_count() and a.edge_count() == b.edge_count()
    assert np.array_equal(a.out_offsets(), b.out_offsets())
    assert np.array_equal(a.out_targets(), b.out_targets())
    assert np.array_equal(a.dangling_nodes(), b.dangling_nodes())
    assert a.fingerprint() == b.fingerprint()


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["selfloop", "uniform", "drop"])
@pytest.mark.parametrize("n,m", [(1, 0), (1, 3), (7, 20), (1000, 5000), (200_000, 3_000_000)])
def test_build_gpu_equals_host(policy, n, m):
    rng = np.random.default_rng(n + m)
    # skewed endpoints, duplicates and self-loops included; isolated nodes likely
    src = (rng.random(m) ** 2 * n).astype(np.uint32) % max(n, 1)
    dst = rng.integers(0, n, m, dtype=np.uint32) if m else np.zeros(0, np.uint32)
    if m > 10:
        src[:5] = dst[:5]          # self-loops in the input stay edges
        src[5:10], dst[5:10] = src[0], dst[0]  # duplicates
    host = P.Graph(n, (src, dst), policy)
    gpu = P.Graph.build_gpu(n, (src, dst), policy)
    _same(host, gpu)


@pytest.mark.gpu
def test_build_gpu_errors_match_reference():
    with pytest.raises(ValueError):
        P.Graph.build_gpu(0, (np.zeros(0, np.uint32), np.zeros(0, np.uint32)))
    src = np.array([0, 1, 9, 2, 7], np.uint32)
    dst = np.array([1, 2, 0, 11, 1], np.uint32)
    with pytest.raises(IndexError) as gpu_err:
        P.Graph.build_gpu(5, (src, dst))
    with pytest.raises(IndexError) as host_err:
        P.Graph(5, (src, dst))
    # the first offending edge in input order, the reference's message
    assert str(gpu_err.value) == str(host_err.value) == "edge endpoint out of range: 9 -> 0"


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["selfloop", "drop"])
@pytest.mark.parametrize("scale,ef,a,b,c", [(1, 1, 0.57, 0.19, 0.19), (6, 3, 0.25, 0.25, 0.25),
                                            (12, 16, 0.57, 0.19, 0.19), (17, 16, 0.57, 0.19, 0.19)])
def test_rmat_gpu_equals_host(policy, scale, ef, a, b, c):
    """The GPU generator replays the host generator's per-chunk mt19937_64
    streams (scale 17 x ef 16 = 2 chunks of 2^20 edges): same edges, same
    graph, same fingerprint."""
    host = P.generate_rmat(scale, ef, a, b, c, rng_seed=11, policy=policy)
    gpu = P.generate_rmat(scale, ef, a, b, c, rng_seed=11, policy=policy, device=0)
    _same(host, gpu)


@pytest.mark.gpu
def test_rmat_gpu_errors():
    with pytest.raises(ValueError):
        P.generate_rmat(0, 16, device=0)
    with pytest.raises(ValueError):
        P.generate_rmat(10, 16, 0.6, 0.3, 0.3, device=0)
