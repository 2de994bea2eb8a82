"""Device top-k: top_k_nodes (metrics.cpp:25-36) for B
vectors on the GPU, checked against the reference's comparator restated in
numpy (score descending, equal scores by ascending id; values compared, so
-0.0 ties +0.0) and the reference's own test case (metrics_test.cpp:42-49)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1708_02574_b200 as P


def ref_top_k(v: np.ndarray, k: int) -> np.ndarray:
    """metrics.cpp:25-36 restated: partial_sort by (score desc, id asc)."""
    ids = np.arange(v.size)
    return np.lexsort((ids, -v))[:k]


def test_ref_top_k_restatement_on_reference_case():
    assert list(ref_top_k(np.array([0.5, 0.9, 0.5, 0.5, 0.1]), 3)) == [1, 0, 2]


@pytest.mark.gpu
def test_top_k_reference_case():
    g = P.Graph(5, [(0, 1), (1, 2), (2, 3), (3, 4)])
    ids, vals = P.top_k(g, np.array([0.5, 0.9, 0.5, 0.5, 0.1]), 3)
    assert list(ids) == [1, 0, 2] and list(vals) == [0.9, 0.5, 0.5]
    with pytest.raises(IndexError):
        P.top_k(g, np.zeros(5), 0)
    with pytest.raises(IndexError):
        P.top_k(g, np.zeros(5), 6)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 7, 100, 4096, 20000])
def test_top_k_random_with_ties(k):
    rng = np.random.default_rng(k)
    g = P.generate_rmat(15, 4, rng_seed=1)
    n = g.node_count()
    B = 5
    v = rng.random((B, n))
    v[0] = np.round(v[0], 2)                  # heavy ties
    v[1, : n // 2] = 0.0                      # a block of exact zeros ...
    v[1, n // 4: n // 2] = -0.0               # ... half of them negative zero
    v[2] = 1e-300 * rng.random(n)             # subnormal-range spread
    v[3] = np.where(rng.random(n) < 0.5, 3.0, -3.0)  # two values only
    ids, vals = P.top_k(g, v, min(k, n))
    for b in range(B):
        want = ref_top_k(v[b], min(k, n))
        assert np.array_equal(ids[b].astype(np.int64), want), f"vector {b}"
        assert np.array_equal(vals[b], v[b][want])


@pytest.mark.gpu
def test_top_k_device_tensors_and_full_k():
    import torch
    g = P.generate_rmat(12, 8, rng_seed=2)
    n = g.node_count()
    v = torch.rand((3, n), dtype=torch.float64, device="cuda")
    ids, vals = P.top_k(g, v, n)  # k = n: the full ranking
    assert ids.is_cuda and vals.is_cuda
    host = v.cpu().numpy()
    for b in range(3):
        assert np.array_equal(ids[b].cpu().numpy().astype(np.int64), ref_top_k(host[b], n))


@pytest.mark.gpu
@pytest.mark.parametrize("na", [False, True])
def test_query_batch_topk_matches_full_vectors(na):
    g = P.generate_rmat(13, 16, rng_seed=9, policy="uniform")
    art = P.preprocess(g, 0.15, 1e-9, 10)
    seeds = P.sample_seeds(g, 70, 3)  # 64 + 6: two device chunks
    k = 50
    ids, vals = P.query_batch_topk(g, art, seeds, 5, k, na=na)
    full = P.query_batch(g, art, seeds, 5, na=na)
    for b in range(len(seeds)):
        want = ref_top_k(full[b], k)
        assert np.array_equal(ids[b].astype(np.int64), want)
        assert np.array_equal(vals[b], full[b][want])
