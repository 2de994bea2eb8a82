"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/tpa_gpu.h declares; the host graph plumbing reproduces the
reference Graph bit-for-bit; parameter validation mirrors the reference.
No kernel is launched here."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

import paper_1708_02574_b200 as P
from paper_1708_02574_b200 import _native


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "tpa_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tpa_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding knows all of them
    assert set(syms) == set(_native.SIGNATURES), set(syms) ^ set(_native.SIGNATURES)


def test_library_is_sm100a_only():
    # the fatbin must hold sm_100a SASS (cuobjdump lists the ELF arch)
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


def test_product_never_touches_the_oracle():
    pkg = os.path.join(ROOT, "paper_1708_02574_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "cpi_oracle" not in text and "librwrank_ref" not in text, f


def test_abi_version_and_nsf():
    assert _native.lib.tpa_abi_version() == 1
    # tpa_test.cpp:40-50
    assert P.neighbor_scale_factor(0.15, 5, 10) == 0.44370531249999995
    assert abs(P.neighbor_scale_factor(0.15, 5, 100000) - 1419857 / 1780143) < 1e-12
    assert P.neighbor_scale_factor(0.15, 5, 5) == 0.0


@pytest.mark.parametrize("policy", ["selfloop", "uniform", "drop"])
def test_random_graph_matches_reference(reference, policy):
    for (n, m, seed) in [(3, 6, 7), (40, 200, 3), (500, 4000, 11), (2000, 30000, 5)]:
        g = P.generate_random_graph(n, m, seed, policy)
        r = reference.graph_random(n, m, seed, policy)
        assert g.fingerprint() == r.fingerprint
        assert np.array_equal(g.out_offsets(), r.out_offsets)
        assert np.array_equal(g.out_targets(), r.out_targets)
        assert np.array_equal(g.dangling_nodes(), r.dangling)


@pytest.mark.parametrize("policy", ["selfloop", "uniform", "drop"])
def test_graph_from_edges_matches_reference(reference, policy):
    rng = np.random.default_rng(7)
    e = rng.integers(0, 300, (5000, 2))  # duplicates, self-loops, dangling nodes
    g = P.Graph(400, e, policy)
    r = reference.graph_from_edges(400, e[:, 0].copy(), e[:, 1].copy(), policy)
    assert g.fingerprint() == r.fingerprint and g.edge_count() == r.m
    assert np.array_equal(g.out_offsets(), r.out_offsets)
    assert np.array_equal(g.out_targets(), r.out_targets)
    assert np.array_equal(g.dangling_nodes(), r.dangling)


def test_rmat_graph_is_deterministic_and_reference_equal(reference):
    a = P.generate_rmat(12, 16, rng_seed=3)
    b = P.generate_rmat(12, 16, rng_seed=3, threads=1)
    assert a == b and a.fingerprint() == b.fingerprint()
    off = a.out_offsets().astype(np.int64)
    src = np.repeat(np.arange(a.node_count(), dtype=np.uint32), np.diff(off))
    r = reference.graph_from_edges(a.node_count(), src, a.out_targets(), "selfloop")
    assert r.fingerprint == a.fingerprint()
    assert len(a.dangling_nodes()) > 0  # R-MAT keeps dangling nodes (repaired)
    assert all(a.out_degree(int(u)) == 1 for u in a.dangling_nodes()[:50])


def test_graph_validation_like_reference():
    # graph_test.cpp:93-96
    with pytest.raises(ValueError, match="at least one node"):
        P.Graph(0, [], "selfloop")
    with pytest.raises(IndexError, match="out of range"):
        P.Graph(2, [(0, 2)], "selfloop")
    with pytest.raises(ValueError):
        P.generate_random_graph(3, 7, 1)
    g = P.Graph(3, [(0, 1), (0, 1), (1, 2)], "selfloop")  # graph_test.cpp:39-48
    assert g.node_count() == 3 and g.edge_count() == 3
    assert list(g.dangling_nodes()) == [2] and list(g.out_neighbors(2)) == [2]
    h = P.Graph(2, [(0, 1)], "uniform")
    assert h.edge_count() == 1 and h.out_degree(1) == 0


def test_sample_seeds():
    g = P.generate_rmat(10, 8, rng_seed=1, policy="uniform")
    s = P.sample_seeds(g, 100, 42)
    assert len(set(s.tolist())) == 100
    dang = set(g.dangling_nodes().tolist())
    assert not (set(s.tolist()) & dang)
    assert np.array_equal(s, P.sample_seeds(g, 100, 42))
    with pytest.raises(RuntimeError, match="non-dangling"):
        P.sample_seeds(g, g.node_count(), 1)


def test_param_validation_like_reference():
    # cpi_test.cpp:19-41, tpa_test.cpp:28-38
    with pytest.raises(ValueError):
        P.SeedSet([])
    with pytest.raises(ValueError):
        P.SeedSet([1, 1])
    s = P.SeedSet([3, 1, 2])
    assert s.size() == 3 and s.ids()[0] == 1
    with pytest.raises(IndexError):
        s.validate_against(3)
    s.validate_against(4)
    p = P.CpiParams()
    p.validate()
    p.restart_prob = 0.0
    with pytest.raises(ValueError):
        p.validate()
    p.restart_prob, p.tolerance = 0.15, 0.0
    with pytest.raises(ValueError):
        p.validate()
    p.tolerance, p.start_iter, p.terminal_iter = 1e-9, 5, 4
    with pytest.raises(ValueError):
        p.validate()
    t = P.TpaParams()
    t.validate()
    t.family_end = 0
    with pytest.raises(ValueError):
        t.validate()
    t.family_end, t.stranger_start = 5, 5
    with pytest.raises(ValueError):
        t.validate()


def test_vec_ptr_rejects_bad_buffers():
    """Outputs must be written in place: wrong dtype, non-contiguous or read-only
    outputs and wrong-dtype tensors are refused, never copied."""
    import torch
    from paper_1708_02574_b200.graph import vec_ptr
    with pytest.raises(TypeError):
        vec_ptr(torch.zeros(8, dtype=torch.float32), 8)
    with pytest.raises(ValueError):
        vec_ptr(np.zeros(8, np.float32), 8, writable=True)
    with pytest.raises(ValueError):
        vec_ptr(np.zeros(16)[::2], 8, writable=True)
    ro = np.zeros(8)
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        vec_ptr(ro, 8, writable=True)
    with pytest.raises(ValueError):
        vec_ptr(np.zeros(9), 8, writable=True)
    a = np.zeros(8)
    p, dev, keep = vec_ptr(a, 8, writable=True)
    assert p == a.ctypes.data and not dev and keep is a
    p, dev, keep = vec_ptr([1, 2, 3], 3)  # inputs may be converted
    assert keep.dtype == np.float64


def test_compute_entry_points_fail_loudly_without_a_gpu():
    """No CPU fallback: on a box without a CUDA device every compute entry
    raises the library's CUDA error instead of returning numbers."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    g = P.generate_rmat(8, 8, rng_seed=3)
    with pytest.raises(P.CudaError):
        P.preprocess(g, 0.15, 1e-9, 10)
    with pytest.raises(P.CudaError):
        P.pagerank(g, P.CpiParams(0.15, 1e-9))
