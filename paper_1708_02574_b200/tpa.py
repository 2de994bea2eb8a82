"""Reference-mirroring CPI / TPA API on the B200 engine.

Same names, argument meaning and error behaviour as
proj/include/rwrank/cpi.hpp and tpa.hpp; every call runs the sm_100a kernels
through the C-ABI (include/tpa_gpu.h).  Python exception types stand in for
the reference's: ValueError = std::invalid_argument, IndexError =
std::out_of_range, RuntimeError = std::runtime_error.  The reference's
``threads`` arguments are accepted and ignored (they select host threads).

Vectors come back as numpy arrays (the reference's ScoreVector).  The batched
extensions (``query_batch``, ``exact_rwr_batch``) also accept a torch CUDA
tensor as ``out`` to keep results resident in HBM.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from ._native import check, lib
from .graph import Graph, vec_ptr

kDefaultRestartProb = 0.15  # cpi.hpp:9
kDefaultTolerance = 1e-9    # cpi.hpp:10


@dataclass
class CpiParams:
    """cpi.hpp:12-20"""
    restart_prob: float = kDefaultRestartProb
    tolerance: float = kDefaultTolerance
    start_iter: int = 0
    terminal_iter: Optional[int] = None
    threads: int = 1

    def validate(self) -> None:  # cpi.cpp:11-17
        if not (self.restart_prob > 0.0 and self.restart_prob < 1.0):
            raise ValueError("restart probability must be in (0, 1)")
        if not (self.tolerance > 0.0):
            raise ValueError("tolerance must be positive")
        if self.terminal_iter is not None and self.terminal_iter < self.start_iter:
            raise ValueError("terminal iteration precedes start iteration")


@dataclass
class CpiResult:
    """cpi.hpp:22-27"""
    scores: np.ndarray
    iterations_run: int = 0
    converged: bool = False
    residual_l1: float = 0.0


class SeedSet:
    """cpi.hpp:30-42: non-empty, stored sorted, no duplicates."""

    def __init__(self, ids: Sequence[int]):
        arr = np.sort(np.asarray(list(ids) if not isinstance(ids, np.ndarray) else ids, dtype=np.int64))
        if arr.size == 0:
            raise ValueError("seed set must not be empty")
        if arr.size > 1 and np.any(arr[1:] == arr[:-1]):
            raise ValueError("seed set contains duplicate ids")
        if arr[0] < 0:
            raise IndexError("seed id out of range")
        self._ids = arr.astype(np.uint32) if arr[-1] <= 0xFFFFFFFF else arr
        self._all = None

    @staticmethod
    def single(node: int) -> "SeedSet":
        return SeedSet([node])

    @staticmethod
    def all_nodes(node_count: int) -> "SeedSet":
        s = SeedSet.__new__(SeedSet)
        s._ids = None
        s._all = int(node_count)
        return s

    def ids(self) -> np.ndarray:
        return np.arange(self._all, dtype=np.uint32) if self._ids is None else self._ids

    def size(self) -> int:
        return self._all if self._ids is None else int(self._ids.size)

    def validate_against(self, node_count: int) -> None:  # cpi.cpp:34-39
        if self._ids is not None and int(self._ids[-1]) >= node_count:
            raise IndexError(f"seed id {int(self._ids[-1])} out of range for graph with {node_count} nodes")


def _dev(g: Graph):
    return g.device(0)


def _terminal(t) -> int:
    return -1 if t is None else int(t)


def cpi_run(g: Graph, seeds: SeedSet, params: CpiParams) -> CpiResult:
    """cpi.hpp:44-49 / cpi.cpp:87-101 on the GPU."""
    params.validate()
    n = g.node_count()
    out = np.empty(n, np.float64)
    it, conv, res = C.c_uint32(), C.c_int(), C.c_double()
    if seeds._ids is None:  # all nodes: pagerank's seed set
        check(lib.tpa_cpi_run(_dev(g).h, None, 0, params.restart_prob, params.tolerance, params.start_iter,
                              _terminal(params.terminal_iter), out.ctypes.data, C.byref(it), C.byref(conv),
                              C.byref(res), 0))
    else:
        ids = np.ascontiguousarray(seeds._ids, np.uint32) if seeds._ids[-1] <= 0xFFFFFFFF else None
        if ids is None:
            seeds.validate_against(n)
        check(lib.tpa_cpi_run(_dev(g).h, ids.ctypes.data, ids.size, params.restart_prob, params.tolerance,
                              params.start_iter, _terminal(params.terminal_iter), out.ctypes.data, C.byref(it),
                              C.byref(conv), C.byref(res), 0))
    return CpiResult(out, it.value, bool(conv.value), res.value)


def exact_rwr(g: Graph, seed: int, c: float = kDefaultRestartProb, eps: float = kDefaultTolerance,
              threads: int = 1) -> np.ndarray:
    """cpi.hpp:52-54 / cpi.cpp:103-109"""
    return cpi_run(g, SeedSet.single(seed), CpiParams(restart_prob=c, tolerance=eps, threads=threads)).scores


def pagerank(g: Graph, params: CpiParams) -> CpiResult:
    """cpi.hpp:56-57 / cpi.cpp:111-113"""
    return cpi_run(g, SeedSet.all_nodes(g.node_count()), params)


def cpi_partition(g: Graph, seeds: SeedSet, c: float, eps: float, boundaries: Sequence[int],
                  threads: int = 1) -> list:
    """cpi.hpp:59-62 / cpi.cpp:115-136: boundaries.size()+1 segment sums."""
    n = g.node_count()
    b = np.ascontiguousarray(np.asarray(list(boundaries), dtype=np.int64).astype(np.uint32))
    ids = np.ascontiguousarray(seeds.ids(), np.uint32)
    out = np.empty((b.size + 1) * n, np.float64)
    check(lib.tpa_cpi_partition(_dev(g).h, ids.ctypes.data, ids.size, float(c), float(eps),
                                b.ctypes.data if b.size else None, b.size, out.ctypes.data, 0))
    return [out[k * n:(k + 1) * n] for k in range(b.size + 1)]


def exact_rwr_batch(g: Graph, seeds, c: float = kDefaultRestartProb, eps: float = kDefaultTolerance,
                    out=None):
    """B independent exact_rwr runs as one batched CPI; returns [B][n]."""
    if type(seeds).__module__.startswith("torch"):
        seeds = seeds.detach().cpu().numpy()
    s = np.ascontiguousarray(seeds, np.uint32)
    n = g.node_count()
    if out is None:
        out = np.empty((s.size, n), np.float64)
    p, dev, keep = vec_ptr(out, s.size * n, writable=True, device=_dev(g).device)
    check(lib.tpa_exact_rwr_batch(_dev(g).h, s.ctypes.data, s.size, float(c), float(eps), p,
                                  N.TPA_DEVICE_PTRS if dev else 0))
    return out


# ---------------------------------------------------------------------------
# TPA (tpa.hpp)
# ---------------------------------------------------------------------------
@dataclass
class TpaParams:
    """tpa.hpp:7-14"""
    family_end: int = 5       # S
    stranger_start: int = 10  # T
    restart_prob: float = kDefaultRestartProb
    tolerance: float = kDefaultTolerance

    def validate(self) -> None:  # tpa.cpp:8-17
        if self.family_end < 1:
            raise ValueError("family_end (S) must be at least 1")
        if self.stranger_start <= self.family_end:
            raise ValueError("stranger_start (T) must exceed family_end (S)")
        CpiParams(self.restart_prob, self.tolerance).validate()


@dataclass(eq=False)
class StrangerArtifact:
    """tpa.hpp:17-23 (+ a cached device copy of the stranger vector).

    Once uploaded, ``stranger_scores`` is read-only (the device copy is keyed
    by the array object); assign a new array to change the scores."""
    stranger_scores: np.ndarray = field(default_factory=lambda: np.empty(0))
    graph_fingerprint: int = 0
    restart_prob: float = kDefaultRestartProb
    tolerance: float = kDefaultTolerance
    stranger_start: int = 0

    def __post_init__(self):
        self._dev = None  # (graph handle, key, tpa_artifact*)

    def _key(self):
        return (id(self.stranger_scores), self.graph_fingerprint, self.restart_prob, self.tolerance,
                self.stranger_start)

    def device(self, g: Graph):
        """tpa_artifact* on g's device, re-uploaded if the fields changed."""
        dg = _dev(g)
        if self._dev is not None and self._dev[0] is dg and self._dev[1] == self._key():
            return self._dev[2]
        self._release()
        st = np.ascontiguousarray(self.stranger_scores, np.float64)
        if st.size != g.node_count():
            raise ValueError("stranger vector length does not match node count")
        h = C.c_void_p()
        check(lib.tpa_artifact_create(dg.h, st.ctypes.data, int(self.graph_fingerprint), float(self.restart_prob),
                                      float(self.tolerance), int(self.stranger_start), 0, C.byref(h)))
        self._dev = (dg, self._key(), h)
        self._freeze()
        return h

    def _freeze(self):
        # the device copy follows the array's identity (_key): freeze the
        # uploaded array so an in-place edit cannot leave a stale device copy
        # -- assign a new array to change the scores (it is re-uploaded)
        if isinstance(self.stranger_scores, np.ndarray):
            self.stranger_scores.flags.writeable = False

    def _release(self):
        if self._dev is not None:
            lib.tpa_artifact_destroy(self._dev[2])
            self._dev = None

    def __del__(self):
        try:
            self._release()
        except Exception:
            pass


def preprocess(g: Graph, c: float, eps: float, stranger_start: int, threads: int = 1) -> StrangerArtifact:
    """tpa.hpp:25-28 / tpa.cpp:19-37: PageRank window [T, convergence) on the GPU."""
    if stranger_start < 1:
        raise ValueError("stranger_start (T) must be at least 1")
    dg = _dev(g)
    out = np.empty(g.node_count(), np.float64)
    h = C.c_void_p()
    check(lib.tpa_preprocess(dg.h, float(c), float(eps), int(stranger_start), out.ctypes.data, C.byref(h), 0))
    art = StrangerArtifact(out, g.fingerprint(), float(c), float(eps), int(stranger_start))
    art._dev = (dg, art._key(), h)
    art._freeze()
    return art


def neighbor_scale_factor(c: float, family_end: int, stranger_start: int) -> float:
    """tpa.hpp:30-32 / tpa.cpp:39-44 (host std::pow, as the reference)."""
    return lib.tpa_neighbor_scale_factor(float(c), int(family_end), int(stranger_start))


def _check_artifact(g: Graph, artifact: StrangerArtifact, family_end: int) -> None:
    # tpa.cpp:63-66, before anything touches the device
    if artifact.graph_fingerprint != g.fingerprint():
        raise RuntimeError("stale artifact: graph fingerprint mismatch")
    if family_end < 1 or family_end >= artifact.stranger_start:
        raise ValueError("family_end (S) must satisfy 1 <= S < T")


def query(g: Graph, artifact: StrangerArtifact, seed: int, family_end: int, threads: int = 1) -> np.ndarray:
    """tpa.hpp:34-38 / tpa.cpp:61-76 on the GPU."""
    _check_artifact(g, artifact, family_end)
    if seed < 0 or seed > 0xFFFFFFFF:
        raise IndexError(f"seed id {seed} out of range for graph with {g.node_count()} nodes")
    out = np.empty(g.node_count(), np.float64)
    check(lib.tpa_query(_dev(g).h, artifact.device(g), int(seed), int(family_end), out.ctypes.data, 0))
    return out


def query_na(g: Graph, seed: int, params: TpaParams, threads: int = 1) -> np.ndarray:
    """tpa.hpp:40-41 / tpa.cpp:78-86 on the GPU."""
    params.validate()
    if seed < 0 or seed > 0xFFFFFFFF:
        raise IndexError(f"seed id {seed} out of range for graph with {g.node_count()} nodes")
    s = np.array([seed], np.uint32)
    out = np.empty(g.node_count(), np.float64)
    check(lib.tpa_query_na_batch(_dev(g).h, s.ctypes.data, 1, params.family_end, params.stranger_start,
                                 params.restart_prob, params.tolerance, out.ctypes.data, 0))
    return out


def query_batch(g: Graph, artifact: StrangerArtifact, seeds, family_end: int, out=None, na: bool = False,
                node_major: bool = False, sync: bool = True):
    """B independent ``query`` calls as one batched CPI (SpMM over the seeds).

    ``out``: None (returns a numpy [B][n] array), a numpy array, or a torch
    tensor (CUDA: results stay in HBM; with ``sync=False`` the call returns
    once the work is enqueued on the graph's stream).  ``node_major`` lays the
    output out [n][B] (B in {8,16,32,64})."""
    _check_artifact(g, artifact, family_end)
    n = g.node_count()
    dg = _dev(g)
    # seeds always cross the C-ABI as a host array (validated before any launch)
    if type(seeds).__module__.startswith("torch"):
        seeds = seeds.detach().cpu().numpy()
    s = np.ascontiguousarray(np.asarray(seeds).astype(np.int64, copy=False))
    if s.size and (s.min() < 0 or s.max() > 0xFFFFFFFF):
        bad = int(s[(s < 0) | (s > 0xFFFFFFFF)][0])
        raise IndexError(f"seed id {bad} out of range for graph with {n} nodes")
    s = np.ascontiguousarray(s, np.uint32)
    B = int(s.size)
    sp = s.ctypes.data
    if out is None:
        out = np.empty((B, n) if not node_major else (n, B), np.float64)
    p, odev, keep = vec_ptr(out, B * n, writable=True, device=dg.device)
    flags = (N.TPA_DEVICE_PTRS if odev else 0) | (N.TPA_NODE_MAJOR if node_major else 0) | \
            (N.TPA_QUERY_NA if na else 0) | (N.TPA_ASYNC if (odev and not sync) else 0)
    check(lib.tpa_query_batch(dg.h, artifact.device(g), sp, B, int(family_end), p, flags))
    return out


def _seed_array(seeds, n):
    if type(seeds).__module__.startswith("torch"):
        seeds = seeds.detach().cpu().numpy()
    s = np.ascontiguousarray(np.asarray(seeds).astype(np.int64, copy=False))
    if s.size and (s.min() < 0 or s.max() > 0xFFFFFFFF):
        bad = int(s[(s < 0) | (s > 0xFFFFFFFF)][0])
        raise IndexError(f"seed id {bad} out of range for graph with {n} nodes")
    return np.ascontiguousarray(s, np.uint32)


def top_k(g: Graph, scores, k: int):
    """metrics.hpp:17 / metrics.cpp:25-36 ``top_k_nodes`` for one vector [n] or
    B vectors [B][n] on the GPU: (ids [B][k] uint32, scores [B][k]), score
    descending, ties by ascending id.  ``scores``: numpy or torch (CUDA
    tensors stay on the device and the results come back as CUDA tensors)."""
    n = g.node_count()
    if k < 1 or k > n:
        raise IndexError(f"k must be in [1, n], got {k}")
    dg = _dev(g)
    single = getattr(scores, "ndim", 2) == 1
    is_torch = type(scores).__module__.startswith("torch")
    if is_torch and scores.is_cuda:
        import torch
        sc = scores.contiguous().view(-1, n).to(torch.float64)
        B = sc.shape[0]
        ids = torch.empty((B, k), dtype=torch.int32, device=sc.device)
        vals = torch.empty((B, k), dtype=torch.float64, device=sc.device)
        check(lib.tpa_top_k(dg.h, sc.data_ptr(), B, int(k), ids.data_ptr(), vals.data_ptr(), N.TPA_DEVICE_PTRS))
        return (ids[0], vals[0]) if single else (ids, vals)
    sc = np.ascontiguousarray(np.asarray(scores.cpu() if is_torch else scores, np.float64)).reshape(-1, n)
    B = sc.shape[0]
    ids = np.empty((B, k), np.uint32)
    vals = np.empty((B, k), np.float64)
    check(lib.tpa_top_k(dg.h, sc.ctypes.data, B, int(k), ids.ctypes.data, vals.ctypes.data, 0))
    return (ids[0], vals[0]) if single else (ids, vals)


def query_batch_topk(g: Graph, artifact: StrangerArtifact, seeds, family_end: int, k: int, na: bool = False):
    """``query_batch`` + ``top_k_nodes`` per seed on the device (the CLI's query
    output, rwrank_main.cpp:158-165): only B·k ids / scores reach the host."""
    _check_artifact(g, artifact, family_end)
    n = g.node_count()
    if k < 1 or k > n:
        raise IndexError(f"k must be in [1, n], got {k}")
    s = _seed_array(seeds, n)
    B = int(s.size)
    ids = np.empty((B, k), np.uint32)
    vals = np.empty((B, k), np.float64)
    check(lib.tpa_query_batch_topk(_dev(g).h, artifact.device(g), s.ctypes.data, B, int(family_end), int(k),
                                   ids.ctypes.data, vals.ctypes.data, N.TPA_QUERY_NA if na else 0))
    return ids, vals


def save_artifact(artifact: StrangerArtifact, path, g: Graph) -> None:
    """persistence.hpp save_artifact: the TPA1 file (48 + 8n bytes), written
    from the artifact's device copy on g's GPU, CRC-32 computed on the GPU."""
    check(lib.tpa_artifact_save(artifact.device(g), str(path).encode()))


def load_artifact(path, g: Graph) -> StrangerArtifact:
    """persistence.hpp load_artifact (same checks, same order, same messages;
    RuntimeError), CRC-32 on the GPU; the artifact arrives bound to g's GPU."""
    h = C.c_void_p()
    check(lib.tpa_artifact_load(_dev(g).h, str(path).encode(), C.byref(h)))
    n, c, eps, T, fp = C.c_uint64(), C.c_double(), C.c_double(), C.c_uint32(), C.c_uint64()
    check(lib.tpa_artifact_info(h, C.byref(n), C.byref(c), C.byref(eps), C.byref(T), C.byref(fp)))
    scores = np.empty(n.value, np.float64)
    if n.value:
        check(lib.tpa_artifact_scores(h, scores.ctypes.data, 0))
    art = StrangerArtifact(scores, fp.value, c.value, eps.value, T.value)
    if n.value == g.node_count():
        art._dev = (_dev(g), art._key(), h)
    else:
        lib.tpa_artifact_destroy(h)
    return art


def crc32(data, device: int = 0) -> int:
    """CRC-32 of a bytes-like object on the GPU (persistence.cpp:16-32)."""
    buf = np.frombuffer(bytes(data), np.uint8)
    out = C.c_uint32()
    check(lib.tpa_crc32(buf.ctypes.data if buf.size else None, buf.size, 0, int(device), C.byref(out)))
    return out.value
