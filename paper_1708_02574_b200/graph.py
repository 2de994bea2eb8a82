"""Graph type and host-side input plumbing (mirror of proj/include/rwrank/graph.hpp).

``Graph`` has the reference's construction semantics (graph.cpp:53-91) and
accessors (graph.hpp:26-66); it is built by the native library's host code.
``Graph.device()`` returns the device-resident CSR(Ãᵀ) handle (the GPU ingest,
SURVEY §8(a) row A2), created once per graph and device and reused by every
entry point -- the analogue of the reference passing ``const Graph&`` around.
``propagation_sweep`` is graph.hpp:96-103 on the GPU.
"""
from __future__ import annotations

import ctypes as C
import enum

import numpy as np

from . import _native as N
from ._native import check, lib


class DanglingPolicy(enum.IntEnum):
    """graph.hpp:17-19 (declaration order = ABI value)."""
    SelfLoop = 0
    Uniform = 1
    Drop = 2


def to_string(policy: DanglingPolicy) -> str:
    """graph.cpp:37-44"""
    return {DanglingPolicy.SelfLoop: "selfloop", DanglingPolicy.Uniform: "uniform",
            DanglingPolicy.Drop: "drop"}.get(DanglingPolicy(policy), "unknown")


def dangling_policy_from_string(name: str) -> DanglingPolicy:
    """graph.cpp:46-51"""
    table = {"selfloop": DanglingPolicy.SelfLoop, "uniform": DanglingPolicy.Uniform,
             "drop": DanglingPolicy.Drop}
    if name not in table:
        raise ValueError("unknown dangling policy: " + name)
    return table[name]


def _policy(p) -> DanglingPolicy:
    return dangling_policy_from_string(p) if isinstance(p, str) else DanglingPolicy(int(p))


class Graph:
    """Immutable out-edge CSR graph (graph.hpp:26-66)."""

    def __init__(self, node_count: int, edges, policy=DanglingPolicy.SelfLoop):
        """``edges``: iterable of (u, v) pairs or a (src, dst) pair of arrays.
        Throws ValueError on node_count == 0 and IndexError on an endpoint >=
        node_count, like the reference constructor (graph.cpp:55-61)."""
        src, dst = _edge_arrays(edges)
        if node_count < 0 or node_count > 0xFFFFFFFF:
            raise ValueError("node_count out of uint32 range")
        h = C.c_void_p()
        check(lib.tpa_host_graph_from_edges(int(node_count), src.ctypes.data, dst.ctypes.data,
                                            len(src), int(_policy(policy)), C.byref(h)))
        self._adopt(h)

    @classmethod
    def build_gpu(cls, node_count: int, edges, policy=DanglingPolicy.SelfLoop, device: int = 0) -> "Graph":
        """The constructor's work (graph.cpp:53-91) on the GPU (sort, dedupe,
        dangling list, SelfLoop repair, out-CSR); FNV-1a on the host.  Same
        result and errors as ``Graph(node_count, edges, policy)``."""
        src, dst = _edge_arrays(edges)
        if node_count < 0 or node_count > 0xFFFFFFFF:
            raise ValueError("node_count out of uint32 range")
        h = C.c_void_p()
        check(lib.tpa_host_graph_build_gpu(int(node_count), src.ctypes.data, dst.ctypes.data, len(src),
                                           int(_policy(policy)), int(device), C.byref(h)))
        return cls._from_handle(h)

    @classmethod
    def _from_handle(cls, h) -> "Graph":
        g = cls.__new__(cls)
        g._adopt(h)
        return g

    def _adopt(self, h) -> None:
        n, m, nd, fp, pol = C.c_uint32(), C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        lib.tpa_host_graph_info(h, C.byref(n), C.byref(m), C.byref(nd), C.byref(fp), C.byref(pol))
        self._h = h
        self._n, self._m, self._fp = n.value, m.value, fp.value
        self._policy = DanglingPolicy(pol.value)
        # zero-copy views of the native arrays (the handle owns them)
        self._off = _view(lib.tpa_host_graph_offsets(h), self._n + 1, np.uint64)
        self._tgt = _view(lib.tpa_host_graph_targets(h), self._m, np.uint32)
        self._dang = _view(lib.tpa_host_graph_dangling(h), nd.value, np.uint32)
        self._dev = {}

    def __del__(self):
        # Device handles close themselves once nothing (e.g. an artifact)
        # references them any more.
        try:
            self._dev.clear()
            lib.tpa_host_graph_destroy(self._h)
        except Exception:
            pass

    # --- graph.hpp accessors ------------------------------------------------
    def node_count(self) -> int:
        return self._n

    def edge_count(self) -> int:
        return self._m

    def dangling_policy(self) -> DanglingPolicy:
        return self._policy

    def out_degree(self, u: int) -> int:
        return int(self._off[u + 1] - self._off[u])

    def out_neighbors(self, u: int) -> np.ndarray:
        return self._tgt[int(self._off[u]):int(self._off[u + 1])]

    def out_offsets(self) -> np.ndarray:
        return self._off

    def out_targets(self) -> np.ndarray:
        return self._tgt

    def dangling_nodes(self) -> np.ndarray:
        return self._dang

    def fingerprint(self) -> int:
        return self._fp

    def __eq__(self, other) -> bool:  # graph.cpp:93-96
        return (isinstance(other, Graph) and self._n == other._n and self._policy == other._policy
                and np.array_equal(self._off, other._off) and np.array_equal(self._tgt, other._tgt))

    def device(self, device: int = 0) -> "DeviceGraph":
        """The device-resident CSR(Ãᵀ) of this graph on `device` (built once)."""
        d = self._dev.get(device)
        if d is None:
            d = DeviceGraph(self, device)
            self._dev[device] = d
        return d


def _view(ptr, count, dtype):
    if count == 0:
        return np.empty(0, dtype)
    buf = (C.c_byte * (count * np.dtype(dtype).itemsize)).from_address(ptr)
    a = np.frombuffer(buf, dtype=dtype, count=count)
    a.flags.writeable = False
    return a


def _edge_arrays(edges):
    """(src, dst) uint32 arrays from a sequence of (u, v) pairs, an (m, 2)
    array, or a tuple of two 1-D numpy arrays."""
    if (isinstance(edges, tuple) and len(edges) == 2 and isinstance(edges[0], np.ndarray)
            and edges[0].ndim == 1):
        src = np.asarray(edges[0], dtype=np.int64)
        dst = np.asarray(edges[1], dtype=np.int64)
    else:
        arr = np.asarray(edges if isinstance(edges, np.ndarray) else list(edges), dtype=np.int64)
        arr = arr.reshape(-1, 2)
        src, dst = arr[:, 0], arr[:, 1]
    if src.size and (min(src.min(), dst.min()) < 0 or max(src.max(), dst.max()) > 0xFFFFFFFF):
        raise IndexError("edge endpoint out of range")
    return np.ascontiguousarray(src, np.uint32), np.ascontiguousarray(dst, np.uint32)


def generate_random_graph(node_count: int, edge_count: int, rng_seed: int,
                          policy=DanglingPolicy.SelfLoop) -> Graph:
    """graph.hpp:88-94 / graph.cpp:166-205 semantics (same mt19937_64 stream)."""
    h = C.c_void_p()
    check(lib.tpa_host_graph_random(int(node_count), int(edge_count), int(rng_seed), int(_policy(policy)),
                                    C.byref(h)))
    return Graph._from_handle(h)


def generate_rmat(scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19, c: float = 0.19,
                  rng_seed: int = 1, policy=DanglingPolicy.SelfLoop, threads: int = 0,
                  device: int | None = None) -> Graph:
    """R-MAT (BASELINE configs C1/C2/C4/C5): 2^scale nodes, edge_factor*2^scale raw
    edges, quadrant recursion without noise or permutation, self-loops dropped,
    duplicates removed by the Graph construction, dangling nodes kept.

    ``device``: generate and construct on that GPU (same edge streams, so the
    same graph and fingerprint; needed for the billion-edge scales)."""
    h = C.c_void_p()
    if device is not None:
        check(lib.tpa_host_graph_rmat_gpu(int(scale), int(edge_factor), a, b, c, int(rng_seed),
                                          int(_policy(policy)), int(device), C.byref(h)))
        return Graph._from_handle(h)
    check(lib.tpa_host_graph_rmat(int(scale), int(edge_factor), a, b, c, int(rng_seed), int(_policy(policy)),
                                  int(threads), C.byref(h)))
    return Graph._from_handle(h)


def sample_seeds(g: Graph, count: int, rng_seed: int) -> np.ndarray:
    """rwrank_main.cpp:65-83: uniform sample without replacement of non-dangling nodes."""
    out = np.empty(int(count), np.uint32)
    check(lib.tpa_sample_seeds(g._h, int(count), int(rng_seed), out.ctypes.data))
    return out


def fingerprint(n, off, tgt, policy) -> int:
    off = np.ascontiguousarray(off, np.uint64)
    tgt = np.ascontiguousarray(tgt, np.uint32)
    return lib.tpa_fingerprint(int(n), len(tgt), off.ctypes.data, tgt.ctypes.data, int(_policy(policy)))


# ---------------------------------------------------------------------------
# device handle
# ---------------------------------------------------------------------------
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def vec_ptr(x, count=None, dtype=np.float64, writable=False, device=None):
    """(pointer, is_device, keepalive) for a numpy array or torch tensor.

    Tensors must be contiguous, of exactly `dtype` and, when on a GPU, on
    `device` (the graph's).  A numpy *input* may be converted (a copy); an
    output (`writable`) must already be a C-contiguous, writeable array of
    `dtype` -- results are written straight into it, never into a temporary."""
    if _is_torch(x):
        import torch
        want = {np.dtype(np.float64): torch.float64, np.dtype(np.uint32): torch.int32,
                np.dtype(np.int32): torch.int32}[np.dtype(dtype)]
        if x.dtype != want:
            raise TypeError(f"tensor must be {want}, got {x.dtype}")
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        if count is not None and x.numel() != count:
            raise ValueError("score vector length does not match node count")
        if x.is_cuda and device is not None and x.device.index != int(device):
            raise ValueError(f"tensor is on cuda:{x.device.index}, the graph on cuda:{int(device)}")
        return x.data_ptr(), x.is_cuda, x
    if writable:
        if not isinstance(x, np.ndarray) or x.dtype != np.dtype(dtype) or not x.flags.c_contiguous \
                or not x.flags.writeable:
            raise ValueError(f"output must be a writeable C-contiguous {np.dtype(dtype)} array")
        a = x
    else:
        a = np.ascontiguousarray(x, dtype)
    if count is not None and a.size != count:
        raise ValueError("score vector length does not match node count")
    return a.ctypes.data, False, a


class DeviceGraph:
    """Owner of a tpa_graph* (device CSR(Ãᵀ), schedules and workspaces)."""

    def __init__(self, g: Graph, device: int = 0):
        h = C.c_void_p()
        check(lib.tpa_graph_create(g.node_count(), g.edge_count(), g.out_offsets().ctypes.data,
                                   g.out_targets().ctypes.data if g.edge_count() else None,
                                   int(g.dangling_policy()), g.fingerprint(), int(device), C.byref(h)))
        self.h = h
        self.device = device
        self.n = g.node_count()
        self.m = g.edge_count()
        self.fingerprint = g.fingerprint()

    def close(self):
        if getattr(self, "h", None):
            lib.tpa_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None) -> None:
        check(lib.tpa_graph_set_stream(self.h, stream_ptr))

    def launches(self) -> int:
        return int(lib.tpa_graph_launches(self.h))

    def profile(self, enable: bool) -> None:
        """Start (True) or stop (False) per-sweep-kernel CUDA-event timing."""
        check(lib.tpa_graph_profile(self.h, 1 if enable else 0))

    def profile_read(self, width: int, step: int = -1):
        """(launches, total_ms) of the sweep kernel of batch width `width`
        producing x^(step) (-1: every sweep)."""
        n, ms = C.c_uint64(), C.c_double()
        check(lib.tpa_graph_profile_read(self.h, int(width), int(step), C.byref(n), C.byref(ms)))
        return n.value, ms.value

    def device_bytes(self) -> int:
        b = C.c_uint64()
        check(lib.tpa_graph_info(self.h, None, None, None, None, C.byref(b)))
        return b.value

    def transpose(self):
        rp = np.empty(self.n + 1, np.int64)
        col = np.empty(self.m, np.uint32)
        check(lib.tpa_graph_transpose(self.h, rp.ctypes.data, col.ctypes.data))
        return rp, col


def propagation_sweep(g: Graph, x, c: float, threads: int = 1, out=None):
    """graph.hpp:96-103: y = (1-c)·Ãᵀx (+ dangling term), on the GPU.
    ``threads`` is accepted for signature parity and ignored."""
    n = g.node_count()
    xdev0 = _is_torch(x) and x.is_cuda
    dev = x.device.index if xdev0 else 0
    xp, xdev, keep_x = vec_ptr(x, n, device=dev)
    if out is None:
        if xdev:
            import torch
            out = torch.empty(n, dtype=torch.float64, device=x.device)
        else:
            out = np.empty(n, np.float64)
    yp, ydev, keep_y = vec_ptr(out, n, writable=True, device=dev)
    if xdev != ydev:
        raise ValueError("x and y must both be host or both be device vectors")
    check(lib.tpa_propagation_sweep(g.device(dev).h, xp, yp, float(c),
                                    N.TPA_DEVICE_PTRS if xdev else 0))
    return out
