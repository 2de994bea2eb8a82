"""Row-partitioned CPI across GPUs (csrc/tpa_part.cuh, include/tpa_gpu.h).

The north star's multi-GPU layout for the B = 1 runs (PageRank preprocessing,
cpi_run): the rows of CSR(Ãᵀ) are split into nnz-balanced ranges, one per GPU,
and every sweep ends with one exchange -- an all-reduce of the exact
fixed-point residual / dangling totals and an in-place all-gather of the
iterate's shares.  Results equal the whole-graph run bit for bit.

Two ways to drive it:
  * ``PartitionedGraph`` -- one process per GPU (torch.distributed ranks);
    NCCL inside the library.  Every rank calls the same methods.
  * ``PartitionGroup`` -- one process driving all partitions (peer copies).
Queries (independent seeds) run on whole-graph replicas (``DeviceGraph``).
"""
from __future__ import annotations


import ctypes as C
from typing import Optional, Sequence

import numpy as np

from ._native import check, lib
from . import _native as N
from .graph import Graph, vec_ptr
from .tpa import CpiParams, CpiResult, SeedSet, _terminal

COMM_ID_BYTES = 128
IPC_BLOB_BYTES = 1024  # TPA_IPC_BLOB_BYTES


# SpMV tiling constants (csrc/cpi_kernels.cuh kMvTileNnz / kMvTileRows)
TILE_NNZ, TILE_ROWS = 2048, 512  # the largest tile shape (bounds; tests)
SHAPES = {"S": (1024, 256), "L": (2048, 256)}  # (nnz, rows), cpi_spmv2.cuh


def tile_shape(n: int) -> tuple:
    """(nnz, rows) per SpMV tile for a graph of n nodes (cpi_spmv2.cuh mv_shape)."""
    return SHAPES["L"] if n * 8 > (512 << 20) else SHAPES["S"]


def item_starts(rp: np.ndarray, n: int) -> list:
    """Rows where the whole graph's SpMV tiling (tpa_gpu.cu build_items)
    starts an item: greedy tiles of <= rows rows / tile_nnz nnz, rows
    longer than tile_nnz alone."""
    tile_nnz, rows = tile_shape(n)
    starts, r = [], 0
    while r < n:
        if rp[r + 1] - rp[r] > tile_nnz:
            starts.append(r)
            r += 1
            continue
        start, nnz = r, 0
        while r < n and r - start < rows:
            L = rp[r + 1] - rp[r]
            if L > tile_nnz or (r > start and nnz + L > tile_nnz):
                break
            nnz += L
            r += 1
            if nnz >= tile_nnz:
                break
        starts.append(start)
    return starts


def partition_rows(indeg: np.ndarray, nranks: int) -> np.ndarray:
    """Row boundaries of the library's partitions (tpa_part.cuh partition_rows):
    nnz-balanced, cut only at item starts of the whole graph's tiling, boundary
    k the first cut whose in-degree prefix reaches floor(m*k/G)."""
    indeg = np.asarray(indeg, dtype=np.uint64)
    n = indeg.size
    prefix = np.zeros(n + 1, np.uint64)
    np.cumsum(indeg, out=prefix[1:])
    m = int(prefix[-1])
    rp = prefix.astype(np.int64)
    cuts = np.array(sorted(item_starts(rp, n) + [n]), np.int64)
    cut_prefix = prefix[cuts]
    b = np.zeros(nranks + 1, np.int64)
    b[nranks] = n
    for k in range(1, nranks):
        target = (m * k) // nranks
        i = int(np.searchsorted(cut_prefix, np.uint64(target), side="left"))
        v = int(cuts[i]) if i < cuts.size else n
        b[k] = min(n, max(int(b[k - 1]), v))
    return b


def in_degrees(g: Graph) -> np.ndarray:
    return np.bincount(g.out_targets(), minlength=g.node_count()).astype(np.uint64)


def _prefer_torch_nccl() -> None:
    """Load torch (and its libnccl.so.2) before the library opens NCCL, so the
    process keeps one NCCL, torch's."""
    try:
        import torch  # noqa: F401
    except Exception:
        pass


def comm_unique_id() -> bytes:
    _prefer_torch_nccl()
    buf = C.create_string_buffer(COMM_ID_BYTES)
    check(lib.tpa_comm_unique_id(buf))
    return buf.raw


def _seed_args(seeds: SeedSet, n: int):
    if seeds._ids is None:
        return None, 0, None
    ids = np.ascontiguousarray(seeds._ids, np.uint32) if seeds._ids[-1] <= 0xFFFFFFFF else None
    if ids is None:
        seeds.validate_against(n)
    return ids.ctypes.data, ids.size, ids


class PartitionedGraph:
    """Partition ``rank`` of ``nranks`` of ``g`` on ``device``; collective calls.

    transport "nccl": one in-place NCCL all-gather of the iterate's shares (and
    the exact residual limbs) per sweep.  transport "ipc": the fused exchange --
    every rank's sweep stores its shares straight into the peers' buffers
    (CUDA IPC; ranks may share a device) -- built by ``create_ipc`` +
    ``attach`` (``from_process_group`` does both)."""

    def __init__(self, g: Graph, nranks: int, rank: int, comm_id: Optional[bytes] = None, device: int = 0,
                 transport: str = "nccl"):
        h = C.c_void_p()
        self.blob = None
        if transport == "ipc":
            blob = C.create_string_buffer(IPC_BLOB_BYTES)
            check(lib.tpa_graph_create_part_ipc(g.node_count(), g.edge_count(), g.out_offsets().ctypes.data,
                                                g.out_targets().ctypes.data if g.edge_count() else None,
                                                int(g.dangling_policy()), g.fingerprint(), int(device),
                                                int(nranks), int(rank), blob, C.byref(h)))
            self.blob = blob.raw
        else:
            if comm_id is not None:
                _prefer_torch_nccl()
            idbuf = C.create_string_buffer(comm_id, COMM_ID_BYTES) if comm_id is not None else None
            check(lib.tpa_graph_create_part(g.node_count(), g.edge_count(), g.out_offsets().ctypes.data,
                                            g.out_targets().ctypes.data if g.edge_count() else None,
                                            int(g.dangling_policy()), g.fingerprint(), int(device), int(nranks),
                                            int(rank), idbuf, C.byref(h)))
        self.h = h
        self.n = g.node_count()
        self.fingerprint = g.fingerprint()
        self.transport = transport

    def attach(self, blobs) -> None:
        """IPC transport: every rank's export blob, in rank order."""
        buf = b"".join(bytes(b) for b in blobs)
        check(lib.tpa_part_ipc_attach(self.h, buf))

    @classmethod
    def from_process_group(cls, g: Graph, device: Optional[int] = None, group=None,
                           transport: str = "nccl") -> "PartitionedGraph":
        """One partition per torch.distributed rank: rank 0's NCCL id broadcast,
        or (transport "ipc") every rank's IPC blob all-gathered."""
        import torch.distributed as dist
        nranks, rank = dist.get_world_size(group), dist.get_rank(group)
        if device is None:
            import torch
            device = torch.cuda.current_device()
        if transport == "ipc":
            pg = cls(g, nranks, rank, None, device, transport="ipc")
            blobs = [None] * nranks
            dist.all_gather_object(blobs, pg.blob, group=group)
            pg.attach(blobs)
            dist.barrier(group=group)
            return pg
        obj = [comm_unique_id() if rank == 0 and nranks > 1 else None]
        if nranks > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls(g, nranks, rank, obj[0], device)

    def info(self):
        """(nranks, rank, row_begin, row_end, slice)"""
        v = [C.c_uint32() for _ in range(5)]
        check(lib.tpa_graph_part_info(self.h, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def cpi_run(self, seeds: SeedSet, params: CpiParams) -> CpiResult:
        params.validate()
        out = np.empty(self.n, np.float64)
        it, conv, res = C.c_uint32(), C.c_int(), C.c_double()
        ptr, cnt, _keep = _seed_args(seeds, self.n)
        check(lib.tpa_cpi_run(self.h, ptr, cnt, params.restart_prob, params.tolerance, params.start_iter,
                              _terminal(params.terminal_iter), out.ctypes.data, C.byref(it), C.byref(conv),
                              C.byref(res), 0))
        return CpiResult(out, it.value, bool(conv.value), res.value)

    def pagerank(self, params: CpiParams) -> CpiResult:
        return self.cpi_run(SeedSet.all_nodes(self.n), params)

    def preprocess(self, c: float, eps: float, stranger_start: int) -> np.ndarray:
        """The stranger vector (tpa.cpp:19-37) on every rank."""
        out = np.empty(self.n, np.float64)
        check(lib.tpa_preprocess(self.h, float(c), float(eps), int(stranger_start), out.ctypes.data, None, 0))
        return out

    def close(self):
        if getattr(self, "h", None):
            lib.tpa_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PartitionGroup:
    """All partitions of ``g`` driven by this process, partition r on devices[r]."""

    def __init__(self, g: Graph, devices: Sequence[int]):
        devs = (C.c_int * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        check(lib.tpa_group_create(g.node_count(), g.edge_count(), g.out_offsets().ctypes.data,
                                   g.out_targets().ctypes.data if g.edge_count() else None,
                                   int(g.dangling_policy()), g.fingerprint(), devs, len(devices), C.byref(h)))
        self.h = h
        self.n = g.node_count()
        self.nparts = len(devices)

    def info(self, r: int):
        p = C.c_void_p()
        check(lib.tpa_group_part(self.h, int(r), C.byref(p)))
        v = [C.c_uint32() for _ in range(5)]
        check(lib.tpa_graph_part_info(p, *[C.byref(x) for x in v]))
        return tuple(x.value for x in v)

    def bounds(self) -> np.ndarray:
        return np.array([self.info(r)[2] for r in range(self.nparts)] + [self.n], np.int64)

    def cpi_run(self, seeds: SeedSet, params: CpiParams) -> CpiResult:
        params.validate()
        out = np.empty(self.n, np.float64)
        it, conv, res = C.c_uint32(), C.c_int(), C.c_double()
        ptr, cnt, _keep = _seed_args(seeds, self.n)
        check(lib.tpa_group_cpi_run(self.h, ptr, cnt, params.restart_prob, params.tolerance, params.start_iter,
                                    _terminal(params.terminal_iter), out.ctypes.data, C.byref(it), C.byref(conv),
                                    C.byref(res)))
        return CpiResult(out, it.value, bool(conv.value), res.value)

    def pagerank(self, params: CpiParams) -> CpiResult:
        return self.cpi_run(SeedSet.all_nodes(self.n), params)

    def preprocess(self, c: float, eps: float, stranger_start: int) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        check(lib.tpa_group_preprocess(self.h, float(c), float(eps), int(stranger_start), out.ctypes.data))
        return out

    def query_batch(self, artifact, seeds, family_end: int, out=None, na: bool = False, params=None):
        """query / query_na (tpa.cpp:61-86) for a batch of seeds on the partitioned
        graph; ``artifact`` is a StrangerArtifact (ignored with ``na``, which takes
        ``params`` = TpaParams).  Returns [B][n] (numpy, or fills a CUDA tensor)."""
        from .tpa import _seed_array
        s = _seed_array(seeds, self.n)
        B = int(s.size)
        if out is None:
            out = np.empty((B, self.n), np.float64)
        p, dev, keep = vec_ptr(out, B * self.n, writable=True)
        flags = (N.TPA_DEVICE_PTRS if dev else 0) | (N.TPA_QUERY_NA if na else 0)
        if na:
            prm = params
            check(lib.tpa_group_query_batch(self.h, None, 0, float(prm.restart_prob), float(prm.tolerance),
                                            int(prm.stranger_start), s.ctypes.data, B, int(family_end), p, flags))
        else:
            st = np.ascontiguousarray(artifact.stranger_scores, np.float64)
            if st.size != self.n:
                raise ValueError("stranger vector length does not match node count")
            check(lib.tpa_group_query_batch(self.h, st.ctypes.data, int(artifact.graph_fingerprint),
                                            float(artifact.restart_prob), float(artifact.tolerance),
                                            int(artifact.stranger_start), s.ctypes.data, B, int(family_end), p,
                                            flags))
        return out

    def close(self):
        if getattr(self, "h", None):
            lib.tpa_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
