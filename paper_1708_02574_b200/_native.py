"""ctypes binding of libtpa_gpu.so (the C-ABI declared in include/tpa_gpu.h).

There is no fallback: if the shared library is missing this module raises at
import time, and every compute call goes to the CUDA kernels behind it.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libtpa_gpu.so")

TPA_OK = 0
TPA_ERR_INVALID_ARGUMENT = 1
TPA_ERR_OUT_OF_RANGE = 2
TPA_ERR_RUNTIME = 3
TPA_ERR_CUDA = 4
TPA_ERR_ALLOC = 5

TPA_DEVICE_PTRS = 1
TPA_ASYNC = 2
TPA_NODE_MAJOR = 4
TPA_QUERY_NA = 8

# Every symbol include/tpa_gpu.h declares, with its ctypes signature.
_vp = C.c_void_p
_u32, _u64, _i64, _int, _dbl = C.c_uint32, C.c_uint64, C.c_int64, C.c_int, C.c_double
SIGNATURES = {
    "tpa_abi_version": ([], _int),
    "tpa_last_error": ([], C.c_char_p),
    "tpa_graph_create": ([_u32, _u64, _vp, _vp, _int, _u64, _int, C.POINTER(_vp)], _int),
    "tpa_graph_destroy": ([_vp], _int),
    "tpa_graph_set_stream": ([_vp, _vp], _int),
    "tpa_graph_sync": ([_vp], _int),
    "tpa_graph_info": ([_vp, C.POINTER(_u32), C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_int),
                        C.POINTER(_u64)], _int),
    "tpa_graph_launches": ([_vp], _u64),
    "tpa_graph_profile": ([_vp, _int], _int),
    "tpa_graph_profile_read": ([_vp, _int, _int, C.POINTER(_u64), C.POINTER(_dbl)], _int),
    "tpa_graph_transpose": ([_vp, _vp, _vp], _int),
    "tpa_propagation_sweep": ([_vp, _vp, _vp, _dbl, _int], _int),
    "tpa_cpi_run": ([_vp, _vp, _u64, _dbl, _dbl, _u32, _i64, _vp, C.POINTER(_u32), C.POINTER(_int),
                     C.POINTER(_dbl), _int], _int),
    "tpa_cpi_partition": ([_vp, _vp, _u64, _dbl, _dbl, _vp, _u64, _vp, _int], _int),
    "tpa_exact_rwr_batch": ([_vp, _vp, _u32, _dbl, _dbl, _vp, _int], _int),
    "tpa_neighbor_scale_factor": ([_dbl, _u32, _u32], _dbl),
    "tpa_preprocess": ([_vp, _dbl, _dbl, _u32, _vp, C.POINTER(_vp), _int], _int),
    "tpa_artifact_create": ([_vp, _vp, _u64, _dbl, _dbl, _u32, _int, C.POINTER(_vp)], _int),
    "tpa_artifact_destroy": ([_vp], _int),
    "tpa_query": ([_vp, _vp, _u32, _u32, _vp, _int], _int),
    "tpa_query_batch": ([_vp, _vp, _vp, _u32, _u32, _vp, _int], _int),
    "tpa_query_na_batch": ([_vp, _vp, _u32, _u32, _u32, _dbl, _dbl, _vp, _int], _int),
    "tpa_artifact_save": ([_vp, C.c_char_p], _int),
    "tpa_artifact_load": ([_vp, C.c_char_p, C.POINTER(_vp)], _int),
    "tpa_artifact_info": ([_vp, C.POINTER(_u64), C.POINTER(_dbl), C.POINTER(_dbl), C.POINTER(_u32),
                           C.POINTER(_u64)], _int),
    "tpa_artifact_scores": ([_vp, _vp, _int], _int),
    "tpa_crc32": ([_vp, _u64, _int, _int, C.POINTER(_u32)], _int),
    "tpa_top_k": ([_vp, _vp, _u32, _u32, _vp, _vp, _int], _int),
    "tpa_query_batch_topk": ([_vp, _vp, _vp, _u32, _u32, _u32, _vp, _vp, _int], _int),
    "tpa_comm_unique_id": ([_vp], _int),
    "tpa_graph_create_part": ([_u32, _u64, _vp, _vp, _int, _u64, _int, _u32, _u32, _vp, C.POINTER(_vp)], _int),
    "tpa_graph_create_part_ipc": ([_u32, _u64, _vp, _vp, _int, _u64, _int, _u32, _u32, _vp, C.POINTER(_vp)],
                                  _int),
    "tpa_part_ipc_attach": ([_vp, _vp], _int),
    "tpa_graph_part_info": ([_vp, C.POINTER(_u32), C.POINTER(_u32), C.POINTER(_u32), C.POINTER(_u32),
                             C.POINTER(_u32)], _int),
    "tpa_group_create": ([_u32, _u64, _vp, _vp, _int, _u64, _vp, _u32, C.POINTER(_vp)], _int),
    "tpa_group_destroy": ([_vp], _int),
    "tpa_group_part": ([_vp, _u32, C.POINTER(_vp)], _int),
    "tpa_group_cpi_run": ([_vp, _vp, _u64, _dbl, _dbl, _u32, _i64, _vp, C.POINTER(_u32), C.POINTER(_int),
                           C.POINTER(_dbl)], _int),
    "tpa_group_preprocess": ([_vp, _dbl, _dbl, _u32, _vp], _int),
    "tpa_group_query_batch": ([_vp, _vp, _u64, _dbl, _dbl, _u32, _vp, _u32, _u32, _vp, _int], _int),
    "tpa_host_graph_from_edges": ([_u32, _vp, _vp, _u64, _int, C.POINTER(_vp)], _int),
    "tpa_host_graph_build_gpu": ([_u32, _vp, _vp, _u64, _int, _int, C.POINTER(_vp)], _int),
    "tpa_host_graph_rmat_gpu": ([_u32, _u32, _dbl, _dbl, _dbl, _u64, _int, _int, C.POINTER(_vp)], _int),
    "tpa_host_graph_rmat": ([_u32, _u32, _dbl, _dbl, _dbl, _u64, _int, _int, C.POINTER(_vp)], _int),
    "tpa_host_graph_random": ([_u32, _u64, _u64, _int, C.POINTER(_vp)], _int),
    "tpa_host_graph_destroy": ([_vp], None),
    "tpa_host_graph_info": ([_vp, C.POINTER(_u32), C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64),
                             C.POINTER(_int)], None),
    "tpa_host_graph_offsets": ([_vp], _vp),
    "tpa_host_graph_targets": ([_vp], _vp),
    "tpa_host_graph_dangling": ([_vp], _vp),
    "tpa_sample_seeds": ([_vp, _u64, _u64, _vp], _int),
    "tpa_fingerprint": ([_u32, _u64, _vp, _vp, _int], _u64),
}


class CudaError(RuntimeError):
    """A device or driver failure (no counterpart in the reference)."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python paper_1708_02574_b200/build.py` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in SIGNATURES.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    if lib.tpa_abi_version() != 1:
        raise ImportError("libtpa_gpu.so ABI version mismatch")
    return lib


lib = _load()


def check(rc: int) -> None:
    """Raise the Python counterpart of the reference's exception type."""
    if rc == TPA_OK:
        return
    msg = lib.tpa_last_error().decode(errors="replace")
    if rc == TPA_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if rc == TPA_ERR_OUT_OF_RANGE:
        raise IndexError(msg)  # std::out_of_range
    if rc == TPA_ERR_RUNTIME:
        raise RuntimeError(msg)  # std::runtime_error
    if rc == TPA_ERR_ALLOC:
        raise MemoryError(msg)
    raise CudaError(msg)
