"""B200-native Cumulative Power Iteration (TPA, arXiv 1708.02574).

The reference's C++ entry points (proj/include/rwrank/{graph,cpi,tpa}.hpp)
mirrored over libtpa_gpu.so: hand-written sm_100a kernels behind the C-ABI in
include/tpa_gpu.h.  No CPU fallback: importing fails if the library is absent.
"""
from ._native import CudaError
from .graph import (DanglingPolicy, DeviceGraph, Graph, dangling_policy_from_string, fingerprint,
                    generate_random_graph, generate_rmat, propagation_sweep, sample_seeds, to_string)
from .partition import PartitionedGraph, PartitionGroup, partition_rows
from .tpa import (CpiParams, CpiResult, SeedSet, StrangerArtifact, TpaParams, cpi_partition, cpi_run,
                  exact_rwr, exact_rwr_batch, kDefaultRestartProb, kDefaultTolerance, neighbor_scale_factor,
                  pagerank, preprocess, query, query_batch, query_batch_topk, query_na, top_k,
                  save_artifact, load_artifact, crc32)

__all__ = [
    "CudaError", "DanglingPolicy", "DeviceGraph", "Graph", "dangling_policy_from_string", "fingerprint",
    "generate_random_graph", "generate_rmat", "propagation_sweep", "sample_seeds", "to_string",
    "CpiParams", "CpiResult", "SeedSet", "StrangerArtifact", "TpaParams", "cpi_partition", "cpi_run",
    "exact_rwr", "exact_rwr_batch", "kDefaultRestartProb", "kDefaultTolerance", "neighbor_scale_factor",
    "pagerank", "preprocess", "query", "query_batch", "query_na", "query_batch_topk", "top_k",
    "save_artifact", "load_artifact", "crc32",
    "PartitionedGraph", "PartitionGroup", "partition_rows",
]
