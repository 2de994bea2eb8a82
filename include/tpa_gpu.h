/*
 * tpa_gpu.h -- C-ABI of the B200-native CPI engine (libtpa_gpu.so).
 *
 * Drop-in boundary for the reference's hot path: the C++ entry points of
 * /root/reference/proj/include/rwrank/{cpi,tpa,graph}.hpp.  Every function
 * below names the reference interface it replaces.  Plain pointers and sizes
 * only: no C++ or torch types cross this boundary.
 *
 * Status codes mirror the reference's exception types:
 *   TPA_OK                    0
 *   TPA_ERR_INVALID_ARGUMENT  1  std::invalid_argument
 *   TPA_ERR_OUT_OF_RANGE      2  std::out_of_range
 *   TPA_ERR_RUNTIME           3  std::runtime_error ("stale artifact: ...")
 *   TPA_ERR_CUDA              4  device/driver failure
 *   TPA_ERR_ALLOC             5  device allocation failure
 * The message of the last failure on the calling thread is tpa_last_error();
 * parameter errors use the reference's own message text.
 *
 * Threading: a tpa_graph serialises its own calls (one stream per handle);
 * results are deterministic, so concurrent callers get bitwise-identical
 * vectors (tpa_test.cpp:148-161).  The reference's `threads` argument selects
 * host parallelism; here it has no meaning and is not taken.
 *
 * Memory: unless TPA_DEVICE_PTRS is set, vector (double) arguments are host
 * pointers (pinned or pageable).  With TPA_DEVICE_PTRS they are device
 * pointers on the handle's device and the call returns without a host
 * synchronisation when nothing has to come back to the host (TPA_ASYNC).
 * Seed and boundary lists are ALWAYS host arrays: they are validated on the
 * host before any launch (the reference's error order) and travel to the
 * device as kernel parameters.
 */
#ifndef TPA_GPU_H
#define TPA_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPA_ABI_VERSION 1

enum tpa_status {
    TPA_OK = 0,
    TPA_ERR_INVALID_ARGUMENT = 1,
    TPA_ERR_OUT_OF_RANGE = 2,
    TPA_ERR_RUNTIME = 3,
    TPA_ERR_CUDA = 4,
    TPA_ERR_ALLOC = 5
};

/* rwrank::DanglingPolicy (graph.hpp:19), declaration order. */
enum tpa_policy { TPA_SELFLOOP = 0, TPA_UNIFORM = 1, TPA_DROP = 2 };

enum tpa_flags {
    TPA_DEVICE_PTRS = 1,  /* vector in/out arguments are device pointers */
    TPA_ASYNC = 2,        /* do not synchronise on return (device outputs; batch calls' host
                             outputs drain asynchronously: tpa_graph_sync before reading) */
    TPA_NODE_MAJOR = 4,   /* batch output laid out [n][B] instead of [B][n] */
    TPA_QUERY_NA = 8      /* query_batch: no stranger term (tpa.cpp:78-86) */
};

typedef struct tpa_graph tpa_graph;       /* device-resident CSR(A^T) + workspaces */
typedef struct tpa_artifact tpa_artifact; /* device-resident StrangerArtifact */

int tpa_abi_version(void);
const char *tpa_last_error(void);

/* --- graph ---------------------------------------------------------------
 * Replaces: the rwrank::Graph a caller hands to every entry point
 * (graph.hpp:26-66).  Input is the reference Graph's out-edge CSR exactly as
 * out_offsets()/out_targets() return it (graph.hpp:45-46): sorted, deduped,
 * SelfLoop repair edges included; policy = dangling_policy(); fingerprint =
 * fingerprint() (graph.hpp:56).  The GPU ingest builds CSR(A^T) with
 * ascending sources per row, the out-degree array and the work schedules.
 * out_offsets/out_targets are host pointers. */
int tpa_graph_create(uint32_t n, uint64_t m, const uint64_t *out_offsets,
                     const uint32_t *out_targets, int policy, uint64_t fingerprint, int device,
                     tpa_graph **out);
int tpa_graph_destroy(tpa_graph *g);
/* Make the handle enqueue on an external cudaStream_t (NULL: its own stream). */
/* Waits for every call enqueued on the handle (TPA_ASYNC), including the
 * device-to-host drains of batch calls with host outputs: those compute chunk
 * k+1 while chunk k drains over PCIe (two device staging buffers). */
int tpa_graph_sync(tpa_graph *g);
int tpa_graph_set_stream(tpa_graph *g, void *cuda_stream);
int tpa_graph_info(const tpa_graph *g, uint32_t *n, uint64_t *m, uint64_t *fingerprint,
                   int *policy, uint64_t *device_bytes);
/* Number of kernels this handle has launched so far (instrumentation). */
uint64_t tpa_graph_launches(const tpa_graph *g);
/* Bench instrumentation: while enabled, every CPI sweep kernel launch is
 * bracketed by CUDA events on the handle's stream.  enable != 0 starts a new
 * session.  profile_read sums the recorded launches of the sweep kernel of a
 * given batch width (1 = SpMV; 8/16/32/64 = SpMM) and sweep index `step`
 * (x^(step) produced; -1 = all sweeps); it synchronises. */
int tpa_graph_profile(tpa_graph *g, int enable);
int tpa_graph_profile_read(tpa_graph *g, int width, int step, uint64_t *launches, double *total_ms);
/* Device copy of CSR(A^T) for inspection: row_ptr[n+1] (int64), col[m]. Host ptrs. */
int tpa_graph_transpose(const tpa_graph *g, int64_t *row_ptr, uint32_t *col);

/* --- one sweep ------------------------------------------------------------
 * Replaces: propagation_sweep(g, x, y, c) (graph.hpp:96-103, graph.cpp:230-270).
 * x, y: n doubles.  0 <= c < 1 else TPA_ERR_INVALID_ARGUMENT. */
int tpa_propagation_sweep(tpa_graph *g, const double *x, double *y, double c, int flags);

/* --- CPI -------------------------------------------------------------------
 * Replaces: cpi_run(g, SeedSet(seeds), CpiParams{c, eps, start, terminal})
 * (cpi.hpp:49, cpi.cpp:87-101); with seeds == NULL: pagerank(g, params)
 * (cpi.hpp:57, cpi.cpp:111-113).  terminal_iter < 0 means nullopt.
 * seeds need not be sorted; empty or duplicate -> INVALID_ARGUMENT
 * (cpi.cpp:19-24); any seed >= n -> OUT_OF_RANGE (cpi.cpp:34-39).
 * out_scores: n doubles; the other outputs may be NULL. */
int tpa_cpi_run(tpa_graph *g, const uint32_t *seeds, uint64_t n_seeds, double c, double eps,
                uint32_t start_iter, int64_t terminal_iter, double *out_scores,
                uint32_t *iterations_run, int *converged, double *residual_l1, int flags);

/* Replaces: cpi_partition(g, seeds, c, eps, boundaries) (cpi.hpp:60-62,
 * cpi.cpp:115-136).  out: (n_boundaries + 1) x n doubles, segment-major. */
int tpa_cpi_partition(tpa_graph *g, const uint32_t *seeds, uint64_t n_seeds, double c, double eps,
                      const uint32_t *boundaries, uint64_t n_boundaries, double *out, int flags);

/* Batched extension of exact_rwr (cpi.hpp:53-54, cpi.cpp:103-109): B
 * independent full-window single-seed runs.  out: [B][n] (or [n][B]). */
int tpa_exact_rwr_batch(tpa_graph *g, const uint32_t *seeds, uint32_t B, double c, double eps,
                        double *out, int flags);

/* --- TPA -------------------------------------------------------------------
 * Replaces: neighbor_scale_factor (tpa.hpp:32, tpa.cpp:39-44). */
double tpa_neighbor_scale_factor(double c, uint32_t S, uint32_t T);

/* Replaces: preprocess(g, c, eps, T) (tpa.hpp:27-28, tpa.cpp:19-37).
 * T < 1 -> INVALID_ARGUMENT.  out_stranger (n doubles) and out_artifact may
 * each be NULL; the artifact stays on the device for tpa_query*. */
int tpa_preprocess(tpa_graph *g, double c, double eps, uint32_t T, double *out_stranger,
                   tpa_artifact **out_artifact, int flags);

/* A device artifact from a host (or device) StrangerArtifact (tpa.hpp:17-23). */
int tpa_artifact_create(tpa_graph *g, const double *stranger, uint64_t graph_fingerprint, double c,
                        double eps, uint32_t T, int flags, tpa_artifact **out);
int tpa_artifact_destroy(tpa_artifact *a);

/* Replaces: query(g, artifact, seed, S) (tpa.hpp:37-38, tpa.cpp:61-76).
 * Fingerprint mismatch -> RUNTIME "stale artifact: graph fingerprint
 * mismatch"; S < 1 or S >= artifact T -> INVALID_ARGUMENT.  out: n doubles. */
int tpa_query(tpa_graph *g, const tpa_artifact *a, uint32_t seed, uint32_t S, double *out,
              int flags);

/* B independent query() calls in one batched CPI (SpMM over B seeds).  Same
 * validation as tpa_query, in the same order.  out: [B][n] unless
 * TPA_NODE_MAJOR.  With TPA_QUERY_NA the stranger term is omitted and `a`
 * only supplies c, eps, T (it may then be NULL: see tpa_query_na_batch). */
int tpa_query_batch(tpa_graph *g, const tpa_artifact *a, const uint32_t *seeds, uint32_t B,
                    uint32_t S, double *out, int flags);

/* Replaces: query_na(g, seed, TpaParams{S, T, c, eps}) (tpa.hpp:41,
 * tpa.cpp:78-86), batched over B seeds (B = 1 is query_na itself). */
int tpa_query_na_batch(tpa_graph *g, const uint32_t *seeds, uint32_t B, uint32_t S, uint32_t T,
                       double c, double eps, double *out, int flags);

/* --- artifact I/O from device buffers -------------------
 * Replaces: save_artifact / load_artifact (persistence.hpp, persistence.cpp:
 * 69-125), the file format unchanged (48 + 8n bytes, CRC-32 trailer); the
 * CRC-32 runs on the GPU.  Errors: the reference's std::runtime_error texts
 * (TPA_ERR_RUNTIME), checked in the reference's order.  A loaded artifact is
 * bound to graph g (its fingerprint is checked by the queries, tpa.cpp:63-64). */
int tpa_artifact_save(const tpa_artifact *a, const char *path);
int tpa_artifact_load(tpa_graph *g, const char *path, tpa_artifact **out);
int tpa_artifact_info(const tpa_artifact *a, uint64_t *n, double *c, double *eps, uint32_t *T,
                      uint64_t *fingerprint);
/* the stranger scores (n doubles; host, or device with TPA_DEVICE_PTRS) */
int tpa_artifact_scores(const tpa_artifact *a, double *out, int flags);
/* CRC-32 (persistence.cpp:16-32) of `size` bytes on the GPU (data host, or
 * device with TPA_DEVICE_PTRS). */
int tpa_crc32(const void *data, uint64_t size, int flags, int device, uint32_t *out);

/* --- top-k on the device --------------------------------
 * Replaces: top_k_nodes(scores, k) (metrics.hpp:17, metrics.cpp:25-36) for B
 * vectors: score descending, equal scores by ascending node id; k in [1, n]
 * else TPA_ERR_OUT_OF_RANGE ("k must be in [1, n], got k").  scores: [B][n]
 * (what tpa_query_batch writes); out_ids / out_scores: [B][k] (out_scores may
 * be NULL).  All arrays host, or device with TPA_DEVICE_PTRS. */
int tpa_top_k(tpa_graph *g, const double *scores, uint32_t B, uint32_t k, uint32_t *out_ids,
              double *out_scores, int flags);
/* tpa_query_batch (or, with TPA_QUERY_NA, the artifact-free query_na using the
 * artifact's c / eps / T) followed by tpa_top_k on the device: only B*k results
 * leave the GPU (the CLI's query output, rwrank_main.cpp:158-165). */
int tpa_query_batch_topk(tpa_graph *g, const tpa_artifact *a, const uint32_t *seeds, uint32_t B,
                         uint32_t S, uint32_t k, uint32_t *out_ids, double *out_scores, int flags);

/* --- multi-GPU: row-partitioned CPI (B = 1) ---------------------------------
 * The north star's multi-GPU layout: the rows of CSR(Ãᵀ) are split into
 * nnz-balanced ranges, one per GPU; each sweep is the single-GPU kernel on
 * the partition's rows followed by an all-reduce of the exact fixed-point
 * residual / dangling totals and an in-place all-gather of the iterate's
 * shares.  Results equal the whole-graph run bit for bit (the totals are
 * exact integers and the per-row arithmetic is unchanged).
 * Replaces, per rank: cpi_run / pagerank (cpi.hpp:49-57) and preprocess's
 * stranger vector (tpa.hpp:27-28); queries run on whole-graph replicas
 * (tpa_graph_create) since each seed is independent. */
#define TPA_COMM_ID_BYTES 128

/* A fresh NCCL unique id (rank 0 creates it and sends it to the others). */
int tpa_comm_unique_id(void *id_out /* TPA_COMM_ID_BYTES */);

/* One process per GPU: partition `rank` of `nranks`; collective over the
 * ranks (NCCL communicator built from comm_id).  nranks = 1 needs no id.
 * tpa_cpi_run and tpa_preprocess (no artifact) on this handle are collective
 * calls: every rank passes the same arguments and receives the full n-vector;
 * the other compute entry points refuse a partition.  tpa_graph_info reports
 * the graph's n and m. */
int tpa_graph_create_part(uint32_t n, uint64_t m, const uint64_t *out_offsets,
                          const uint32_t *out_targets, int policy, uint64_t fingerprint, int device,
                          uint32_t nranks, uint32_t rank, const void *comm_id, tpa_graph **out);
/* One process per GPU over CUDA IPC: the fused exchange.  Each rank's SpMV
 * epilogue stores its shares (and its exact residual limbs) straight into
 * every peer's share buffer -- over NVLink between GPUs -- so the exchange
 * overlaps the sweep instead of following it as a collective.  Two steps:
 * create (every rank; fills its TPA_IPC_BLOB_BYTES export blob), exchange the
 * blobs out of band (e.g. torch.distributed all_gather_object), then attach
 * with all nranks blobs in rank order.  Ranks may share a device (the stream
 * waits are interprocess events, no kernel waits on another).  Calls as for
 * tpa_graph_create_part; 1..16 ranks.  Same results as one GPU, bit for bit. */
#define TPA_IPC_BLOB_BYTES 1024
int tpa_graph_create_part_ipc(uint32_t n, uint64_t m, const uint64_t *out_offsets,
                              const uint32_t *out_targets, int policy, uint64_t fingerprint,
                              int device, uint32_t nranks, uint32_t rank, void *blob_out,
                              tpa_graph **out);
int tpa_part_ipc_attach(tpa_graph *g, const void *blobs /* nranks x TPA_IPC_BLOB_BYTES */);

/* Partition geometry: rows [row_begin, row_end) of `nranks`; `slice` = padded
 * rows per partition in the share layout. */
int tpa_graph_part_info(const tpa_graph *g, uint32_t *nranks, uint32_t *rank, uint32_t *row_begin,
                        uint32_t *row_end, uint32_t *slice);

/* One process driving `nparts` partitions on devices[0..nparts) (a device may
 * repeat); exchanges by stream-ordered peer copies, no NCCL. */
typedef struct tpa_group tpa_group;
int tpa_group_create(uint32_t n, uint64_t m, const uint64_t *out_offsets, const uint32_t *out_targets,
                     int policy, uint64_t fingerprint, const int *devices, uint32_t nparts,
                     tpa_group **out);
int tpa_group_destroy(tpa_group *grp);
int tpa_group_part(tpa_group *grp, uint32_t r, tpa_graph **out); /* borrowed; info calls only */
/* cpi_run semantics (as tpa_cpi_run); out_scores: n doubles, host or device (UVA). */
int tpa_group_cpi_run(tpa_group *grp, const uint32_t *seeds, uint64_t n_seeds, double c, double eps,
                      uint32_t start_iter, int64_t terminal_iter, double *out_scores,
                      uint32_t *iterations_run, int *converged, double *residual_l1);
/* preprocess's stranger vector (window [T, inf)); out: n doubles. */
int tpa_group_preprocess(tpa_group *grp, double c, double eps, uint32_t T, double *out_stranger);
/* query / query_na for B seeds on the row-partitioned graph (graphs beyond one
 * GPU): tpa_query_batch's semantics and errors (tpa.cpp:61-86) with the
 * artifact given by its fields -- stranger (n doubles, host or device via UVA;
 * unused with TPA_QUERY_NA), the graph fingerprint it was built for, c, eps, T.
 * The B-seed sweep runs on every partition's rows of the padded share layout;
 * spans, frontier words and exact residual limbs are exchanged per sweep
 * (peer copies).  out: [B][n] seed-major, host, or device with
 * TPA_DEVICE_PTRS.  Up to 16 partitions.  Scores equal the whole-graph
 * tpa_query_batch bit for bit under SelfLoop / Drop (Uniform: within rounding). */
int tpa_group_query_batch(tpa_group *grp, const double *stranger, uint64_t fingerprint, double c, double eps,
                          uint32_t T, const uint32_t *seeds, uint32_t B, uint32_t S, double *out, int flags);

/* --- host-side graph plumbing (not on the hot path) -----------------------
 * A host graph with the reference Graph's construction semantics
 * (graph.cpp:53-91: sort, dedupe, pre-policy dangling list, SelfLoop repair,
 * out-CSR, FNV-1a fingerprint), plus the generators the benchmarks use. */
typedef struct tpa_host_graph tpa_host_graph;

int tpa_host_graph_from_edges(uint32_t n, const uint32_t *src, const uint32_t *dst, uint64_t m,
                              int policy, tpa_host_graph **out);
/* R-MAT 2^scale nodes, edge_factor * 2^scale raw edges, quadrant probs
 * (a,b,c,1-a-b-c), mt19937_64(seed), no noise, no permutation, self-loops
 * dropped, duplicates removed by the construction. */
int tpa_host_graph_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                        uint64_t seed, int policy, int threads, tpa_host_graph **out);
/* The same construction on the GPU: sort + dedupe, dangling
 * list, SelfLoop repair and out-CSR on `device`, FNV-1a on the host; the
 * result is identical to tpa_host_graph_from_edges.  Errors as the reference
 * constructor (first out-of-range edge in input order -> TPA_ERR_OUT_OF_RANGE). */
int tpa_host_graph_build_gpu(uint32_t n, const uint32_t *src, const uint32_t *dst, uint64_t m,
                             int policy, int device, tpa_host_graph **out);
/* tpa_host_graph_rmat generated AND constructed on the GPU: the same
 * per-chunk mt19937_64 streams (one thread per 2^20-edge chunk), so the
 * edge list, the graph and its fingerprint equal the host generator's; the
 * construction as tpa_host_graph_build_gpu (keys sorted in place: peak
 * device memory 2 x 8 x edge_factor x 2^scale bytes).  The billion-edge
 * configs (BASELINE C5: scale 28) are generated in seconds this way. */
int tpa_host_graph_rmat_gpu(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                            uint64_t seed, int policy, int device, tpa_host_graph **out);
/* generate_random_graph(n, m, seed, policy) semantics (graph.cpp:166-205). */
int tpa_host_graph_random(uint32_t n, uint64_t m, uint64_t seed, int policy,
                          tpa_host_graph **out);
void tpa_host_graph_destroy(tpa_host_graph *h);
void tpa_host_graph_info(const tpa_host_graph *h, uint32_t *n, uint64_t *m,
                         uint64_t *n_dangling, uint64_t *fingerprint, int *policy);
const uint64_t *tpa_host_graph_offsets(const tpa_host_graph *h);
const uint32_t *tpa_host_graph_targets(const tpa_host_graph *h);
const uint32_t *tpa_host_graph_dangling(const tpa_host_graph *h);
/* Uniform sample without replacement of non-dangling nodes
 * (rwrank_main.cpp:65-83 sample_seeds, restated). */
int tpa_sample_seeds(const tpa_host_graph *h, uint64_t count, uint64_t rng_seed, uint32_t *out);
/* FNV-1a over (n, m, offsets, targets, policy) as graph.cpp:84-90. */
uint64_t tpa_fingerprint(uint32_t n, uint64_t m, const uint64_t *off, const uint32_t *tgt,
                         int policy);

#ifdef __cplusplus
}
#endif
#endif /* TPA_GPU_H */
