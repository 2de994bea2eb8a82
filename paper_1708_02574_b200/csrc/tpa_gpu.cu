// tpa_gpu.cu -- libtpa_gpu.so: GPU ingest, CPI driver and the C-ABI of
// include/tpa_gpu.h.  The hot kernels live in cpi_kernels.cuh.
//
// Device layout of a graph handle:
//   row_ptr  int64[n+1]  CSR(Ãᵀ) row offsets (row v = in-neighbours of v)
//   col      uint32[m]   sources, ascending within each row
//   deg      uint32[n]   out-degree (after SelfLoop repair)
//   items    uint2[]     work schedule per kernel family (SpMV, SpMM)
// Per-width workspace (B = 1, 8, 16, 32, 64): share ping-pong [n][B] fp64,
// acc [n][B] fp64, reduction partials, ticket counters, ColState x2.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "cpi_kernels.cuh"
#include "cpi_spmm.cuh"
#include "cpi_spmm5.cuh"
#include "cpi_spmv2.cuh"
#include "cpi_sweep1.cuh"
#include "tpa_gpu.h"
#include "tpa_internal.hpp"

namespace tpa {

std::string& last_error() {
    thread_local std::string s;
    return s;
}

// Set by an atexit hook registered at the first graph creation (so it runs
// before the static CUDA runtime tears down): handles destroyed after that
// point (static destructors of a host program) are leaked instead of freed.
std::atomic<bool> g_exiting{false};
void mark_exiting() { g_exiting = true; }

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            cudaGetLastError(); /* consume it: never leak into a later launch check */   \
            throw ::tpa::cuda_error(std::string(#x) + ": " + cudaGetErrorString(e_));    \
        }                                                                                \
    } while (0)

// After a kernel launch: name the kernel in the error.
#define CKL(name)                                                                        \
    do {                                                                                 \
        cudaError_t e_ = cudaGetLastError();                                             \
        if (e_ != cudaSuccess)                                                           \
            throw ::tpa::cuda_error(std::string("launch of ") + name + ": " +            \
                                    cudaGetErrorString(e_));                             \
    } while (0)

// ---------------------------------------------------------------------------
// Device memory
// ---------------------------------------------------------------------------
// Stream-ordered allocation (cudaMallocAsync pool): allocating and freeing
// never synchronises the device, so per-call temporaries and artifacts are
// cheap and the query pipeline stays asynchronous.
// The buffer remembers the owning handle's stream *variable*, so frees follow
// the handle if tpa_graph_set_stream switches streams.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    const cudaStream_t* sp = nullptr;
    bool plain = false;  // cudaMalloc'd (exportable by CUDA IPC), freed by cudaFree
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    void release() {
        if (p) {
            if (plain) {
                cudaStreamSynchronize(*sp);
                cudaFree(p);
            } else {
                cudaFreeAsync(p, *sp);
            }
        }
        p = nullptr;
        bytes = 0;
        plain = false;
    }
    // A buffer another process can map (cudaIpcGetMemHandle needs a cudaMalloc base).
    void ensure_plain(size_t nbytes, const cudaStream_t& stream) {
        if (bytes >= nbytes && p && plain) return;
        release();
        const size_t want = nbytes ? nbytes : 16;
        if (cudaMalloc(&p, want) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            throw alloc_error("cudaMalloc of " + std::to_string(want) + " bytes failed");
        }
        CK(cudaMemsetAsync(p, 0, want, stream));
        sp = &stream;
        bytes = want;
        plain = true;
    }
    void ensure(size_t nbytes, const cudaStream_t& stream) {
        if (bytes >= nbytes && p) return;
        release();
        const size_t want = nbytes ? nbytes : 16;
        if (cudaMallocAsync(&p, want, stream) != cudaSuccess) {
            cudaGetLastError();
            p = nullptr;
            throw alloc_error("cudaMallocAsync of " + std::to_string(want) + " bytes failed");
        }
        sp = &stream;
        bytes = want;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
    void swap(DevBuf& o) {
        std::swap(p, o.p);
        std::swap(bytes, o.bytes);
        std::swap(sp, o.sp);
        std::swap(plain, o.plain);
    }
};

// Ranked share layout (B = 1 sweeps): node u's share lives at slot rank[u],
// nodes ordered by out-degree, descending (ties by id).  The hot sources --
// C4: the top 10% of nodes feed 89% of the gathers -- then share 32-byte
// sectors and L2 lines instead of being spread over the whole vector.
__global__ void k_rank_keys(const uint32_t* __restrict__ deg, uint32_t n, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ ids) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x) {
        keys[u] = ~deg[u];
        ids[u] = (uint32_t)u;
    }
}
__global__ void k_rank_scatter(const uint32_t* __restrict__ perm, uint32_t n, uint32_t* __restrict__ rank) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x)
        rank[perm[k]] = (uint32_t)k;
}
__global__ void k_col_rank(const uint32_t* __restrict__ col, uint64_t m, const uint32_t* __restrict__ rank,
                           uint32_t* __restrict__ col_rank) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
        col_rank[e] = __ldg(rank + col[e]);
}

// ---------------------------------------------------------------------------
// K1: ingest -- out-edge CSR -> CSR(Ãᵀ) (stable radix sort by target keeps
// sources ascending inside every row: the reference's scatter order).
// ---------------------------------------------------------------------------
__global__ void k_degrees(const uint64_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ deg) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n;
         u += (uint64_t)gridDim.x * blockDim.x)
        deg[u] = (uint32_t)(off[u + 1] - off[u]);
}

// One warp per source u writes u into its out-edge slots.
__global__ void k_expand_src(const uint64_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ src) {
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (uint64_t u = warp; u < n; u += nwarps)
        for (uint64_t e = off[u] + lane; e < off[u + 1]; e += 32) src[e] = (uint32_t)u;
}

// row_ptr[v] = first position of key v in the sorted targets (lower bound).
__global__ void k_row_ptr(const uint32_t* __restrict__ keys, uint64_t m, uint32_t n,
                          int64_t* __restrict__ row_ptr) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = 0, hi = m;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (keys[mid] < v) lo = mid + 1;
            else hi = mid;
        }
        row_ptr[v] = (int64_t)lo;
    }
}

// ---------------------------------------------------------------------------
// K4: initial iterate x⁽⁰⁾ (cpi.cpp:59-67).
// ---------------------------------------------------------------------------
// Dense B = 1 start: PageRank (x == null: every node gets `weight`,
// SeedSet::all_nodes) or an explicit x (propagation_sweep / multi-seed sets).
// |x⁰| and the dangling mass go into exact fixed-point totals (fx[4], zero on
// entry) like the sweeps', so a row partition sees the same x⁰ state.
__global__ void __launch_bounds__(kThreads)
k_init_dense(const double* __restrict__ x, double weight, uint32_t n,
             const uint32_t* __restrict__ deg, double keep, double* __restrict__ share0,
             double* __restrict__ acc0, unsigned long long* fx, double* __restrict__ dm_part,
             const uint32_t* __restrict__ rank) {
    __shared__ unsigned long long s_w[4 * (kThreads / 32)];
    __shared__ double s_dm[kThreads / 32];
    unsigned long long f0 = 0, f1 = 0, f2 = 0, f3 = 0;
    double sdm = 0.0;
    for (uint64_t u = blockIdx.x * (uint64_t)kThreads + threadIdx.x; u < n; u += (uint64_t)gridDim.x * kThreads) {
        const double xv = x ? x[u] : weight;
        const uint32_t d = deg[u];
        share0[rank ? rank[u] : u] = d ? ddiv(dmul(keep, xv), (double)d) : 0.0;
        if (acc0) acc0[u] = xv;
        fx_add(f0, f1, xv);
        if (d == 0) {
            if (dm_part) sdm = dadd(sdm, xv);
            else fx_add(f2, f3, xv);
        }
    }
    if (dm_part) {
        // a caller-supplied x (propagation_sweep): any sign and magnitude, so the
        // dangling mass is a signed double sum (graph.cpp:213-225 sums signed
        // doubles) in a fixed order -- grid-stride per thread, a fixed warp tree,
        // warps in order, blocks in order (k_init_finish)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sdm = dadd(sdm, __shfl_down_sync(0xffffffffu, sdm, o));
        if ((threadIdx.x & 31) == 0) s_dm[threadIdx.x >> 5] = sdm;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = s_dm[0];
            for (int k = 1; k < kThreads / 32; ++k) t = dadd(t, s_dm[k]);
            dm_part[blockIdx.x] = t;
        }
    }
    fx_cta_flush(f0, f1, f2, f3, s_w, fx);
}

// x⁰'s ColState from the totals (then fx is zeroed for the sweeps); a
// partition instead publishes limbs for the all-reduce + k_part_finalize.
// dm_part (n_parts block sums, in block order) replaces the fixed-point
// dangling total when the start vector was caller-supplied.
__global__ void k_init_finish(unsigned long long* fx, unsigned long long* limbs, int policy, double keep,
                              uint32_t n, int active0, ColState* state0, const double* dm_part,
                              int n_parts) {
    if (limbs) {
        fx_to_limbs(fx[0], fx[1], limbs);
        fx_to_limbs(fx[2], fx[3], limbs + 3);
    } else {
        const double l1 = fx_decode(fx[0], fx[1]);
        double dm = fx_decode(fx[2], fx[3]);
        if (dm_part) {
            dm = dm_part[0];
            for (int k = 1; k < n_parts; ++k) dm = dadd(dm, dm_part[k]);
        }
        ColState s;
        s.residual = l1;
        s.iters = 0;
        s.active = active0;
        s.converged = 0;
        s.has_spread = policy == kUniform && dm != 0.0;
        s.spread = s.has_spread ? ddiv(dmul(keep, dm), (double)n) : 0.0;
        state0[0] = s;
    }
    fx[0] = fx[1] = fx[2] = fx[3] = 0ull;
}


// Batch of single-seed starts x⁽⁰⁾_b = c·e_{seed_b}; share0/acc0 pre-zeroed.
__global__ void k_init_seeds(const SeedList seeds, uint32_t b_valid, int B, double c,
                             double keep, uint32_t n, int policy, const uint32_t* __restrict__ deg,
                             double* __restrict__ share0, double* __restrict__ acc0, int active0,
                             ColState* state0, const uint32_t* __restrict__ rank) {
    const int b = threadIdx.x;
    if (b >= B) return;
    ColState s;
    s.iters = 0;
    s.converged = 0;
    if (b < (int)b_valid) {
        const uint32_t seed = seeds.s[b];
        const uint32_t d = deg[seed];
        const double w = c;  // c / |S| with |S| = 1
        share0[(size_t)(rank ? rank[seed] : seed) * B + b] = d ? ddiv(dmul(keep, w), (double)d) : 0.0;  // rank: B = 1
        if (acc0) acc0[(size_t)seed * B + b] = w;
        s.residual = w;
        s.active = active0;
        s.has_spread = policy == kUniform && d == 0;
        s.spread = s.has_spread ? ddiv(dmul(keep, w), (double)n) : 0.0;
    } else {
        s.residual = 0.0;
        s.active = 0;
        s.has_spread = 0;
        s.spread = 0.0;
    }
    state0[b] = s;
}

// SpMM batches: x⁽⁰⁾ rows of the seeds only.  Each seed's thread writes the
// seed's whole B-wide row of share0 / acc0 (identical data when two columns
// share a seed) and marks it in the frontier and acc_valid bitmaps; nothing
// else is zero-filled (cpi.cpp:59-63).
__global__ void k_init_seeds_mm(const SeedList seeds, uint32_t b_valid, int B, double c, double keep,
                                uint32_t n, int policy, const uint32_t* __restrict__ deg,
                                double* __restrict__ share0, double* __restrict__ acc0,
                                uint32_t* __restrict__ nz0, uint32_t* __restrict__ acc_valid, int active0,
                                ColState* state0) {
    const int b = threadIdx.x;
    if (b >= B) return;
    ColState s;
    s.iters = 0;
    s.converged = 0;
    if (b < (int)b_valid) {
        const uint32_t seed = seeds.s[b];
        const uint32_t d = deg[seed];
        const double w = c;  // c / |S|, |S| = 1
        const double sh = d ? ddiv(dmul(keep, w), (double)d) : 0.0;
        for (int k = 0; k < B; ++k) {
            const bool mine = k < (int)b_valid && seeds.s[k] == seed;
            share0[(size_t)seed * B + k] = mine ? sh : 0.0;
            if (acc0) acc0[(size_t)seed * B + k] = mine ? w : 0.0;
        }
        atomicOr(nz0 + (seed >> 5), 1u << (seed & 31));
        if (acc0) atomicOr(acc_valid + (seed >> 5), 1u << (seed & 31));
        s.residual = w;
        s.active = active0;
        s.has_spread = policy == kUniform && d == 0;
        s.spread = s.has_spread ? ddiv(dmul(keep, w), (double)n) : 0.0;
    } else {
        s.residual = 0.0;
        s.active = 0;
        s.has_spread = 0;
        s.spread = 0.0;
    }
    state0[b] = s;
}

__device__ __forceinline__ bool row_valid(const uint32_t* acc_valid, uint32_t v) {
    return !acc_valid || ((__ldg(acc_valid + (v >> 5)) >> (v & 31)) & 1u);
}

// K5 standalone combine (S = 1, or every column stopped before sweep S-1).
__global__ void k_combine(const double* __restrict__ acc, const uint32_t* __restrict__ acc_valid,
                          uint32_t n, int B, uint32_t b_valid, const double* __restrict__ stranger,
                          double scale, int node_major, double* __restrict__ out) {
    const uint64_t total = (uint64_t)n * B;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = (uint32_t)(i / B), b = (uint32_t)(i % B);
        if (b >= b_valid) continue;
        const double f = row_valid(acc_valid, v) ? acc[i] : 0.0;
        const size_t o = node_major ? i : (size_t)b * n + v;
        out[o] = stranger ? dadd(dmul(scale, f), stranger[v]) : dmul(f, scale);
    }
}

// acc [n][B] (rows outside acc_valid are zero) -> [B][n] or [n][B].
__global__ void k_acc_export(const double* __restrict__ src, const uint32_t* __restrict__ acc_valid,
                             uint32_t n, int B, uint32_t b_valid, int node_major, double* __restrict__ dst) {
    const uint64_t total = (uint64_t)n * B;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = (uint32_t)(i / B), b = (uint32_t)(i % B);
        if (b >= b_valid) continue;
        const double x = row_valid(acc_valid, v) ? src[i] : 0.0;
        dst[node_major ? i : (size_t)b * n + v] = x;
    }
}

// ---------------------------------------------------------------------------
// Work schedules (host, once per graph): long rows first (largest first) so
// they start early, then tiles of consecutive short rows in row order.
// ---------------------------------------------------------------------------
struct Schedule {
    DevBuf items;
    DevBuf item_nnz;  // {nnz begin, nnz end} per item (SpMV v2)
    uint32_t n_items = 0;
    uint32_t n_groups = 0;
};

std::vector<uint2> build_items(const std::vector<int64_t>& rp, uint32_t n, int64_t tile_nnz,
                               uint32_t tile_rows, int64_t long_row) {
    std::vector<std::pair<int64_t, uint32_t>> longs;
    std::vector<uint2> tiles;
    uint32_t r = 0;
    while (r < n) {
        const int64_t L = rp[r + 1] - rp[r];
        if (L > long_row) {
            longs.push_back({L, r});
            ++r;
            continue;
        }
        const uint32_t start = r;
        int64_t nnz = 0;
        while (r < n && r - start < tile_rows) {
            const int64_t L2 = rp[r + 1] - rp[r];
            if (L2 > long_row) break;
            if (r > start && nnz + L2 > tile_nnz) break;
            nnz += L2;
            ++r;
            if (nnz >= tile_nnz) break;
        }
        tiles.push_back(make_uint2(start, r));
    }
    std::stable_sort(longs.begin(), longs.end(),
                     [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<uint2> items;
    items.reserve(longs.size() + tiles.size());
    for (auto& l : longs) items.push_back(make_uint2(l.second, (l.second + 1) | kLongFlag));
    items.insert(items.end(), tiles.begin(), tiles.end());
    return items;
}

// Rows per block of the fused sweep: B = 16 in 16-row blocks (2.2 KB of shared
// memory per warp either way: 1.23 -> 1.13 ms per C2 batch), B = 32 / 64 in
// 8-row blocks (32 resident warps per SM instead of 24).
static int mm5_rows(int B) { return B == 16 ? 16 : 8; }

template <int B, bool L, int RB>
static void launch_fused(const Mm4Args& P, int num_sms, cudaStream_t stream) {
    using Sh = Mm5<B, RB>;
    static const int grid = [num_sms] {
        CK(cudaFuncSetAttribute(k_mm_fused<B, L, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)Sh::kDynSmem));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mm_fused<B, L, RB>, Sh::NT, Sh::kDynSmem));
        return std::max(occ, 1) * num_sms;
    }();
    k_mm_fused<B, L, RB><<<grid, Sh::NT, Sh::kDynSmem, stream>>>(P);
}

template <int B, bool L>
static void launch_fused_rb(const Mm4Args& P, int rb, int num_sms, cudaStream_t stream) {
    (void)rb;  // mm5_rows(B): 16 for B = 16, 8 otherwise
    launch_fused<B, L, B == 16 ? 16 : 8>(P, num_sms, stream);
}

// Sweeps (of a seed batch) run frontier-driven: push-mark then pull.
constexpr uint32_t kSparseSweeps = 3;

// Persistent-grid sizing of the B = 8 sweep (k_step_spmm2; dynamic smem = row buffers).
template <int B>
static int mm_occupancy() {
    int occ = 0;
    const size_t dyn = MmShape<B>::kDynSmem;
    CK(cudaFuncSetAttribute(k_step_spmm2<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_step_spmm2<B>, MmShape<B>::NT, dyn));
    return occ;
}

struct Workspace {
    int B = 0;
    DevBuf share[2], acc, part, gpart, group_cnt, done_cnt, state;
    // SpMM (B > 1) extras
    DevBuf nz[2], acc_valid, long_cnt, seg_part, work_cnt, fx;
    DevBuf s1_skip, s1_fx;  // the seed push took sweep 1 (cpi_sweep1.cuh); its exact totals
    int grid = 0;  // persistent grid of k_step_spmm2<8>
    DevBuf rowflag, sparse_ctl;  // sparse sweeps: reachable rows; {cost, dense, window count}
    DevBuf wbits, wl;            // sparse sweeps: marked windows (bitmap, list)
    DevBuf big;                  // sparse sweeps: edge chunks of high out-degree frontier rows
    DevBuf limbs;                // partition mode: [3][6] fixed-point limbs (sweep parity 0/1, init) + [6] totals
    DevBuf sl;                   // sparse sweeps: segments of the marked long rows
    DevBuf dm_part;              // caller-supplied x: per-block signed dangling sums
};

// Long rows of CSR(Ãᵀ) (in-degree > kLong) cut into kLong-nnz segments, the
// SpMM's first work items (longest rows first).
struct LongRows {
    DevBuf seg_row, seg_lo, seg_long, long_first, long_nseg;
    uint32_t n_segs = 0, n_long = 0;
    DevBuf blocks;  // short-row blocks {first row, rows} (kMmRows windows)
    DevBuf blocks_w[4];  // the same inside 4 / 8 / 16 / 32-row windows (SpMM v5, SpMV v3)
    uint32_t n_blocks_w[4] = {0, 0, 0, 0};
    DevBuf win_blk_w[4];  // per window: index of its first block (n_windows + 1 entries)
    static int wi(int rows) { return rows == 4 ? 0 : rows == 8 ? 1 : rows == 16 ? 2 : 3; }
};

// A row partition of CSR(Ãᵀ) for multi-GPU CPI (the north star's layout):
// partition r owns rows [bounds[r], bounds[r+1]) (balanced by nnz) and their
// y / acc; the iterate's shares live in a padded global layout of
// nranks x slice doubles (row v of partition r at r*slice + v - bounds[r]),
// so one in-place all-gather per sweep assembles the full share vector and
// the column indices are stored pre-mapped to that layout.
// After its S rows, every partition's span in the share buffer carries its
// residual limbs (6 uint64 as doubles' bits), so one all-gather per sweep
// moves the shares and the totals together.
constexpr uint32_t kLimbPad = 8;

// One process per GPU over CUDA IPC (tpa_part.cuh): every rank maps its
// peers' share ping-pong buffers and limb slots and stores its shares into
// them from the sweep epilogue (the exchange IS the sweep's stores); per
// exchange point each rank records an interprocess event and the ranks meet
// on a host-side stage counter in POSIX shared memory, so each stream waits
// on exactly the peers' matching records (no kernel ever waits on a kernel).
constexpr int kIpcRing = 4;
struct IpcState {
    struct Peer {
        double* share[2] = {nullptr, nullptr};
        unsigned long long* limbs = nullptr;
        cudaEvent_t ev[kIpcRing] = {};
    };
    std::vector<Peer> peers;  // nranks; the own entry holds local pointers
    cudaEvent_t own_ev[kIpcRing] = {};
    uint64_t stage = 0;       // exchange points passed (the same sequence on every rank)
    char shm_name[64] = {0};
    volatile uint64_t* shm = nullptr;  // nranks stage counters, 64 bytes apart
    size_t shm_bytes = 0;
    bool shm_owner = false;
    bool attached = false;
};

struct PartInfo {
    uint32_t nranks = 1, rank = 0;
    uint32_t n_global = 0;
    uint64_t m_global = 0;
    std::vector<uint32_t> bounds;  // nranks + 1
    uint32_t slice = 0;            // S: rows of the largest partition
    uint32_t stride = 0;           // S + kLimbPad: a partition's span in the share layout
    ncclComm_t comm = nullptr;     // one rank per process; null: in-process group or nranks = 1
    std::unique_ptr<IpcState> ipc;  // one rank per process over CUDA IPC (tpa_part.cuh)
    uint32_t row_begin() const { return bounds[rank]; }
    uint32_t rows(uint32_t r) const { return bounds[r + 1] - bounds[r]; }
};

}  // namespace tpa

using namespace tpa;

struct tpa_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint32_t n = 0;
    uint64_t m = 0;
    int policy = 0;
    uint64_t fingerprint = 0;
    DevBuf row_ptr, col, deg;
    // ranked layout of the B = 1 sweeps (PageRank, single-vector CPI): nodes
    // numbered by out-degree (descending) in the share vector only -- rows stay
    // in id order; col_rank = rank[col]; empty when not built (small graphs)
    DevBuf rank, col_rank;
    DevBuf out_off, out_tgt;  // the out-edge CSR itself (frontier push-marking)
    Schedule mv;  // SpMV work items
    MvShape mv_shape = kMvShapeS;  // SpMV tile shape (mv_shape of the global node count)
    LongRows longs;
    uint32_t n_blocks = 0;  // kMmRows-row blocks
    std::map<int, std::unique_ptr<Workspace>> ws;
    DevBuf init_part;
    // host-output pipeline of batch calls: chunk k computes into stage[k % 2] on
    // `stream` while chunk k-1's results drain to the host on `copy`
    struct HostPipe {
        cudaStream_t copy = nullptr;
        DevBuf stage[2];
        cudaEvent_t done[2] = {nullptr, nullptr}, free_[2] = {nullptr, nullptr};
        bool pending[2] = {false, false};
        int slot = 0;
    } pipe;
    std::set<tpa_artifact*> artifacts;  // detached (buffers freed) on destroy
    std::unique_ptr<PartInfo> part;     // row partition (multi-GPU), or null: whole graph
    PeerOut peer_out{};                 // set by the group driver around a sweep (tpa_part.cuh)
    struct TopkWork {
        DevBuf st, hist, cand, ids;  // device top-k (tpa_topk.cuh): state, histograms, candidates, picks
    } topk;
    uint64_t launches = 0;
    int num_sms = 148;
    std::mutex mu;
    static constexpr uint64_t sparse_div = 32;  // sparse sweep if the push touches <= m / 32 edges
    // optional per-sweep-kernel CUDA-event timing (bench instrumentation)
    bool profile = false;
    struct ProfEvent {
        int width;
        uint32_t step;
        cudaEvent_t e0, e1;
    };
    std::vector<ProfEvent> prof_events;
    std::vector<cudaEvent_t> event_pool;
    cudaEvent_t take_event() {
        cudaEvent_t e;
        if (!event_pool.empty()) {
            e = event_pool.back();
            event_pool.pop_back();
        } else {
            CK(cudaEventCreate(&e));
        }
        return e;
    }

    Workspace& workspace(int B) {
        auto& p = ws[B];
        if (!p) {
            p = std::make_unique<Workspace>();
            p->B = B;
        }
        Workspace& w = *p;
        // SpMV partials / tickets (B = 1); the SpMM reduces in fixed point instead
        const uint32_t items = B == 1 ? mv.n_items : 1, groups = B == 1 ? mv.n_groups : 1;
        // B > 1: one extra all-zero row (index n) that dead sources gather
        const size_t nb = (size_t)n * B * sizeof(double);
        // a partition's shares span the padded global layout (all partitions)
        // (the padded rows of every partition, then for B > 1 the zero row)
        const size_t rows_sh = part ? (size_t)part->nranks * part->stride : (size_t)n;
        const size_t nbs = rows_sh * B * sizeof(double) + (B > 1 ? (size_t)B * sizeof(double) : 0);
        if (w.share[0].bytes < nbs) {
            w.share[0].ensure(nbs, stream);
            w.share[1].ensure(nbs, stream);
            if (B > 1) {
                CK(cudaMemsetAsync(w.share[0].as<double>() + rows_sh * B, 0, (size_t)B * 8, stream));
                CK(cudaMemsetAsync(w.share[1].as<double>() + rows_sh * B, 0, (size_t)B * 8, stream));
            }
        }
        w.acc.ensure(nb, stream);
        w.part.ensure((size_t)items * 2 * B * sizeof(double), stream);
        w.gpart.ensure((size_t)groups * 2 * B * sizeof(double), stream);
        if (!w.group_cnt.p) {
            w.group_cnt.ensure((size_t)groups * sizeof(uint32_t), stream);
            w.done_cnt.ensure(sizeof(uint32_t), stream);
            CK(cudaMemsetAsync(w.group_cnt.p, 0, w.group_cnt.bytes, stream));
            CK(cudaMemsetAsync(w.done_cnt.p, 0, w.done_cnt.bytes, stream));
        }
        w.state.ensure(2 * (size_t)B * sizeof(ColState), stream);
        if (B == 1 && !w.fx.p) {
            w.fx.ensure(4 * 8 * kMvFxSlots, stream);
            CK(cudaMemsetAsync(w.fx.p, 0, w.fx.bytes, stream));
            w.long_cnt.ensure((size_t)std::max<uint32_t>(longs.n_long, 1) * 4, stream);
            w.seg_part.ensure((size_t)std::max<uint32_t>(longs.n_segs, 1) * 8, stream);
            CK(cudaMemsetAsync(w.long_cnt.p, 0, w.long_cnt.bytes, stream));
        }
        if (B > 1 && !w.work_cnt.p) {
            const size_t words = (rows_sh + 31) / 32 + 1;  // frontier bitmaps span the share rows
            w.nz[0].ensure(words * 4, stream);
            w.nz[1].ensure(words * 4, stream);
            w.acc_valid.ensure(words * 4, stream);
            w.long_cnt.ensure((size_t)std::max<uint32_t>(longs.n_long, 1) * 4, stream);
            w.seg_part.ensure((size_t)std::max<uint32_t>(longs.n_segs, 1) * B * 8, stream);
            w.work_cnt.ensure(4, stream);
            w.fx.ensure(4 * (size_t)B * 8, stream);
            CK(cudaMemsetAsync(w.long_cnt.p, 0, w.long_cnt.bytes, stream));
            CK(cudaMemsetAsync(w.work_cnt.p, 0, w.work_cnt.bytes, stream));
            CK(cudaMemsetAsync(w.fx.p, 0, w.fx.bytes, stream));
            if (B == 8) w.grid = std::max(1, mm_occupancy<8>()) * num_sms;
            if (B >= 16) {  // the fused sweep's sparse-sweep lists
                w.rowflag.ensure((size_t)n + 16, stream);
                w.sparse_ctl.ensure(32, stream);
                w.big.ensure(mark_chunk_cap(m) * sizeof(ulonglong2), stream);
                w.sl.ensure(((size_t)longs.n_segs + 1) * 4, stream);
                w.wbits.ensure(((size_t)n / 4 / 32 + 2) * 4, stream);
                w.wl.ensure(((size_t)n / 4 + 2) * 4, stream);
            }
        }
        return w;
    }
};

struct tpa_artifact {
    tpa_graph* g = nullptr;  // null once the graph is gone (buffers freed then)
    DevBuf stranger;
    uint64_t n = 0;  // entries of `stranger`
    uint64_t fingerprint = 0;
    double c = 0.15, eps = 1e-9;
    uint32_t T = 10;
};

static void detach_artifact(tpa_artifact* a) {
    a->stranger.release();
    a->g = nullptr;
}

namespace tpa {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) CK(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

static int grid_for(uint64_t work, int per_block, int max_blocks) {
    uint64_t b = (work + per_block - 1) / per_block;
    if (b < 1) b = 1;
    if (b > (uint64_t)max_blocks) b = max_blocks;
    return (int)b;
}

// Steps needed for ||x⁽ⁱ⁾||₁ = c(1-c)^i < eps (exact for SelfLoop/Uniform,
// an upper bound for Drop); the driver re-checks the device state after.
static uint32_t sweeps_estimate(double c, double eps) {
    const double k = std::ceil(std::log(eps / c) / std::log(1.0 - c));
    if (!(k >= 1.0)) return 1;
    if (k > 1e6) return 1000000;
    return (uint32_t)k;
}

// cpi.cpp:11-17 (CpiParams::validate)
static void validate_cpi(double c, double eps, uint32_t start, int64_t terminal) {
    if (!(c > 0.0 && c < 1.0)) throw std::invalid_argument("restart probability must be in (0, 1)");
    if (!(eps > 0.0)) throw std::invalid_argument("tolerance must be positive");
    if (terminal >= 0 && (uint64_t)terminal < start)
        throw std::invalid_argument("terminal iteration precedes start iteration");
}

// cpi.cpp:34-39 (SeedSet::validate_against), for a sorted seed list.
static void validate_seed(uint32_t seed, uint32_t n) {
    if (seed >= n)
        throw std::out_of_range("seed id " + std::to_string(seed) + " out of range for graph with " +
                                std::to_string(n) + " nodes");
}

enum class Init { Dense, Seeds };

struct RunCfg {
    int B = 1;
    uint32_t b_valid = 1;
    double c = 0.15, eps = 1e-9;
    uint32_t start = 0;
    int64_t terminal = -1;
    Init init = Init::Dense;
    const double* d_x = nullptr;     // Dense: explicit x⁽⁰⁾ (null -> uniform weight)
    bool signed_x = false;           // d_x caller-supplied (any sign / magnitude): signed dangling sum
    double weight = 0.0;             // Dense with d_x == null
    SeedList seeds{};                // Seeds (by value)
    // accumulation: windowed single acc, or partition segment accs
    double* acc = nullptr;
    std::vector<double*> seg_acc;
    std::vector<uint32_t> bounds;
    // fused combine at the terminal sweep
    double* out = nullptr;
    const double* stranger = nullptr;
    double scale = 1.0;
    bool node_major = false;
    // single-sweep API
    double* y_out = nullptr;
    bool want_state = true;
};

struct RunOut {
    std::vector<ColState> state;
};

static size_t seg_of(const std::vector<uint32_t>& bounds, uint32_t i) {
    return std::upper_bound(bounds.begin(), bounds.end(), i) - bounds.begin();
}

// K2 v2 at one tile shape: dynamic shared memory sized for it, set once per
// instantiation.
template <bool RF, int THR, int NNZ, int ROWS, bool MULTI>
static void launch_mv2_(const MvArgs& M, uint32_t grid, cudaStream_t stream);
template <bool RF, int THR, int NNZ, int ROWS>
static void launch_mv2(const MvArgs& M, uint32_t grid, cudaStream_t stream) {
    if (M.per_cta > 1) launch_mv2_<RF, THR, NNZ, ROWS, true>(M, grid, stream);
    else launch_mv2_<RF, THR, NNZ, ROWS, false>(M, grid, stream);
}
template <bool RF, int THR, int NNZ, int ROWS, bool MULTI>
static void launch_mv2_(const MvArgs& M, uint32_t grid, cudaStream_t stream) {
    constexpr size_t smem = mv_dyn_smem<NNZ, ROWS>();
    static const bool ok = [] {
        CK(cudaFuncSetAttribute(k_step_spmv2<RF, THR, NNZ, ROWS, MULTI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
        return true;
    }();
    (void)ok;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(THR);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_step_spmv2<RF, THR, NNZ, ROWS, MULTI>, M));  // programmatic dependent launch
}

static void launch_step(tpa_graph* g, Workspace& w, const StepArgs& a, const MmArgs* mm, int B,
                        const SeedList* push_seeds = nullptr) {
    const Schedule& s = g->mv;
    const dim3 grid(B == 1 ? s.n_items : (uint32_t)w.grid);
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (g->profile) {
        e0 = g->take_event();
        e1 = g->take_event();
        CK(cudaEventRecord(e0, g->stream));
    }
    const bool fused = B >= 16;  // B = 8: k_step_spmm2<8>
    const int rb = mm5_rows(B);
    if (fused) {
        Mm4Args P{*mm, nullptr, nullptr, g->longs.blocks_w[LongRows::wi(rb)].as<uint2>(),
                  g->longs.n_blocks_w[LongRows::wi(rb)]};
        // the first sweeps of a seed batch usually see a small frontier: if it
        // pushes along at most m/32 edges, mark the rows it reaches (push over
        // the out-CSR) and pull only those; the decision is taken on the device
        if (push_seeds) {  // sweep 1 by a push from the seeds (cpi_sweep1.cuh): no pull
            if (!w.s1_skip.p) {
                w.s1_skip.ensure(16, g->stream);
                w.s1_fx.ensure(4 * 64 * 8, g->stream);
                CK(cudaMemsetAsync(w.s1_fx.p, 0, w.s1_fx.bytes, g->stream));
                CK(cudaMemsetAsync(w.s1_skip.p, 0, w.s1_skip.bytes, g->stream));
            }
            Sweep1Args S1{a, w.s1_fx.as<unsigned long long>(), g->out_off.as<uint64_t>(),
                          g->out_tgt.as<uint32_t>(), *push_seeds, mm->nz_out, mm->acc_valid,
                          w.s1_skip.as<uint32_t>()};
            const dim3 g1(8, B);  // 8 chunks per column: a hub seed's out-list is spread
            if (B == 16) {
                k_s1_rows<16><<<g1, 256, 0, g->stream>>>(S1);
                k_s1_push<16><<<g1, 256, 0, g->stream>>>(S1);
            } else if (B == 32) {
                k_s1_rows<32><<<g1, 256, 0, g->stream>>>(S1);
                k_s1_push<32><<<g1, 256, 0, g->stream>>>(S1);
            } else {
                k_s1_rows<64><<<g1, 256, 0, g->stream>>>(S1);
                k_s1_push<64><<<g1, 256, 0, g->stream>>>(S1);
            }
            CKL("k_s1_push");
            g->launches += 2;  // k_s1_rows + k_s1_push (the common ++ below is cancelled)
        } else if (mm->nz_in && a.step <= kSparseSweeps && !g->part) {
            const uint32_t words = (g->n + 31) / 32;
            auto* ctl = w.sparse_ctl.as<unsigned long long>();
            CK(cudaMemsetAsync(w.sparse_ctl.p, 0, 32, g->stream));
            CK(cudaMemsetAsync(w.rowflag.p, 0, g->n, g->stream));
            const bool by_win = true;
            const int rb_shift = rb == 4 ? 2 : rb == 8 ? 3 : rb == 16 ? 4 : 5;
            if (by_win) CK(cudaMemsetAsync(w.wbits.p, 0, ((size_t)(g->n >> rb_shift) / 32 + 1) * 4, g->stream));
            uint32_t* wl_cnt = reinterpret_cast<uint32_t*>(w.sparse_ctl.as<char>() + 12);
            const int gb = grid_for(words, 8, 16 * g->num_sms);
            k_frontier_cost<<<gb, 256, 0, g->stream>>>(mm->nz_in, words, g->out_off.as<uint64_t>(), ctl,
                                                       a.state_in, B, g->m / g->sparse_div);
            CKL("k_frontier_cost");
            MarkArgs MA{mm->nz_in, words, g->out_off.as<uint64_t>(), g->out_tgt.as<uint32_t>(), ctl,
                        g->m / g->sparse_div, w.rowflag.as<uint8_t>(), reinterpret_cast<int*>(ctl + 1),
                        w.wbits.as<uint32_t>(), by_win ? w.wl.as<uint32_t>() : nullptr, wl_cnt, rb_shift,
                        w.big.as<ulonglong2>(), wl_cnt + 1};
            k_mark_out<<<gb, 256, 0, g->stream>>>(MA);
            CKL("k_mark_out");
            k_mark_big<<<4 * g->num_sms, 256, 0, g->stream>>>(MA);
            if (by_win) {
                CKL("k_mark_big");
                const LongRows& L = g->longs;
                k_long_list<<<grid_for(std::max<uint32_t>(L.n_long, 1), 256, 4 * g->num_sms), 256, 0, g->stream>>>(
                    MA, L.seg_row.as<uint32_t>(), L.long_first.as<uint32_t>(), L.long_nseg.as<uint32_t>(),
                    L.n_long, w.sl.as<uint32_t>(), wl_cnt + 2);
                g->launches += 1;
            }
            CKL("k_mark_big");
            g->launches += 3;
            P.rowflag = w.rowflag.as<uint8_t>();
            P.dense = reinterpret_cast<const int*>(ctl + 1);
            if (by_win) {
                P.wl = w.wl.as<uint32_t>();
                P.wl_cnt = wl_cnt;
                P.win_blk = g->longs.win_blk_w[LongRows::wi(rb)].as<uint32_t>();
                P.sl = w.sl.as<uint32_t>();
                P.sl_cnt = wl_cnt + 2;
            }
        }
        if (push_seeds) {
            g->launches -= 1;  // no pull this sweep: cancels the common ++ below
        } else {
            const bool last = a.out != nullptr;
            if (B == 16) {
                if (last) launch_fused_rb<16, true>(P, rb, g->num_sms, g->stream);
                else launch_fused_rb<16, false>(P, rb, g->num_sms, g->stream);
            } else if (B == 32) {
                if (last) launch_fused_rb<32, true>(P, rb, g->num_sms, g->stream);
                else launch_fused_rb<32, false>(P, rb, g->num_sms, g->stream);
            } else {
                if (last) launch_fused_rb<64, true>(P, rb, g->num_sms, g->stream);
                else launch_fused_rb<64, false>(P, rb, g->num_sms, g->stream);
            }
            g->launches -= 1;  // one kernel (the common ++ below counts it)
        }
        g->launches += 1;  // + the epilogue below
    } else switch (B) {
        case 1:
            {
                MvArgs M{a, s.item_nnz.as<longlong2>(), w.fx.as<unsigned long long>(),
                         !g->part ? nullptr
                         : a.share_out ? reinterpret_cast<unsigned long long*>(a.share_out + g->part->slice)
                                       : w.limbs.as<unsigned long long>() + (a.step & 1) * 6,
                         PeerOut{}, g->part ? g->part->slice : 0u, mv_items_per_cta(s.n_items, g->num_sms)};
                if (g->part && a.share_out) M.peers = g->peer_out;
                const uint32_t mv_grid = (s.n_items + M.per_cta - 1) / M.per_cta;
                const MvShape& sh = g->mv_shape;
                const bool ranked = a.rank != nullptr;
                if (sh.thr == kMvShapeS.thr && sh.nnz == kMvShapeS.nnz && sh.rows == kMvShapeS.rows) {
                    if (ranked) launch_mv2<true, kMvShapeS.thr, kMvShapeS.nnz, kMvShapeS.rows>(M, mv_grid, g->stream);
                    else launch_mv2<false, kMvShapeS.thr, kMvShapeS.nnz, kMvShapeS.rows>(M, mv_grid, g->stream);
                } else {
                    if (ranked) launch_mv2<true, kMvShapeL.thr, kMvShapeL.nnz, kMvShapeL.rows>(M, mv_grid, g->stream);
                    else launch_mv2<false, kMvShapeL.thr, kMvShapeL.nnz, kMvShapeL.rows>(M, mv_grid, g->stream);
                }
            }
            break;
        case 8: k_step_spmm2<8><<<grid, MmShape<8>::NT, MmShape<8>::kDynSmem, g->stream>>>(*mm); break;
        default: throw std::invalid_argument("unsupported batch width");
    }
    CKL("k_step (sweep)");
    ++g->launches;
    if (g->profile) {
        CK(cudaEventRecord(e1, g->stream));
        g->prof_events.push_back({B, a.step, e0, e1});
    }
}

// The CPI driver: x⁽⁰⁾, then sweeps 1..K enqueued without host syncs; the
// per-column state (cpi.cpp:70-81) advances on the device.  Only a run to
// convergence (terminal < 0) checks the state on the host after the
// estimated horizon, and continues if a column is still active.

static void run_cpi(tpa_graph* g, RunCfg& cfg, RunOut* res) {
    const int B = cfg.B;
    Workspace& w = g->workspace(B);
    const Schedule& sch = g->mv;
    const uint32_t n = g->n;
    const bool mm = B > 1;  // SpMM path: frontier bitmaps, lazily valid acc rows
    if (mm && (cfg.init != Init::Seeds || cfg.start != 0 || !cfg.bounds.empty() || cfg.y_out))
        throw std::logic_error("batched CPI supports single-seed windows starting at 0 only");
    const size_t bm_bytes = (((size_t)n + 31) / 32 + 1) * 4;
    const double keep = 1.0 - cfg.c;
    ColState* st = w.state.as<ColState>();
    const bool partition = !cfg.bounds.empty() || !cfg.seg_acc.empty();
    double* acc_run = cfg.acc;
    const uint32_t* const deg_run = g->deg.as<uint32_t>();
    // B = 1 over the ranked share layout when the graph has one (rows unchanged)
    const uint32_t* const rank = (B == 1 && !partition && g->rank.p) ? g->rank.as<uint32_t>() : nullptr;
    // ranked B = 1 sweeps over a share vector far beyond the L2 (C5: 2.1 GB): the
    // hottest shares (the first slots) in a persisting L2 window -- C5's DRAM-bound
    // PageRank sweep 36.4 -> 34.9 ms; none at C4 (134 MB: LSU-bound), so not used there
    size_t persist = 0;
    if (rank && (size_t)n * 8 > (1ull << 30)) {
        static const size_t maxp = [] {
            int dev = 0, v = 0;
            CK(cudaGetDevice(&dev));
            CK(cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, dev));
            if (v > 0) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)v));
            return (size_t)std::max(v, 0);
        }();
        persist = std::min<size_t>(maxp, (size_t)n * 8);
    }

    // accumulator for x⁽⁰⁾, zero the rest
    double* acc0 = nullptr;
    if (partition) {
        const size_t s0 = seg_of(cfg.bounds, 0);
        for (size_t k = 0; k < cfg.seg_acc.size(); ++k)
            if (k != s0 || cfg.init == Init::Seeds)
                CK(cudaMemsetAsync(cfg.seg_acc[k], 0, (size_t)n * B * 8, g->stream));
        acc0 = cfg.seg_acc[s0];
    } else if (cfg.acc && mm) {
        acc0 = cfg.acc;  // validity tracked by acc_valid
        CK(cudaMemsetAsync(w.acc_valid.p, 0, bm_bytes, g->stream));
    } else if (acc_run) {
        const bool in0 = cfg.start == 0;
        if (!in0 || cfg.init == Init::Seeds)
            CK(cudaMemsetAsync(acc_run, 0, (size_t)n * B * 8, g->stream));
        acc0 = in0 ? acc_run : nullptr;
    }
    const int active0 = cfg.terminal != 0;
    if (cfg.init == Init::Dense) {
        const int nblk = grid_for(n, 4 * kThreads, 4 * g->num_sms);
        double* dm_part = nullptr;
        if (cfg.signed_x) {
            w.dm_part.ensure((size_t)nblk * 8, g->stream);
            dm_part = w.dm_part.as<double>();
        }
        k_init_dense<<<nblk, kThreads, 0, g->stream>>>(cfg.d_x, cfg.weight, n, deg_run, keep,
                                                       w.share[0].as<double>(), acc0,
                                                       w.fx.as<unsigned long long>(), dm_part, rank);
        CKL("k_init_dense");
        k_init_finish<<<1, 1, 0, g->stream>>>(w.fx.as<unsigned long long>(), nullptr, g->policy, keep, n,
                                              active0, st, dm_part, nblk);
        CKL("k_init_finish");
        g->launches += 2;
    } else if (mm) {
        CK(cudaMemsetAsync(w.nz[0].p, 0, bm_bytes, g->stream));
        CK(cudaMemsetAsync(w.work_cnt.p, 0, 4, g->stream));
        CK(cudaMemsetAsync(w.done_cnt.p, 0, 4, g->stream));
        k_init_seeds_mm<<<1, 64, 0, g->stream>>>(cfg.seeds, cfg.b_valid, B, cfg.c, keep, n, g->policy,
                                                 g->deg.as<uint32_t>(), w.share[0].as<double>(), acc0,
                                                 w.nz[0].as<uint32_t>(), w.acc_valid.as<uint32_t>(), active0, st);
        CKL("k_init_seeds_mm");
        g->launches += 1;
    } else {
        CK(cudaMemsetAsync(w.share[0].p, 0, (size_t)n * B * 8, g->stream));
        k_init_seeds<<<1, 64, 0, g->stream>>>(cfg.seeds, cfg.b_valid, B, cfg.c, keep, n, g->policy,
                                              g->deg.as<uint32_t>(), w.share[0].as<double>(), acc0,
                                              active0, st, rank);
        CKL("k_init_seeds");
        g->launches += 1;
    }

    StepArgs a{};
    a.row_ptr = g->row_ptr.as<int64_t>();
    a.col = rank ? g->col_rank.as<uint32_t>() : g->col.as<uint32_t>();
    a.rank = rank;
    a.deg = deg_run;
    a.items = sch.items.as<uint2>();
    a.n_items = sch.n_items;
    a.n = n;
    a.policy = g->policy;
    a.keep = keep;
    a.eps = cfg.eps;
    a.terminal = cfg.terminal;
    a.stranger = cfg.stranger;
    a.scale = cfg.scale;
    a.out_node_major = cfg.node_major ? 1 : 0;
    a.b_valid = cfg.b_valid;
    a.part = w.part.as<double>();
    a.gpart = w.gpart.as<double>();
    a.group_cnt = w.group_cnt.as<uint32_t>();
    a.done_cnt = w.done_cnt.as<uint32_t>();
    MmArgs ma{};
    if (mm) {
        ma.seg_row = g->longs.seg_row.as<uint32_t>();
        ma.seg_lo = g->longs.seg_lo.as<int64_t>();
        ma.seg_long = g->longs.seg_long.as<uint32_t>();
        ma.long_first = g->longs.long_first.as<uint32_t>();
        ma.long_nseg = g->longs.long_nseg.as<uint32_t>();
        ma.long_cnt = w.long_cnt.as<uint32_t>();
        ma.seg_part = w.seg_part.as<double>();
        ma.n_segs = g->longs.n_segs;
        ma.n_blocks = g->n_blocks;
        ma.blocks = g->longs.blocks.as<uint2>();
        ma.zero_row = n;
        ma.work_cnt = w.work_cnt.as<uint32_t>();
        ma.fx = w.fx.as<unsigned long long>();
        ma.acc_valid = cfg.acc ? w.acc_valid.as<uint32_t>() : nullptr;
    }

    const int64_t target = cfg.terminal >= 0 ? cfg.terminal : std::numeric_limits<int64_t>::max();
    const uint32_t est = sweeps_estimate(cfg.c, cfg.eps);
    uint64_t done = 0;
    bool combined = false;
    int64_t chunk = std::min<int64_t>(target, (int64_t)est + 1);
    std::vector<ColState> hst(B);
    while (chunk > 0) {
        for (int64_t j = 0; j < chunk; ++j) {
            const uint32_t i = (uint32_t)(done + 1 + j);
            a.step = i;
            a.share_in = w.share[(i - 1) & 1].as<double>();
            const bool last = (int64_t)i == target;
            a.share_out = (last || cfg.y_out) ? nullptr : w.share[i & 1].as<double>();
            a.y_out = cfg.y_out;
            if (partition) {
                a.acc = cfg.seg_acc[seg_of(cfg.bounds, i)];
            } else {
                const bool inw = i >= cfg.start && (cfg.terminal < 0 || (int64_t)i <= cfg.terminal);
                a.acc = inw ? acc_run : nullptr;
            }
            a.out = (last && cfg.out) ? cfg.out : nullptr;
            combined = combined || a.out != nullptr;
            a.state_in = st + ((i - 1) & 1) * B;
            a.state_out = st + (i & 1) * B;
            if (mm) {
                ma.s = a;
                ma.nz_in = w.nz[(i - 1) & 1].as<uint32_t>();
                ma.nz_out = a.share_out ? w.nz[i & 1].as<uint32_t>() : nullptr;
                if (ma.nz_out) CK(cudaMemsetAsync(ma.nz_out, 0, bm_bytes, g->stream));
            }
            // sweep 1 of a seed batch: a push from the seeds (one term per
            // element) instead of a pull over every nonzero
            const bool s1 = mm && i == 1 && cfg.init == Init::Seeds && a.acc && a.share_out && !a.out &&
                            !cfg.y_out && g->policy != kUniform && B >= 16 && !g->part;
            if (persist) {  // the hot (lowest-rank) shares of this sweep's input persist in L2
                cudaStreamAttrValue av{};
                av.accessPolicyWindow.base_ptr = const_cast<double*>(a.share_in);
                av.accessPolicyWindow.num_bytes = persist;
                av.accessPolicyWindow.hitRatio = 1.0f;
                av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                CK(cudaStreamSetAttribute(g->stream, cudaStreamAttributeAccessPolicyWindow, &av));
            }
            launch_step(g, w, a, mm ? &ma : nullptr, B, s1 ? &cfg.seeds : nullptr);
        }
        done += chunk;
        if ((int64_t)done >= target) break;
        CK(cudaMemcpyAsync(hst.data(), st + (done & 1) * B, B * sizeof(ColState),
                           cudaMemcpyDeviceToHost, g->stream));
        CK(cudaStreamSynchronize(g->stream));
        bool any = false;
        for (int b = 0; b < B; ++b) any = any || hst[b].active;
        if (!any) break;
        chunk = std::min<int64_t>(target - (int64_t)done, 16);
    }
    if (cfg.out && !combined) {
        double* acc_final = cfg.acc;
        k_combine<<<grid_for((uint64_t)n * B, 256, 8 * g->num_sms), 256, 0, g->stream>>>(
            acc_final, mm ? w.acc_valid.as<uint32_t>() : nullptr, n, B, cfg.b_valid, cfg.stranger, cfg.scale,
            cfg.node_major ? 1 : 0, cfg.out);
        CKL("k_combine");
        ++g->launches;
    }
    if (persist) {
        cudaStreamAttrValue av{};
        av.accessPolicyWindow.num_bytes = 0;
        CK(cudaStreamSetAttribute(g->stream, cudaStreamAttributeAccessPolicyWindow, &av));
        CK(cudaCtxResetPersistingL2Cache());
    }
    if (res && cfg.want_state) {
        res->state.resize(B);
        CK(cudaMemcpyAsync(res->state.data(), st + (done & 1) * B, B * sizeof(ColState),
                           cudaMemcpyDeviceToHost, g->stream));
        CK(cudaStreamSynchronize(g->stream));
    }
}

static void upload(tpa_graph* g, void* dst, const void* src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, g->stream));
}
static void download(tpa_graph* g, void* dst, const void* src, size_t bytes) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, g->stream));
}
static void finish(tpa_graph* g, int flags) {
    if (!((flags & TPA_DEVICE_PTRS) && (flags & TPA_ASYNC))) CK(cudaStreamSynchronize(g->stream));
}

static int batch_width(uint32_t b) {
    if (b <= 1) return 1;
    if (b <= 8) return 8;
    if (b <= 16) return 16;
    if (b <= 32) return 32;
    return 64;
}

// Batched single-seed runs over seeds[0..B): query / query_na / exact_rwr.
// `seeds` is a host array; `out` is host or device per flags.
static void run_seed_batch(tpa_graph* g, const uint32_t* seeds, uint32_t Btot, double c, double eps,
                           uint32_t start, int64_t terminal, const double* stranger, double scale,
                           bool combine, double* out, int flags) {
    const bool dev = flags & TPA_DEVICE_PTRS;
    const bool node_major = flags & TPA_NODE_MAJOR;
    const uint32_t n = g->n;
    std::vector<uint32_t> hseeds(seeds, seeds + Btot);  // host copy (callers resolve device lists)
    for (uint32_t b = 0; b < Btot; ++b) validate_seed(hseeds[b], n);
    if (node_major && Btot != (uint32_t)batch_width(Btot))
        throw std::invalid_argument("node-major output needs B in {8, 16, 32, 64}");
    if (node_major && Btot == 1)
        throw std::invalid_argument("node-major output needs B in {8, 16, 32, 64}");
    auto& P = g->pipe;
    if (!dev && !P.copy) {
        CK(cudaStreamCreateWithFlags(&P.copy, cudaStreamNonBlocking));
        for (int k = 0; k < 2; ++k) {
            CK(cudaEventCreateWithFlags(&P.done[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&P.free_[k], cudaEventDisableTiming));
        }
    }
    for (uint32_t b0 = 0; b0 < Btot; b0 += 64) {
        int slot = 0;
        if (!dev) {
            slot = P.slot;
            P.slot ^= 1;
            // the slot's previous drain must finish before it is overwritten (or reallocated)
            if (P.pending[slot]) CK(cudaStreamWaitEvent(g->stream, P.free_[slot], 0));
            P.stage[slot].ensure((size_t)std::min<uint32_t>(Btot, 64) * n * sizeof(double), g->stream);
        }
        const uint32_t bv = std::min<uint32_t>(64, Btot - b0);
        const int B = batch_width(bv);
        Workspace& w = g->workspace(B);
        (void)w;
        RunCfg cfg;
        cfg.B = B;
        cfg.b_valid = bv;
        cfg.c = c;
        cfg.eps = eps;
        cfg.start = start;
        cfg.terminal = terminal;
        cfg.want_state = false;
        if (B == 1) {
            // single seed through the SpMV path: dense x⁽⁰⁾ = c·e_seed
            cfg.init = Init::Seeds;
        } else {
            cfg.init = Init::Seeds;
        }
        for (uint32_t b = 0; b < bv; ++b) cfg.seeds.s[b] = hseeds[b0 + b];
        cfg.acc = w.acc.as<double>();
        double* dst = dev ? out + (node_major ? 0 : (size_t)b0 * n) : P.stage[slot].as<double>();
        if (combine) {
            cfg.out = dst;
            cfg.stranger = stranger;
            cfg.scale = scale;
            cfg.node_major = node_major;
        }
        RunOut ro;
        run_cpi(g, cfg, &ro);
        if (!combine) {
            // exact_rwr: the accumulator is the answer
            if (B == 1) {
                CK(cudaMemcpyAsync(dst, w.acc.p, (size_t)n * 8, cudaMemcpyDeviceToDevice, g->stream));
            } else {
                k_acc_export<<<grid_for((uint64_t)n * B, 256, 8 * g->num_sms), 256, 0, g->stream>>>(
                    w.acc.as<double>(), w.acc_valid.as<uint32_t>(), n, B, bv, node_major ? 1 : 0, dst);
                CKL("k_acc_export");
                ++g->launches;
            }
        }
        if (!dev) {
            CK(cudaEventRecord(P.done[slot], g->stream));
            CK(cudaStreamWaitEvent(P.copy, P.done[slot], 0));
            CK(cudaMemcpyAsync(out + (size_t)b0 * n, P.stage[slot].p, (size_t)bv * n * 8, cudaMemcpyDeviceToHost,
                               P.copy));
            CK(cudaEventRecord(P.free_[slot], P.copy));
            P.pending[slot] = true;
        }
    }
    if (!(flags & TPA_ASYNC)) {
        if (!dev) CK(cudaStreamSynchronize(P.copy));
        CK(cudaStreamSynchronize(g->stream));
    }
}

}  // namespace tpa

// ===========================================================================
// C-ABI
// ===========================================================================
namespace tpa {
static void require_whole(const tpa_graph* g, const char* what);
static void part_comm_destroy(ncclComm_t c);
static void ipc_teardown(tpa_graph* g);
static void part_cpi_run(std::vector<tpa_graph*>& Pg, const uint32_t* seeds, uint64_t n_seeds, double c,
                         double eps, uint32_t start_iter, int64_t terminal_iter, double* out_scores,
                         uint32_t* iterations_run, int* converged, double* residual_l1);
static void part_preprocess(std::vector<tpa_graph*>& Pg, double c, double eps, uint32_t T, double* out);
static void require_solo_part(const tpa_graph* g) {
    if (g->part->nranks > 1 && !g->part->comm && !g->part->ipc)
        throw std::invalid_argument("a group partition runs through the tpa_group_* calls");
}
}  // namespace tpa

// Work schedules over the rows of CSR(Ãᵀ) (row_ptr rp, n rows): SpMV tiles,
// SpMM long-row segments and short-row blocks.
static void build_schedules(tpa_graph* g, const std::vector<int64_t>& rp, uint32_t n) {
    cudaStream_t s = g->stream;
    g->mv_shape = mv_shape(g->part ? g->part->n_global : n);
    auto mv = build_items(rp, n, g->mv_shape.nnz, (uint32_t)g->mv_shape.rows, g->mv_shape.nnz);
    if (mv.size() >= 0x7fffffffu) throw std::invalid_argument("graph too large for one grid");
    {
        // SpMM long rows: kLong-nnz segments, longest rows first
        std::vector<std::pair<int64_t, uint32_t>> lr;
        for (uint32_t v = 0; v < n; ++v)
            if (rp[v + 1] - rp[v] > kLong) lr.push_back({rp[v + 1] - rp[v], v});
        std::stable_sort(lr.begin(), lr.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
        std::vector<uint32_t> seg_row, seg_long, long_first, long_nseg;
        std::vector<int64_t> seg_lo;
        for (uint32_t li = 0; li < lr.size(); ++li) {
            const uint32_t v = lr[li].second;
            const uint32_t ns = (uint32_t)((lr[li].first + kLong - 1) / kLong);
            long_first.push_back((uint32_t)seg_row.size());
            long_nseg.push_back(ns);
            for (uint32_t k = 0; k < ns; ++k) {
                seg_row.push_back(v);
                seg_lo.push_back(rp[v] + (int64_t)k * kLong);
                seg_long.push_back(li);
            }
        }
        LongRows& L = g->longs;
        L.n_long = (uint32_t)lr.size();
        L.n_segs = (uint32_t)seg_row.size();
        auto put = [&](DevBuf& d, const void* src, size_t bytes) {
            d.ensure(std::max<size_t>(bytes, 16), g->stream);
            if (bytes) CK(cudaMemcpyAsync(d.p, src, bytes, cudaMemcpyHostToDevice, s));
        };
        put(L.seg_row, seg_row.data(), seg_row.size() * 4);
        put(L.seg_lo, seg_lo.data(), seg_lo.size() * 8);
        put(L.seg_long, seg_long.data(), seg_long.size() * 4);
        put(L.long_first, long_first.data(), long_first.size() * 4);
        put(L.long_nseg, long_nseg.data(), long_nseg.size() * 4);
        // short-row blocks: consecutive short rows inside one aligned
        // window, at most kBlockNnz nnz (a lone row may reach kLong)
        std::vector<uint32_t> win_first;
        auto make_blocks = [&](uint32_t win) {
            std::vector<uint2> blocks;
            win_first.clear();
            for (uint32_t w0 = 0; w0 < n; w0 += win) {
                win_first.push_back((uint32_t)blocks.size());
                const uint32_t w1 = std::min<uint32_t>(n, w0 + win);
                uint32_t r = w0;
                while (r < w1) {
                    if (rp[r + 1] - rp[r] > kLong) {
                        ++r;
                        continue;
                    }
                    const uint32_t b0 = r;
                    int64_t nnz = 0;
                    while (r < w1 && rp[r + 1] - rp[r] <= kLong) {
                        const int64_t L2 = rp[r + 1] - rp[r];
                        if (r > b0 && nnz + L2 > kBlockNnz) break;
                        nnz += L2;
                        ++r;
                    }
                    blocks.push_back(make_uint2(b0, r - b0));
                }
            }
            win_first.push_back((uint32_t)blocks.size());
            return blocks;
        };
        std::vector<uint2> blocks = make_blocks(kMmRows);
        put(L.blocks, blocks.data(), blocks.size() * sizeof(uint2));
        for (int rows : {4, 8, 16, 32}) {
            std::vector<uint2> bw = make_blocks(rows);
            put(L.blocks_w[LongRows::wi(rows)], bw.data(), bw.size() * sizeof(uint2));
            put(L.win_blk_w[LongRows::wi(rows)], win_first.data(), win_first.size() * 4);
            L.n_blocks_w[LongRows::wi(rows)] = (uint32_t)bw.size();
        }
        g->n_blocks = (uint32_t)blocks.size();
        CK(cudaStreamSynchronize(s));
    }
    g->mv.n_items = (uint32_t)mv.size();
    g->mv.n_groups = (g->mv.n_items + kGroupItems - 1) / kGroupItems;
    g->mv.items.ensure(mv.size() * sizeof(uint2), g->stream);
    CK(cudaMemcpyAsync(g->mv.items.p, mv.data(), mv.size() * sizeof(uint2), cudaMemcpyHostToDevice, s));
    {
        std::vector<longlong2> nr(mv.size());
        for (size_t i = 0; i < mv.size(); ++i) {
            const uint32_t rb = mv[i].x, re = mv[i].y & ~kLongFlag;
            nr[i] = make_longlong2(rp[rb], rp[re]);
        }
        g->mv.item_nnz.ensure(nr.size() * sizeof(longlong2), g->stream);
        CK(cudaMemcpyAsync(g->mv.item_nnz.p, nr.data(), nr.size() * sizeof(longlong2), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
}

extern "C" {

int tpa_abi_version(void) { return TPA_ABI_VERSION; }
const char* tpa_last_error(void) { return tpa::last_error().c_str(); }

int tpa_graph_create(uint32_t n, uint64_t m, const uint64_t* out_offsets,
                     const uint32_t* out_targets, int policy, uint64_t fingerprint, int device,
                     tpa_graph** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output handle");
        if (n == 0) throw std::invalid_argument("graph must have at least one node");
        if (policy < 0 || policy > 2) throw std::invalid_argument("unknown dangling policy");
        if (out_offsets[n] != m) throw std::invalid_argument("out_offsets[n] != m");
        DeviceGuard dg(device);
        static std::once_flag once;
        std::call_once(once, [] { std::atexit(mark_exiting); });
        {
            const cudaError_t stale = cudaGetLastError();
            if (stale != cudaSuccess && std::getenv("TPA_DEBUG"))
                fprintf(stderr, "tpa: stale CUDA error before graph create: %s\n", cudaGetErrorString(stale));
        }
        auto g = std::make_unique<tpa_graph>();
        g->device = device;
        g->n = n;
        g->m = m;
        g->policy = policy;
        g->fingerprint = fingerprint;
        CK(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
        g->own_stream = true;
        cudaStream_t s = g->stream;
        {
            // keep freed blocks in the device pool (no release at sync points)
            cudaMemPool_t pool;
            CK(cudaDeviceGetDefaultMemPool(&pool, device));
            uint64_t thr = UINT64_MAX;
            CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
        }
        DevBuf d_off, d_tgt, d_src, d_keys;
        d_off.ensure((n + 1ull) * 8, g->stream);
        d_tgt.ensure(m * 4, g->stream);
        d_src.ensure(m * 4, g->stream);
        d_keys.ensure(m * 4, g->stream);
        g->col.ensure(m * 4, g->stream);
        g->deg.ensure((size_t)n * 4, g->stream);
        g->row_ptr.ensure((n + 1ull) * 8, g->stream);
        // one upload per array: the out-edge CSR stays on the device (frontier
        // push-marking of sparse sweeps) and the sort keys are a device copy
        g->out_tgt.ensure(std::max<uint64_t>(m, 1) * 4, g->stream);
        CK(cudaMemcpyAsync(d_off.p, out_offsets, (n + 1ull) * 8, cudaMemcpyHostToDevice, s));
        if (m) {
            CK(cudaMemcpyAsync(g->out_tgt.p, out_targets, m * 4, cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(d_tgt.p, g->out_tgt.p, m * 4, cudaMemcpyDeviceToDevice, s));
        }
        const int blocks = 8 * g->num_sms;
        k_degrees<<<blocks, 256, 0, s>>>(d_off.as<uint64_t>(), n, g->deg.as<uint32_t>());
        k_expand_src<<<blocks, 256, 0, s>>>(d_off.as<uint64_t>(), n, d_src.as<uint32_t>());
        CKL("k_expand_src");
        int end_bit = 1;
        while (end_bit < 32 && ((uint64_t)1 << end_bit) < n) ++end_bit;
        if (m) {
            // double-buffered (the key / value pairs ping-pong in place): no
            // third m-sized copy in the sort's temporary storage
            cub::DoubleBuffer<uint32_t> kb(d_tgt.as<uint32_t>(), d_keys.as<uint32_t>());
            cub::DoubleBuffer<uint32_t> vb(d_src.as<uint32_t>(), g->col.as<uint32_t>());
            size_t temp = 0;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, temp, kb, vb, (int64_t)m, 0, end_bit, s));
            DevBuf d_temp;
            d_temp.ensure(temp, g->stream);
            CK(cub::DeviceRadixSort::SortPairs(d_temp.p, temp, kb, vb, (int64_t)m, 0, end_bit, s));
            if (kb.Current() != d_keys.as<uint32_t>()) d_keys.swap(d_tgt);
            if (vb.Current() != g->col.as<uint32_t>()) g->col.swap(d_src);
        }
        d_src.release();
        d_tgt.release();
        k_row_ptr<<<blocks, 256, 0, s>>>(d_keys.as<uint32_t>(), m, n, g->row_ptr.as<int64_t>());
        g->out_off.swap(d_off);  // the uploaded offsets are the out-CSR's
        CKL("k_row_ptr");
        d_keys.release();
        // the ranked layout of the B = 1 sweeps, for share vectors beyond half
        // the L2 (C4: 134 MB, C5: 2.1 GB), if the column copy fits comfortably
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        if (m && (uint64_t)n * 8 > (64ull << 20) && m * 4 + (uint64_t)n * 24 < free_b / 2) {
            DevBuf keys, keys2, ids, perm, tmp;
            keys.ensure((size_t)n * 4, s);
            keys2.ensure((size_t)n * 4, s);
            ids.ensure((size_t)n * 4, s);
            perm.ensure((size_t)n * 4, s);
            k_rank_keys<<<blocks, 256, 0, s>>>(g->deg.as<uint32_t>(), n, keys.as<uint32_t>(), ids.as<uint32_t>());
            CKL("k_rank_keys");
            size_t temp = 0;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                               ids.as<uint32_t>(), perm.as<uint32_t>(), (int64_t)n, 0, 32, s));
            tmp.ensure(temp, s);
            CK(cub::DeviceRadixSort::SortPairs(tmp.p, temp, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                               ids.as<uint32_t>(), perm.as<uint32_t>(), (int64_t)n, 0, 32, s));
            g->rank.ensure((size_t)n * 4, g->stream);  // (DevBuf keeps the stream variable's address)
            k_rank_scatter<<<blocks, 256, 0, s>>>(perm.as<uint32_t>(), n, g->rank.as<uint32_t>());
            CKL("k_rank_scatter");
            g->col_rank.ensure(m * 4, g->stream);
            k_col_rank<<<blocks, 256, 0, s>>>(g->col.as<uint32_t>(), m, g->rank.as<uint32_t>(),
                                             g->col_rank.as<uint32_t>());
            CKL("k_col_rank");
            g->launches += 3;
        }
        std::vector<int64_t> rp(n + 1ull);
        CK(cudaMemcpyAsync(rp.data(), g->row_ptr.p, (n + 1ull) * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        g->launches += 4;

        build_schedules(g.get(), rp, n);
        CK(cudaStreamSynchronize(s));
        *out = g.release();
    });
}

int tpa_graph_destroy(tpa_graph* g) {
    return guard([&] {
        if (!g) return;
        if (g_exiting) return;  // process exit: the CUDA runtime may already be gone
        {
            DeviceGuard dg(g->device);
            if (g->part && g->part->ipc) ipc_teardown(g);  // peers' mappings before our buffers
            // stream-ordered frees first, then drain and drop the stream
            g->ws.clear();
            g->row_ptr.release();
            g->col.release();
            g->rank.release();
            g->col_rank.release();
            g->deg.release();
            g->out_off.release();
            g->out_tgt.release();
            g->mv.items.release();
            g->mv.item_nnz.release();
            for (DevBuf* d : {&g->longs.seg_row, &g->longs.seg_lo, &g->longs.seg_long, &g->longs.long_first,
                              &g->longs.long_nseg, &g->longs.blocks, &g->longs.blocks_w[0],
                              &g->longs.blocks_w[1], &g->longs.blocks_w[2], &g->longs.blocks_w[3],
                              &g->longs.win_blk_w[0], &g->longs.win_blk_w[1], &g->longs.win_blk_w[2],
                              &g->longs.win_blk_w[3]})
                d->release();
            g->init_part.release();
            for (DevBuf* d : {&g->topk.st, &g->topk.hist, &g->topk.cand, &g->topk.ids}) d->release();
            if (g->pipe.copy) {
                cudaStreamSynchronize(g->pipe.copy);
                for (int k = 0; k < 2; ++k) {
                    g->pipe.stage[k].release();
                    cudaEventDestroy(g->pipe.done[k]);
                    cudaEventDestroy(g->pipe.free_[k]);
                }
            }
            for (tpa_artifact* a : g->artifacts) detach_artifact(a);
            g->artifacts.clear();
            cudaStreamSynchronize(g->stream);
            for (auto& pe : g->prof_events) {
                cudaEventDestroy(pe.e0);
                cudaEventDestroy(pe.e1);
            }
            for (auto e : g->event_pool) cudaEventDestroy(e);
            if (g->own_stream) cudaStreamDestroy(g->stream);
            if (g->pipe.copy) cudaStreamDestroy(g->pipe.copy);
            if (g->part) part_comm_destroy(g->part->comm);
        }
        delete g;
    });
}

int tpa_graph_sync(tpa_graph* g) {
    return guard([&] {
        if (!g) throw std::invalid_argument("null graph");
        DeviceGuard dg(g->device);
        CK(cudaStreamSynchronize(g->stream));
        if (g->pipe.copy) CK(cudaStreamSynchronize(g->pipe.copy));
    });
}

int tpa_graph_set_stream(tpa_graph* g, void* cuda_stream) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        CK(cudaStreamSynchronize(g->stream));
        if (g->own_stream) cudaStreamDestroy(g->stream);
        if (cuda_stream) {
            g->stream = static_cast<cudaStream_t>(cuda_stream);
            g->own_stream = false;
        } else {
            CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
            g->own_stream = true;
        }
    });
}

int tpa_graph_info(const tpa_graph* g, uint32_t* n, uint64_t* m, uint64_t* fingerprint, int* policy,
                   uint64_t* device_bytes) {
    return guard([&] {
        if (n) *n = g->part ? g->part->n_global : g->n;  // the graph's size, also for a partition
        if (m) *m = g->part ? g->part->m_global : g->m;
        if (fingerprint) *fingerprint = g->fingerprint;
        if (policy) *policy = g->policy;
        if (device_bytes) {
            uint64_t b = g->row_ptr.bytes + g->col.bytes + g->rank.bytes + g->col_rank.bytes + g->deg.bytes + g->mv.items.bytes + g->longs.seg_lo.bytes * 2 +
                         g->out_off.bytes + g->out_tgt.bytes;
            for (auto& kv : g->ws) {
                const Workspace& w = *kv.second;
                b += w.share[0].bytes + w.share[1].bytes + w.acc.bytes + w.part.bytes + w.gpart.bytes;
            }
            *device_bytes = b;
        }
    });
}

uint64_t tpa_graph_launches(const tpa_graph* g) { return g ? g->launches : 0; }

int tpa_graph_profile(tpa_graph* g, int enable) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        if (enable) {
            CK(cudaStreamSynchronize(g->stream));
            for (auto& pe : g->prof_events) {
                g->event_pool.push_back(pe.e0);
                g->event_pool.push_back(pe.e1);
            }
            g->prof_events.clear();
        }
        g->profile = enable != 0;
    });
}

int tpa_graph_profile_read(tpa_graph* g, int width, int step, uint64_t* launches, double* total_ms) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        CK(cudaStreamSynchronize(g->stream));
        uint64_t cnt = 0;
        double tot = 0.0;
        for (auto& pe : g->prof_events) {
            if (pe.width != width || (step >= 0 && (int)pe.step != step)) continue;
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, pe.e0, pe.e1));
            tot += ms;
            ++cnt;
        }
        if (launches) *launches = cnt;
        if (total_ms) *total_ms = tot;
    });
}

int tpa_graph_transpose(const tpa_graph* g, int64_t* row_ptr, uint32_t* col) {
    return guard([&] {
        require_whole(g, "tpa_graph_transpose");
        DeviceGuard dg(g->device);
        if (row_ptr) CK(cudaMemcpy(row_ptr, g->row_ptr.p, (g->n + 1ull) * 8, cudaMemcpyDeviceToHost));
        if (col && g->m) CK(cudaMemcpy(col, g->col.p, g->m * 4, cudaMemcpyDeviceToHost));
    });
}

int tpa_propagation_sweep(tpa_graph* g, const double* x, double* y, double c, int flags) {
    return guard([&] {
        require_whole(g, "tpa_propagation_sweep");
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        // graph.cpp:233-235
        if (c < 0.0 || c >= 1.0) throw std::invalid_argument("restart probability must be in [0, 1)");
        const bool dev = flags & TPA_DEVICE_PTRS;
        const size_t nb = (size_t)g->n * 8;
        DevBuf dx, dy;
        const double* xd = x;
        double* yd = y;
        if (!dev) {
            dx.ensure(nb, g->stream);
            dy.ensure(nb, g->stream);
            upload(g, dx.p, x, nb);
            xd = dx.as<double>();
            yd = dy.as<double>();
        }
        RunCfg cfg;
        cfg.B = 1;
        cfg.c = c;
        cfg.eps = 1.0;  // no convergence semantics for a single sweep
        cfg.terminal = 1;
        cfg.init = Init::Dense;
        cfg.d_x = xd;
        cfg.signed_x = true;
        cfg.y_out = yd;
        cfg.want_state = false;
        // c == 0 is legal for a sweep; the driver only uses keep = 1 - c.
        run_cpi(g, cfg, nullptr);
        if (!dev) download(g, y, yd, nb);
        finish(g, flags);
    });
}

int tpa_cpi_run(tpa_graph* g, const uint32_t* seeds, uint64_t n_seeds, double c, double eps,
                uint32_t start_iter, int64_t terminal_iter, double* out_scores,
                uint32_t* iterations_run, int* converged, double* residual_l1, int flags) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        if (g->part) {  // collective over the partitions (cpi.cpp:87-101 per rank)
            require_solo_part(g);
            std::vector<tpa_graph*> Pg{g};
            part_cpi_run(Pg, seeds, n_seeds, c, eps, start_iter, terminal_iter, out_scores, iterations_run,
                         converged, residual_l1);
            return;
        }
        const bool dev = flags & TPA_DEVICE_PTRS;
        std::vector<uint32_t> hs;
        if (seeds) {
            // SeedSet (cpi.cpp:19-24): non-empty, sorted, duplicate-free
            if (n_seeds == 0) throw std::invalid_argument("seed set must not be empty");
            hs.assign(seeds, seeds + n_seeds);  // host array (see tpa_gpu.h)
            std::sort(hs.begin(), hs.end());
            if (std::adjacent_find(hs.begin(), hs.end()) != hs.end())
                throw std::invalid_argument("seed set contains duplicate ids");
        }
        validate_cpi(c, eps, start_iter, terminal_iter);
        if (seeds) validate_seed(hs.back(), g->n);
        const uint32_t n = g->n;
        Workspace& w = g->workspace(1);
        RunCfg cfg;
        cfg.B = 1;
        cfg.c = c;
        cfg.eps = eps;
        cfg.start = start_iter;
        cfg.terminal = terminal_iter;
        cfg.acc = dev ? out_scores : w.acc.as<double>();
        DevBuf dx;
        if (!seeds) {
            cfg.init = Init::Dense;
            cfg.weight = c / (double)n;  // cpi.cpp:61
        } else if (hs.size() == 1) {
            cfg.init = Init::Seeds;
            cfg.seeds.s[0] = hs[0];
        } else {
            std::vector<double> x0(n, 0.0);
            const double wgt = c / (double)hs.size();
            for (uint32_t s : hs) x0[s] = wgt;
            dx.ensure((size_t)n * 8, g->stream);
            upload(g, dx.p, x0.data(), (size_t)n * 8);
            cfg.init = Init::Dense;
            cfg.d_x = dx.as<double>();
            CK(cudaStreamSynchronize(g->stream));
        }
        RunOut ro;
        run_cpi(g, cfg, &ro);
        if (!dev) download(g, out_scores, cfg.acc, (size_t)n * 8);
        CK(cudaStreamSynchronize(g->stream));
        if (iterations_run) *iterations_run = ro.state[0].iters;
        if (converged) *converged = ro.state[0].converged;
        if (residual_l1) *residual_l1 = ro.state[0].residual;
    });
}

int tpa_cpi_partition(tpa_graph* g, const uint32_t* seeds, uint64_t n_seeds, double c, double eps,
                      const uint32_t* boundaries, uint64_t n_boundaries, double* out, int flags) {
    return guard([&] {
        require_whole(g, "tpa_cpi_partition");
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        const bool dev = flags & TPA_DEVICE_PTRS;
        // cpi.cpp:117-125
        std::vector<uint32_t> hs;
        if (seeds == nullptr || n_seeds == 0) throw std::invalid_argument("seed set must not be empty");
        hs.assign(seeds, seeds + n_seeds);
        std::sort(hs.begin(), hs.end());
        if (std::adjacent_find(hs.begin(), hs.end()) != hs.end())
            throw std::invalid_argument("seed set contains duplicate ids");
        validate_cpi(c, eps, 0, -1);
        std::vector<uint32_t> bounds(boundaries, boundaries + n_boundaries);
        for (size_t k = 0; k < bounds.size(); ++k) {
            const uint32_t lo = k == 0 ? 1 : bounds[k - 1] + 1;
            if (bounds[k] < lo)
                throw std::invalid_argument("partition boundaries must be strictly increasing and >= 1");
        }
        validate_seed(hs.back(), g->n);
        const uint32_t n = g->n;
        const size_t nseg = bounds.size() + 1;
        DevBuf segs, dx;
        double* base = out;
        if (!dev) {
            segs.ensure(nseg * n * 8, g->stream);
            base = segs.as<double>();
        }
        RunCfg cfg;
        cfg.B = 1;
        cfg.c = c;
        cfg.eps = eps;
        cfg.bounds = bounds;
        for (size_t k = 0; k < nseg; ++k) cfg.seg_acc.push_back(base + k * n);
        Workspace& w = g->workspace(1);
        if (hs.size() == 1) {
            cfg.init = Init::Seeds;
            cfg.seeds.s[0] = hs[0];
        } else {
            std::vector<double> x0(n, 0.0);
            const double wgt = c / (double)hs.size();
            for (uint32_t s : hs) x0[s] = wgt;
            dx.ensure((size_t)n * 8, g->stream);
            upload(g, dx.p, x0.data(), (size_t)n * 8);
            cfg.init = Init::Dense;
            cfg.d_x = dx.as<double>();
            CK(cudaStreamSynchronize(g->stream));
        }
        RunOut ro;
        run_cpi(g, cfg, &ro);
        if (!dev) download(g, out, base, nseg * n * 8);
        finish(g, flags);
    });
}

int tpa_exact_rwr_batch(tpa_graph* g, const uint32_t* seeds, uint32_t B, double c, double eps,
                        double* out, int flags) {
    return guard([&] {
        require_whole(g, "tpa_exact_rwr_batch");
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        if (B == 0) throw std::invalid_argument("seed set must not be empty");
        validate_cpi(c, eps, 0, -1);
        run_seed_batch(g, seeds, B, c, eps, 0, -1, nullptr, 1.0, false, out, flags);
    });
}

double tpa_neighbor_scale_factor(double c, uint32_t S, uint32_t T) {
    // tpa.cpp:39-44 -- host std::pow, exactly as the reference.
    const double keep = 1.0 - c;
    const double family_mass = 1.0 - std::pow(keep, S);
    const double neighbor_mass = std::pow(keep, S) - std::pow(keep, T);
    return neighbor_mass / family_mass;
}

int tpa_preprocess(tpa_graph* g, double c, double eps, uint32_t T, double* out_stranger,
                   tpa_artifact** out_artifact, int flags) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        if (g->part) {  // collective over the partitions; no device artifact (queries run on replicas)
            require_solo_part(g);
            if (out_artifact) throw std::invalid_argument("a row-partitioned graph returns the stranger vector only");
            std::vector<tpa_graph*> Pg{g};
            part_preprocess(Pg, c, eps, T, out_stranger);
            return;
        }
        if (T < 1) throw std::invalid_argument("stranger_start (T) must be at least 1");  // tpa.cpp:21-22
        validate_cpi(c, eps, T, -1);
        const bool dev = flags & TPA_DEVICE_PTRS;
        auto art = std::make_unique<tpa_artifact>();
        art->g = g;
        art->fingerprint = g->fingerprint;
        art->c = c;
        art->eps = eps;
        art->T = T;
        art->n = g->n;
        art->stranger.ensure((size_t)g->n * 8, g->stream);
        RunCfg cfg;
        cfg.B = 1;
        cfg.c = c;
        cfg.eps = eps;
        cfg.start = T;
        cfg.terminal = -1;
        cfg.init = Init::Dense;
        cfg.weight = c / (double)g->n;
        cfg.acc = art->stranger.as<double>();
        cfg.want_state = false;
        run_cpi(g, cfg, nullptr);
        if (out_stranger) {
            if (dev)
                CK(cudaMemcpyAsync(out_stranger, art->stranger.p, (size_t)g->n * 8, cudaMemcpyDeviceToDevice,
                                   g->stream));
            else
                download(g, out_stranger, art->stranger.p, (size_t)g->n * 8);
        }
        finish(g, flags);
        if (out_artifact) {
            g->artifacts.insert(art.get());
            *out_artifact = art.release();
        }
    });
}

int tpa_artifact_create(tpa_graph* g, const double* stranger, uint64_t graph_fingerprint, double c,
                        double eps, uint32_t T, int flags, tpa_artifact** out) {
    return guard([&] {
        require_whole(g, "tpa_artifact_create");
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        auto art = std::make_unique<tpa_artifact>();
        art->g = g;
        art->fingerprint = graph_fingerprint;
        art->c = c;
        art->eps = eps;
        art->T = T;
        art->n = g->n;
        art->stranger.ensure((size_t)g->n * 8, g->stream);
        CK(cudaMemcpyAsync(art->stranger.p, stranger, (size_t)g->n * 8,
                           (flags & TPA_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                           g->stream));
        CK(cudaStreamSynchronize(g->stream));
        g->artifacts.insert(art.get());
        *out = art.release();
    });
}

int tpa_artifact_destroy(tpa_artifact* a) {
    return guard([&] {
        if (!a) return;
        if (g_exiting) return;
        if (tpa_graph* g = a->g) {
            std::lock_guard<std::mutex> lk(g->mu);
            DeviceGuard dg(g->device);
            g->artifacts.erase(a);
            a->stranger.release();
        }
        delete a;
    });
}

static void check_query(tpa_graph* g, const tpa_artifact* a, uint32_t S) {
    // tpa.cpp:63-66, then cpi_run's CpiParams::validate with the artifact's c/eps (tpa.cpp:69)
    if (a->fingerprint != g->fingerprint)
        throw std::runtime_error("stale artifact: graph fingerprint mismatch");
    if (a->n != g->n) throw std::runtime_error("stale artifact: graph fingerprint mismatch");
    if (a->g == nullptr) throw std::runtime_error("artifact outlived its graph handle");
    if (a->g->device != g->device) throw std::invalid_argument("artifact lives on another device");
    if (S < 1 || S >= a->T) throw std::invalid_argument("family_end (S) must satisfy 1 <= S < T");
    validate_cpi(a->c, a->eps, 0, (int64_t)S - 1);
}

int tpa_query(tpa_graph* g, const tpa_artifact* a, uint32_t seed, uint32_t S, double* out, int flags) {
    return guard([&] {
        require_whole(g, "tpa_query");
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        if (!a) throw std::invalid_argument("null artifact");
        check_query(g, a, S);
        const double scale = 1.0 + tpa_neighbor_scale_factor(a->c, S, a->T);
        run_seed_batch(g, &seed, 1, a->c, a->eps, 0, (int64_t)S - 1, a->stranger.as<double>(), scale, true,
                       out, flags);
    });
}

int tpa_query_batch(tpa_graph* g, const tpa_artifact* a, const uint32_t* seeds, uint32_t B, uint32_t S,
                    double* out, int flags) {
    return guard([&] {
        require_whole(g, "tpa_query_batch");
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        if (!a) throw std::invalid_argument("null artifact");
        check_query(g, a, S);
        if (B == 0) return;
        const bool na = flags & TPA_QUERY_NA;
        const double scale = 1.0 + tpa_neighbor_scale_factor(a->c, S, a->T);  // tpa.cpp:71-72
        run_seed_batch(g, seeds, B, a->c, a->eps, 0, (int64_t)S - 1, na ? nullptr : a->stranger.as<double>(),
                       scale, true, out, flags);
    });
}

int tpa_query_na_batch(tpa_graph* g, const uint32_t* seeds, uint32_t B, uint32_t S, uint32_t T, double c,
                       double eps, double* out, int flags) {
    return guard([&] {
        require_whole(g, "tpa_query_na_batch");
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        // TpaParams::validate (tpa.cpp:8-17)
        if (S < 1) throw std::invalid_argument("family_end (S) must be at least 1");
        if (T <= S) throw std::invalid_argument("stranger_start (T) must exceed family_end (S)");
        validate_cpi(c, eps, 0, -1);
        if (B == 0) return;
        const double scale = 1.0 + tpa_neighbor_scale_factor(c, S, T);
        run_seed_batch(g, seeds, B, c, eps, 0, (int64_t)S - 1, nullptr, scale, true, out, flags);
    });
}

}  // extern "C"

#include "tpa_part.cuh"
#include "tpa_topk.cuh"
#include "tpa_graph_build.cuh"
#include "tpa_artifact_io.cuh"
