// cpi_kernels.cuh -- sm_100a kernels for the Cumulative Power Iteration step.
//
// Replaces the reference's CPU hot loop:
//   propagation_sweep / sweep_range   proj/src/graph.cpp:211-270
//   l1_sum / add_into / run_series    proj/src/cpi.cpp:43-83
//   query combine                     proj/src/tpa.cpp:70-74, :84
//
// Representation.  The reference pushes x[u]·keep/deg(u) along
// out-edges.  Here every sweep is a PULL over CSR(Ãᵀ): row v lists its
// in-neighbours u in ascending order.  The iterate is stored as its *share*
//   share[u] = (keep · x[u]) / deg(u)            (graph.cpp:222, same rounding)
// so a sweep is a pure gather-sum  y[v] = Σ_u share[u]  and the n divisions
// per column happen once per row in the epilogue (not once per edge).  The
// epilogue of sweep i fuses, per row and column:
//   + Uniform spread   (graph.cpp:265-268, from the dangling mass of x⁽ⁱ⁻¹⁾)
//   acc += y           (cpi.cpp:49-51, predicated on the window cpi.cpp:95-96)
//   out = scale·acc + stranger          (tpa.cpp:73-74, last family sweep)
//   share_next = keep·y / deg           (input of sweep i+1)
//   L1 residual and dangling-mass partials (cpi.cpp:74, graph.cpp:218-221)
// and the last CTA to finish reduces the partials in a FIXED order and
// advances the per-column convergence state (cpi.cpp:75-80), so no host
// synchronisation is needed between sweeps and results are deterministic.
//
// All fp64 arithmetic goes through __dadd_rn/__dmul_rn/__ddiv_rn so nothing is
// contracted into an FMA (the reference is compiled without FMA).  Row sums:
//   SpMM (B >= 8 seeds, lane = column): strictly sequential ascending-source
//     order for rows <= kMmLongRow, i.e. bitwise the reference's scatter order;
//     longer rows: 8 fixed chunks, each sequential, combined in chunk order.
//   SpMV (B = 1): rows <= 32 sequential; longer rows a fixed lane/warp tree.
// Both orders depend on the row alone, never on timing.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tpa {

constexpr int kSelfLoop = 0, kUniform = 1, kDrop = 2;
constexpr uint32_t kLongFlag = 0x80000000u;
constexpr int kThreads = 256;         // CTA size of every step kernel
constexpr int kGroupItems = 128;      // items per first-level ticket group

// SpMV (B = 1) tiling.
constexpr int kMvTileNnz = 2048;  // largest SpMV tile (nnz); see mv_shape (cpi_spmv2.cuh)
constexpr int kMvTileRows = 512;
constexpr int kMvShortRow = 32;       // rows <= this: one thread, sequential

// Per-column CPI state, double-buffered by sweep parity.
struct ColState {
    double residual;    // ||x^(iters)||_1
    double spread;      // Uniform: (keep*dm)/n added by the next sweep
    uint32_t iters;     // index of the last interim vector computed
    int32_t active;     // next sweep computes this column
    int32_t converged;  // tolerance break fired
    int32_t has_spread; // dm != 0 under Uniform
};

// Up to 64 seeds travel as a kernel parameter: no host->device copy, so
// back-to-back query batches never wait on a staging buffer.
struct SeedList {
    uint32_t s[64];
};

struct StepArgs {
    const int64_t* __restrict__ row_ptr;  // CSR(Ãᵀ) n+1
    const uint32_t* __restrict__ col;     // m, ascending per row
    const uint32_t* __restrict__ deg;     // out-degree per node (n)
    const uint32_t* __restrict__ rank;    // B = 1 ranked layout: share slot of node v (null: v)
    const uint2* __restrict__ items;      // {row_begin, row_end | kLongFlag}
    uint32_t n_items;
    uint32_t n;
    int policy;
    double keep;                          // 1 - c
    double eps;
    int64_t terminal;                     // -1: run to convergence
    uint32_t step;                        // i of x^(i) produced by this sweep

    const double* __restrict__ share_in;  // n x B
    double* __restrict__ share_out;       // n x B, null on the last sweep
    double* __restrict__ y_out;           // n x B raw x^(i) (sweep API), or null
    double* __restrict__ acc;             // n x B, null outside the window
    double* __restrict__ out;             // combine target, or null
    const double* __restrict__ stranger;  // n, null for query_na
    double scale;                         // 1 + nsf
    int out_node_major;                   // out layout: 1 -> [n][B], 0 -> [B][n]
    uint32_t b_valid;                     // columns < b_valid are real seeds

    const ColState* state_in;
    ColState* state_out;
    double* part;                         // n_items x 2B   (l1 | dm)
    double* gpart;                        // n_groups x 2B
    uint32_t* group_cnt;                  // n_groups, zero between launches
    uint32_t* done_cnt;                   // 1, zero between launches
};

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

__device__ __forceinline__ uint32_t ld_nc_u32(const uint32_t* p) { return __ldg(p); }

// Streaming read of the CSR index array: read once per sweep, keep it out of L1.
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// Loads of the sweeps' read-once streams and the gathered iterate.  (L2
// eviction-priority hints on these were measured without gain and with extra
// register pressure: profiles/r02_experiments.md.)
__device__ __forceinline__ uint32_t ld_col(const uint32_t* p) {  // CSR indices: keep them out of L1
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// Deterministic warp sum: xor butterfly, every lane ends with the same value.
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = dadd(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic CTA sum (fixed tree); result valid in every thread.
__device__ __forceinline__ double block_sum(double v, double* s_red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) s_red[w] = v;
    __syncthreads();
    double r = s_red[0];
#pragma unroll
    for (int k = 1; k < kThreads / 32; ++k) r = dadd(r, s_red[k]);
    __syncthreads();
    return r;
}

// Column sums of src[count][2B] (l1 | dm halves) in a fixed order into
// dst[2B] (shared).  B2 = 2B <= kThreads, power of two.
__device__ __forceinline__ void ordered_column_sums(const double* src, uint32_t count, int B2,
                                                    double* s_scr, double* dst) {
    const int tid = threadIdx.x;
    const int nsl = kThreads / B2;
    const int b = tid % B2, sl = tid / B2;
    const uint32_t per = (count + nsl - 1) / nsl;
    const uint32_t k0 = sl * per;
    const uint32_t k1 = min(count, k0 + per);
    double s = 0.0;
    for (uint32_t k = k0; k < k1; ++k) s = dadd(s, __ldcg(src + (size_t)k * B2 + b));
    s_scr[tid] = s;
    __syncthreads();
    for (int w = nsl / 2; w > 0; w >>= 1) {
        if (sl < w) s_scr[tid] = dadd(s_scr[tid], s_scr[tid + w * B2]);
        __syncthreads();
    }
    if (sl == 0) dst[b] = s_scr[b];
    __syncthreads();
}

// Publishes this item's (l1 | dm) partials (smem s_part[2B]) and, if it is the
// last item of its group and then the last group, reduces everything in fixed
// order and writes the next column state.  Must be reached by all threads.
__device__ __forceinline__ void finish_item(const StepArgs& a, uint32_t item, int B,
                                            const double* s_part, double* s_scr,
                                            double* s_fin) {
    const int tid = threadIdx.x;
    const int B2 = 2 * B;
    __shared__ uint32_t s_ticket;
    for (int b = tid; b < B2; b += kThreads) a.part[(size_t)item * B2 + b] = s_part[b];
    __threadfence();
    __syncthreads();
    const uint32_t g = item / kGroupItems;
    const uint32_t g0 = g * kGroupItems;
    const uint32_t gsize = min((uint32_t)kGroupItems, a.n_items - g0);
    if (tid == 0) s_ticket = atomicAdd(&a.group_cnt[g], 1u);
    __syncthreads();
    if (s_ticket != gsize - 1) return;
    __threadfence();
    ordered_column_sums(a.part + (size_t)g0 * B2, gsize, B2, s_scr, s_fin);
    for (int b = tid; b < B2; b += kThreads) a.gpart[(size_t)g * B2 + b] = s_fin[b];
    if (tid == 0) a.group_cnt[g] = 0;
    __threadfence();
    __syncthreads();
    const uint32_t n_groups = (a.n_items + kGroupItems - 1) / kGroupItems;
    if (tid == 0) s_ticket = atomicAdd(a.done_cnt, 1u);
    __syncthreads();
    if (s_ticket != n_groups - 1) return;
    __threadfence();
    ordered_column_sums(a.gpart, n_groups, B2, s_scr, s_fin);
    // cpi.cpp:73-80 -- iterations_run, residual, convergence break, terminal.
    for (int b = tid; b < B; b += kThreads) {
        ColState s = a.state_in[b];
        if (s.active) {
            const double res = s_fin[b];
            const double dm = s_fin[B + b];
            s.residual = res;
            s.iters = a.step;
            s.converged = res < a.eps;
            s.active = !s.converged && (a.terminal < 0 || (int64_t)a.step < a.terminal);
            s.has_spread = (a.policy == kUniform && dm != 0.0);
            s.spread = s.has_spread ? ddiv(dmul(a.keep, dm), (double)a.n) : 0.0;
        }
        a.state_out[b] = s;
    }
    if (tid == 0) *a.done_cnt = 0;
}

// Row/column epilogue shared by both kernels.  idx = storage index of (v, b)
// in the n x B node-major iterate.  Returns y (= x^(i)[v][b]).
__device__ __forceinline__ double epilogue(const StepArgs& a, const ColState& st, uint32_t v,
                                           uint32_t b, int B, size_t idx, double y,
                                           uint32_t d) {
    if (st.has_spread) y = dadd(y, st.spread);  // graph.cpp:265-268
    if (a.y_out) a.y_out[idx] = y;
    if (a.acc) {
        const double f = dadd(a.acc[idx], y);   // cpi.cpp:50
        if (a.out) {
            if (b < a.b_valid) {
                const size_t o = a.out_node_major ? idx : (size_t)b * a.n + v;
                a.out[o] = a.stranger ? dadd(dmul(a.scale, f), a.stranger[v])  // tpa.cpp:73-74
                                      : dmul(f, a.scale);                     // tpa.cpp:84
            }
        } else {
            a.acc[idx] = f;
        }
    }
    if (a.share_out) a.share_out[idx] = d ? ddiv(dmul(a.keep, y), (double)d) : 0.0;  // graph.cpp:222
    return y;
}

// Combine for a column that already stopped before the last family sweep.
__device__ __forceinline__ void combine_only(const StepArgs& a, uint32_t v, uint32_t b, int B,
                                             size_t idx) {
    if (a.out && a.acc && b < a.b_valid) {
        const double f = a.acc[idx];
        const size_t o = a.out_node_major ? idx : (size_t)b * a.n + v;
        a.out[o] = a.stranger ? dadd(dmul(a.scale, f), a.stranger[v]) : dmul(f, a.scale);
    }
}

// ---------------------------------------------------------------------------
// K3 (SpMM, B in {8,16,32,64}) lives in cpi_spmm.cuh.  Shape helpers: G =
// min(B,32) lanes per row, CPL = B/G columns per lane.
// ---------------------------------------------------------------------------
template <int B>
struct MmVec;
template <> struct MmVec<8> { static constexpr int G = 8, CPL = 1; };
template <> struct MmVec<16> { static constexpr int G = 16, CPL = 1; };
template <> struct MmVec<32> { static constexpr int G = 32, CPL = 1; };
template <> struct MmVec<64> { static constexpr int G = 32, CPL = 2; };

// One lane's CPL columns of a gathered share row (B >= 8).
template <int CPL>
__device__ __forceinline__ void ld_cols(const double* p, double (&v)[CPL]) {
    if constexpr (CPL == 1) {
        v[0] = __ldg(p);
    } else {
        const double2 t = __ldg(reinterpret_cast<const double2*>(p));
        v[0] = t.x;
        v[1] = t.y;
    }
}

}  // namespace tpa
