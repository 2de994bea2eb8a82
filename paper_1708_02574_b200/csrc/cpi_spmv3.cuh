// cpi_spmv3.cuh -- K2 v3: the B = 1 sweep (PageRank / single-vector CPI) as
// independent warps, no CTA-wide barrier on the data path.
//
// v2 (cpi_spmv2.cuh) staged 2048-nnz tiles through shared memory with two
// __syncthreads per tile; ncu showed "barrier" as the top stall and the L2
// sector rate at ~18% of peak.  Here every warp owns its work:
//   * a block = up to 32 consecutive rows (one per lane) with <= 512 nnz,
//     or one 512-nnz segment of a longer row (the SpMM's LongRows lists);
//   * the warp loads the block's indices coalesced (16 per lane in flight),
//     then gathers share_in[u] (16 per lane in flight) and parks them in its
//     shared-memory slice (LDG, not cp.async: tools/gather8_micro.cu measures
//     ~1 gather/clk/SM for LDG and 0.38 for 8-byte cp.async);
//   * lane k then sums row k in ascending source order from shared memory
//     (rows <= 32 nnz: bitwise the reference's sequential order, graph.cpp:
//     249-259); rows of 33..512 nnz use the fixed lane-strided + butterfly
//     order of v2; a segmented row's partials are added in segment order by
//     the last finisher (deterministic);
//   * |y| and the dangling mass go into exact 128-bit fixed-point
//     accumulators per lane (order-free), reduced once per CTA at the end;
//     the last CTA advances the ColState (cpi.cpp:73-80).
// Persistent grid, static round-robin over equal-cost blocks.
#pragma once

#include "cpi_spmv2.cuh"

namespace tpa {

constexpr int kMv3Nnz = 512;  // nnz per block (== kLong: longer rows are segmented)
constexpr int kMv3Pl = kMv3Nnz / 32;
#ifndef TPA_MV3_WARPS
#define TPA_MV3_WARPS 8
#endif
#ifndef TPA_MV3_MINB
#define TPA_MV3_MINB 1
#endif
constexpr int kMv3Warps = TPA_MV3_WARPS;
constexpr int kMv3Threads = kMv3Warps * 32;

struct Mv3Args {
    StepArgs s;
    const uint32_t* __restrict__ seg_row;
    const int64_t* __restrict__ seg_lo;
    const uint32_t* __restrict__ seg_long;
    const uint32_t* __restrict__ long_first;
    const uint32_t* __restrict__ long_nseg;
    uint32_t n_segs;
    const uint2* __restrict__ blocks;  // {first row, rows <= 32}
    uint32_t n_blocks;
    uint32_t* long_cnt;                // [n_long], zero between launches
    double* seg_part;                  // [n_segs]
    unsigned long long* fx;            // [4], zero between launches
};

__device__ __forceinline__ void cp_async_f64(double* dst_smem, const double* src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst_smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}

// One row's epilogue (graph.cpp:222, 265-268; cpi.cpp:50; tpa.cpp:73-74, 84),
// with the accumulator value already loaded; returns the spread-adjusted y.
__device__ __forceinline__ double mv3_row(const StepArgs& a, const ColState& st, uint32_t v, double y,
                                          uint32_t d, double acc_v) {
    if (st.has_spread) y = dadd(y, st.spread);
    if (a.y_out) a.y_out[v] = y;
    if (a.acc) {
        const double f = dadd(acc_v, y);
        if (a.out) a.out[v] = a.stranger ? dadd(dmul(a.scale, f), a.stranger[v]) : dmul(f, a.scale);
        else a.acc[v] = f;
    }
    if (a.share_out) a.share_out[v] = d ? ddiv(dmul(a.keep, y), (double)d) : 0.0;
    return y;
}

__global__ void __launch_bounds__(kMv3Threads, TPA_MV3_MINB) k_step_spmv3(Mv3Args M) {
    const StepArgs& a = M.s;
    __shared__ __align__(16) double s_v[kMv3Warps][kMv3Nnz];
    __shared__ unsigned long long s_fx[4];
    __shared__ uint32_t s_ticket;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const ColState st = a.state_in[0];
    if (!st.active) {
        // column stopped earlier: only a pending combine remains (tpa.cpp:73)
        if (a.out)
            for (uint32_t v = blockIdx.x * kMv3Threads + tid; v < a.n; v += gridDim.x * kMv3Threads)
                combine_only(a, v, 0, 1, v);
        if (blockIdx.x == 0 && tid == 0) a.state_out[0] = st;
        return;
    }
    if (tid < 4) s_fx[tid] = 0ull;
    const bool want_dm = a.policy == kUniform;
    unsigned long long f0 = 0, f1 = 0, f2 = 0, f3 = 0;
    double* sv = s_v[wid];
    const uint32_t total = M.n_segs + M.n_blocks;
    const uint32_t nwarps = gridDim.x * kMv3Warps;

    for (uint32_t item = blockIdx.x * kMv3Warps + wid; item < total; item += nwarps) {
        if (item < M.n_segs) {
            // one 512-nnz segment of a long row: lane-strided sum + butterfly
            const uint32_t r = M.seg_row[item];
            const int64_t lo = M.seg_lo[item];
            const int64_t hi = min(lo + (int64_t)kMv3Nnz, (int64_t)__ldg(a.row_ptr + r + 1));
            const int len = (int)(hi - lo);
            uint32_t u[kMv3Pl];
#pragma unroll
            for (int j = 0; j < kMv3Pl; ++j) u[j] = j * 32 + lane < len ? ld_stream_u32(a.col + lo + j * 32 + lane) : 0u;
            {
                double v[kMv3Pl];
#pragma unroll
                for (int j = 0; j < kMv3Pl; ++j) v[j] = j * 32 + lane < len ? __ldg(a.share_in + u[j]) : 0.0;
#pragma unroll
                for (int j = 0; j < kMv3Pl; ++j) sv[j * 32 + lane] = v[j];
            }
            __syncwarp();
            double s = 0.0;
            for (int k = lane; k < len; k += 32) s = dadd(s, sv[k]);
            s = warp_sum(s);
            __syncwarp();
            uint32_t t = 0;
            const uint32_t li = M.seg_long[item];
            if (lane == 0) {
                M.seg_part[item] = s;
                __threadfence();
                t = atomicAdd(M.long_cnt + li, 1u);
            }
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t != M.long_nseg[li] - 1) continue;
            if (lane == 0) {
                __threadfence();
                const uint32_t fs = M.long_first[li], ns = M.long_nseg[li];
                double y = seg_sum(M.seg_part + fs, 1, ns);
                const uint32_t d = __ldg(a.deg + r);
                y = mv3_row(a, st, r, y, d, a.acc ? a.acc[r] : 0.0);
                fx_add(f0, f1, y);
                if (want_dm && d == 0 && y != 0.0) fx_add(f2, f3, y);  // sign: dm >= 0 here
                M.long_cnt[li] = 0;
            }
            continue;
        }
        // a block of <= 32 short rows, lane k <-> row r0 + k
        const uint2 blk = M.blocks[item - M.n_segs];
        const uint32_t r0 = blk.x;
        const int nr = (int)blk.y;
        const bool has = lane < nr;
        const int64_t e0 = __ldg(a.row_ptr + r0);
        const int64_t rend = has ? __ldg(a.row_ptr + r0 + lane + 1) : 0;
        const uint32_t d = has ? __ldg(a.deg + r0 + lane) : 0u;
        const double acc_v = (has && a.acc) ? a.acc[r0 + lane] : 0.0;
        const int64_t e1 = __shfl_sync(0xffffffffu, rend, nr - 1);
        uint32_t u[kMv3Pl];
#pragma unroll
        for (int j = 0; j < kMv3Pl; ++j) {
            const int64_t e = e0 + j * 32 + lane;
            u[j] = e < e1 ? ld_stream_u32(a.col + e) : 0u;
        }
        // gathers through L1 into registers (LDG: ~1 line/clk/SM on B200, 2.6x
        // the rate of 8-byte cp.async), then to the warp's shared slice
        {
            double v[kMv3Pl];
#pragma unroll
            for (int j = 0; j < kMv3Pl; ++j) v[j] = (e0 + j * 32 + lane < e1) ? __ldg(a.share_in + u[j]) : 0.0;
#pragma unroll
            for (int j = 0; j < kMv3Pl; ++j) sv[j * 32 + lane] = v[j];
        }
        int64_t rbeg = __shfl_up_sync(0xffffffffu, rend, 1);
        if (lane == 0) rbeg = e0;
        const int lo = (int)(rbeg - e0), hi = (int)(rend - e0);
        __syncwarp();
        double y = 0.0;
        if (has && hi - lo <= kMvShortRow)
            for (int k = lo; k < hi; ++k) y = dadd(y, sv[k]);  // ascending sources
        unsigned longm = __ballot_sync(0xffffffffu, has && hi - lo > kMvShortRow);
        while (longm) {
            const int j = __ffs(longm) - 1;
            longm &= longm - 1;
            const int jl = __shfl_sync(0xffffffffu, lo, j), jh = __shfl_sync(0xffffffffu, hi, j);
            double s = 0.0;
            for (int k = jl + lane; k < jh; k += 32) s = dadd(s, sv[k]);
            s = warp_sum(s);
            if (lane == j) y = s;
        }
        __syncwarp();  // sv is reused by the next block
        if (has) {
            y = mv3_row(a, st, r0 + lane, y, d, acc_v);
            fx_add(f0, f1, y);
            if (want_dm && d == 0 && y != 0.0) fx_add(f2, f3, y);
        }
    }
    // exact integer totals: lane -> CTA (shared) -> grid; last CTA advances state
    __syncthreads();
    if (f0 | f1) fx_atomic_add(&s_fx[0], &s_fx[1], f0, f1);
    if (f2 | f3) fx_atomic_add(&s_fx[2], &s_fx[3], f2, f3);
    __syncthreads();
    if (tid == 0) {
        if (s_fx[0] | s_fx[1]) fx_atomic_add(&M.fx[0], &M.fx[1], s_fx[0], s_fx[1]);
        if (s_fx[2] | s_fx[3]) fx_atomic_add(&M.fx[2], &M.fx[3], s_fx[2], s_fx[3]);
        __threadfence();
        s_ticket = atomicAdd(a.done_cnt, 1u);
    }
    __syncthreads();
    if (s_ticket != gridDim.x - 1 || tid != 0) return;
    __threadfence();
    ColState s = st;
    const double res = fx_decode(atomicAdd(&M.fx[0], 0ull), atomicAdd(&M.fx[1], 0ull));
    const double dmt = fx_decode(atomicAdd(&M.fx[2], 0ull), atomicAdd(&M.fx[3], 0ull));
    s.residual = res;
    s.iters = a.step;
    s.converged = res < a.eps;
    s.active = !s.converged && (a.terminal < 0 || (int64_t)a.step < a.terminal);
    s.has_spread = (a.policy == kUniform && dmt != 0.0);
    s.spread = s.has_spread ? ddiv(dmul(a.keep, dmt), (double)a.n) : 0.0;
    a.state_out[0] = s;
    M.fx[0] = M.fx[1] = M.fx[2] = M.fx[3] = 0ull;
    *a.done_cnt = 0;
}

}  // namespace tpa
