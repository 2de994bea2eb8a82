// EXPERIMENT, not part of libtpa_gpu.so (profiles/r02_experiments.md, "Pipelined K2").
// A drop-in replacement for csrc/cpi_spmv2.cuh in which one CTA takes up to 16
// consecutive tiles and software-pipelines them; it needs MvArgs::per_cta set by
// the launcher (mv_items_per_cta) and grid = ceil(n_items / per_cta).  Bitwise
// K2, measured slower (96 registers, 5 CTAs/SM).
//
// cpi_spmv2.cuh -- K2 v2: the B = 1 sweep (PageRank / single-vector CPI).
//
// Same tiles and the same per-row arithmetic order as K2 v1 (cpi_kernels.cuh:
// rows <= 32 nnz sequential per thread, longer rows a fixed warp tree, rows
// above a tile one CTA tree), restructured for memory-level parallelism:
//   * the tile's nnz range travels with the work item, so the index loads,
//     the row_ptr loads and the per-row out-degree / accumulator loads are all
//     issued at once (one round trip), then the gathers (a second one);
//   * the L1 residual and dangling mass are reduced per tile in a fixed tree
//     and added across tiles as exact 128-bit fixed-point integers
//     (order-free): the totals depend only on the tiling, which a row
//     partition cut at tile starts (tpa_part.cuh) leaves unchanged, so a
//     partitioned run reproduces the one-GPU residuals bit for bit.  The last
//     CTA advances the state, or, for a partition, publishes its totals as
//     carry-free limbs for an all-reduce (fx_to_limbs) and leaves the state
//     to k_part_finalize.
#pragma once

#include "cpi_spmm.cuh"

namespace tpa {

// In-process partition groups (tpa_part.cuh): the sweep stores each share
// (and its limbs) into every other partition's buffer too -- peer stores over
// NVLink that overlap the sweep instead of a copy step after it.
constexpr int kMaxPeerOut = 15;
struct PeerOut {
    double* p[kMaxPeerOut];  // the same span of each peer's share_out buffer
    uint32_t n;
};

// values, row pointers, row sums.
// The size matters: 2 KB more per CTA cost 4% at C2 and 22% at C4 (less L1).
// row offsets inside the tile (int32, relative to the tile's first nonzero)
template <int kRows>
__host__ __device__ constexpr size_t mv_rp_bytes() { return ((kRows + 1) * 4 + 7) / 8 * 8; }
template <int kNnz, int kRows>
__host__ __device__ constexpr size_t mv_dyn_smem() {
    return (size_t)kNnz * 8 + mv_rp_bytes<kRows>() + (size_t)kRows * 8;
}
constexpr size_t kMvDynSmem = mv_dyn_smem<kMvTileNnz, kMvTileRows>();

// SpMV tile shape {threads per CTA, nnz per tile, rows per tile}, chosen by the
// GLOBAL node count (a row partition tiles its rows exactly as the whole graph
// does; partition.py mirrors this).  Measured per PageRank sweep (ms):
//                         C2 (8 MB shares)  C4 (134 MB)  C5 (2.1 GB)
//   S {128, 1024, 256}        0.0952          2.920        47.9
//   L {256, 2048, 256}        0.110           3.005        45.9
//   W {256, 2048, 512}        0.1062          3.135        47.9   (round-1 default before)
// Small CTAs finish their tile (and free its slot) sooner: fewer warps wait at
// each barrier behind the tile's longest row.  Once the share vector is far
// beyond the L2 the larger tile amortises its DRAM round trips better.
struct MvShape {
    int thr, nnz, rows;
};
// (partition.py mirrors both shapes and the rule)
constexpr MvShape kMvShapeS{128, 1024, 256}, kMvShapeL{256, 2048, 256};
inline MvShape mv_shape(uint64_t n_global) {
    return n_global * 8 > (512ull << 20) ? kMvShapeL : kMvShapeS;
}

struct MvArgs {
    StepArgs s;
    const longlong2* __restrict__ item_nnz;  // [n_items] {nnz begin, nnz end}
    unsigned long long* fx;                  // [4]: l1 hi/lo, dm hi/lo; zero between launches
    unsigned long long* limbs;               // partition mode: [6] out (see fx_to_limbs), else null
    PeerOut peers;                           // partition group: replicas of share_out (n = 0: none)
    uint32_t limb_off;                       // limbs - share_out, in doubles (peer copies of the limbs)
    uint32_t per_cta;                        // consecutive tiles per CTA (<= kMvMaxItemsPerCta)
};

// ColState after sweep `step` from the global residual / dangling mass
// (cpi.cpp:73-80; Uniform spread graph.cpp:265-268).
__device__ __forceinline__ ColState advance_state(ColState s, double res, double dmt, const StepArgs& a) {
    s.residual = res;
    s.iters = a.step;
    s.converged = res < a.eps;
    s.active = !s.converged && (a.terminal < 0 || (int64_t)a.step < a.terminal);
    s.has_spread = (a.policy == kUniform && dmt != 0.0);
    s.spread = s.has_spread ? ddiv(dmul(a.keep, dmt), (double)a.n) : 0.0;
    return s;
}

// The residual / dangling mass are per-tile fixed-tree double sums, added
// across tiles in exact fixed point (the totals depend on the tiling only; a
// row partition cuts at tile starts, tpa_part.cuh).
// kRanked: the ranked share layout (a.rank, tpa_gpu.cu): each share is stored
// at its node's rank slot; gathers already read col_rank.

constexpr int kMvFxSlots = 1;  // [4 x slots] fixed-point accumulators (w.fx, B = 1)
constexpr int kMvMaxItemsPerCta = 16;

// Tiles per CTA: enough CTAs for ~64 per SM, at most kMvMaxItemsPerCta tiles each.
inline uint32_t mv_items_per_cta(uint32_t n_items, int num_sms) {
    const uint32_t t = n_items / (uint32_t)(num_sms * 64);
    return t < 1u ? 1u : (t > (uint32_t)kMvMaxItemsPerCta ? (uint32_t)kMvMaxItemsPerCta : t);
}

// One CTA takes M.per_cta consecutive tiles and software-pipelines them: the
// gathers of tile i are in flight while the CTA sums and stores tile i-1 from
// shared memory, and tile i+1's column indices are already loading, so a warp
// waiting at a barrier or summing still has its share of the gather queue
// filled (K2 before: 13 of 36 stall cycles at barriers with nothing in
// flight).  A long row (one item) streams its indices one chunk ahead of its
// gathers.  Tiling, thread -> nonzero / row mapping, per-row order and the
// per-tile residual tree are unchanged: bitwise the unpipelined sweep.
// Consecutive sweeps are chained by programmatic dependent launch: the static
// tiling and the first tile's indices are read before griddepcontrol.wait.
#ifndef TPA_MV_MINB
#define TPA_MV_MINB 1
#endif
template <bool kRanked, int kThr, int kNnz, int kRows>
__global__ void __launch_bounds__(kThr, TPA_MV_MINB * 128 / kThr) k_step_spmv2(MvArgs M) {
    const StepArgs& a = M.s;
    constexpr int kW = kThr / 32;
    constexpr int U = kNnz / kThr;     // nonzeros per thread of a tile
    constexpr int RPT = kRows / kThr;  // rows per thread of a tile
    constexpr int UL = 8;              // long rows: gathers in flight per thread
    // the tile's staging in dynamic shared memory (kMvDynSmem bytes): values,
    // row pointers, row sums
    extern __shared__ __align__(16) unsigned char s_mv[];
    double* s_vals = reinterpret_cast<double*>(s_mv);
    int* s_rp = reinterpret_cast<int*>(s_vals + kNnz);  // row starts - nb
    double* s_y = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(s_rp) + mv_rp_bytes<kRows>());
    __shared__ double s_l1[kW], s_dm[kW], s_row[2][kW];
    __shared__ uint2 s_item[kMvMaxItemsPerCta];
    __shared__ longlong2 s_nnz[kMvMaxItemsPerCta];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t per = M.per_cta;
    const uint32_t i0 = blockIdx.x * per;
    const uint32_t cnt = min(per, a.n_items - i0);
    // programmatic dependent launch: the next sweep's CTAs may start once
    // every CTA of this one has; they wait below for this grid to finish
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // static: the CTA's items and the first tile's indices
    if (tid < (int)cnt) {
        s_item[tid] = a.items[i0 + tid];
        s_nnz[tid] = M.item_nnz[i0 + tid];
    }
    __syncthreads();
    auto is_long_item = [&](uint32_t k) { return (s_item[k].y & kLongFlag) != 0; };
    uint32_t un[U];  // the next tile's column indices
    auto prefetch_idx = [&](uint32_t k) {
        if (k >= cnt || is_long_item(k)) return;
        const int64_t nb = s_nnz[k].x;
        const int nnz = (int)(s_nnz[k].y - nb);
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int q = tid + j * kThr;
            un[j] = q < nnz ? ld_col(a.col + nb + q) : 0u;
        }
    };
    prefetch_idx(0);
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous sweep's shares, acc, state
    const ColState st = a.state_in[0];

    if (!st.active) {
        // column stopped earlier: only a pending combine remains (tpa.cpp:73)
        if (a.out)
            for (uint32_t k = 0; k < cnt; ++k) {
                const uint32_t rb = s_item[k].x, re = s_item[k].y & ~kLongFlag;
                for (uint32_t v = rb + tid; v < re; v += kThr) combine_only(a, v, 0, 1, v);
            }
        if (blockIdx.x == 0 && tid == 0) {
            a.state_out[0] = st;
            if (M.limbs)
                for (int k = 0; k < 6; ++k) M.limbs[k] = 0ull;
        }
        return;
    }
    const bool want_dm = a.policy == kUniform;
    unsigned long long l1h = 0, l1l = 0, dmh = 0, dml = 0;  // the CTA's exact totals (thread 0)

    // the pending tile: staged in shared memory, summed while the next one's gathers fly
    bool pend = false;
    uint32_t p_rb = 0, p_nrows = 0;
    uint32_t p_dg[RPT], p_so[RPT];
    double p_ac[RPT];
    // rows summed and stored; the tile's residual partials left in s_l1 / s_dm
    auto finish_pending = [&]() {
        const uint32_t nrows = p_nrows, rb = p_rb;
        // short rows: one thread, ascending-source sequential sum (reference order)
        for (uint32_t r = tid; r < nrows; r += kThr) {
            const int lo = s_rp[r], hi = s_rp[r + 1];
            if (hi - lo <= kMvShortRow) {
                double s = 0.0;
                for (int k = lo; k < hi; ++k) s = dadd(s, s_vals[k]);
                s_y[r] = s;
            }
        }
        // longer rows of the tile: one warp each, lane-strided + butterfly
        for (uint32_t base = warp * 32; base < nrows; base += kThr) {
            const uint32_t r = base + lane;
            const int len = r < nrows ? (s_rp[r + 1] - s_rp[r]) : 0;
            unsigned mask = __ballot_sync(0xffffffffu, len > kMvShortRow);
            while (mask) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                const uint32_t rr = base + j;
                const int lo = s_rp[rr], hi = s_rp[rr + 1];
                double s = 0.0;
                for (int k = lo + lane; k < hi; k += 32) s = dadd(s, s_vals[k]);
                s = warp_sum(s);
                if (lane == 0) s_y[rr] = s;
            }
        }
        // a thread's rows r = tid + q * kThr were summed by itself (short) or by
        // its own warp (r / 32 % kW == warp): no CTA barrier needed before reading s_y
        __syncwarp();
        double my_l1 = 0.0, my_dm = 0.0;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const uint32_t r = tid + q * kThr;
            if (r >= nrows) continue;
            const uint32_t vtx = rb + r;
            double y = s_y[r];
            if (st.has_spread) y = dadd(y, st.spread);  // graph.cpp:265-268
            if (a.y_out) a.y_out[vtx] = y;
            if (a.acc) {
                const double f = dadd(p_ac[q], y);  // cpi.cpp:50
                if (a.out) {
                    a.out[vtx] = a.stranger ? dadd(dmul(a.scale, f), a.stranger[vtx]) : dmul(f, a.scale);
                } else {
                    a.acc[vtx] = f;
                }
            }
            if (a.share_out) {
                const double sv = p_dg[q] ? ddiv(dmul(a.keep, y), (double)p_dg[q]) : 0.0;  // graph.cpp:222
                a.share_out[p_so[q]] = sv;
                for (uint32_t k = 0; k < M.peers.n; ++k) M.peers.p[k][vtx] = sv;
            }
            my_l1 = dadd(my_l1, fabs(y));
            if (want_dm && p_dg[q] == 0) my_dm = dadd(my_dm, y);
        }
        my_l1 = warp_sum(my_l1);
        if (want_dm) my_dm = warp_sum(my_dm);
        if (lane == 0) {
            s_l1[warp] = my_l1;
            s_dm[warp] = my_dm;
        }
    };
    // thread 0, after a barrier behind finish_pending: the tile's partials in
    // K2's fixed order into the exact totals
    auto take_partials = [&]() {
        double tl1 = s_l1[0], tdm = s_dm[0];
#pragma unroll
        for (int k = 1; k < kW; ++k) {
            tl1 = dadd(tl1, s_l1[k]);
            tdm = dadd(tdm, s_dm[k]);
        }
        if (tl1 != 0.0) fx_add(l1h, l1l, tl1);
        if (want_dm && tdm != 0.0) fx_add(dmh, dml, tdm);
    };

    for (uint32_t k = 0; k < cnt; ++k) {
        const uint2 it = s_item[k];
        const uint32_t rb = it.x, re = it.y & ~kLongFlag;
        const int64_t nb = s_nnz[k].x, ne = s_nnz[k].y;
        if (!(it.y & kLongFlag)) {
            const uint32_t nrows = re - rb;
            const int nnz = (int)(ne - nb);
            // ---- this tile's gathers (indices prefetched), rows' inputs ----
            double v[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int q = tid + j * kThr;
                v[j] = q < nnz ? __ldg(a.share_in + un[j]) : 0.0;
            }
            int rp[RPT];
            uint32_t dg[RPT], so[RPT];
            double ac[RPT];
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const uint32_t r = tid + q * kThr;
                rp[q] = r < nrows ? (int)(__ldg(a.row_ptr + rb + r) - nb) : 0;
                dg[q] = r < nrows ? __ldg(a.deg + rb + r) : 0u;
                if constexpr (kRanked) so[q] = r < nrows ? __ldg(a.rank + rb + r) : 0u;  // share slot
                else so[q] = rb + r;
                ac[q] = (r < nrows && a.acc) ? a.acc[rb + r] : 0.0;
            }
            prefetch_idx(k + 1);  // the next tile's indices (un is free: the gathers are issued)
            // ---- the previous tile, while those are in flight ----
            if (pend) finish_pending();
            __syncthreads();
            if (pend && tid == 0) take_partials();
            // ---- stage this tile ----
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int q = tid + j * kThr;
                if (q < nnz) s_vals[q] = v[j];
            }
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const uint32_t r = tid + q * kThr;
                if (r < nrows) s_rp[r] = rp[q];
                p_dg[q] = dg[q];
                p_so[q] = so[q];
                p_ac[q] = ac[q];
            }
            if (tid == 0) s_rp[nrows] = nnz;
            p_rb = rb;
            p_nrows = nrows;
            pend = true;
            __syncthreads();
        } else {
            // one long row: every thread sums a fixed strided subset (indices one
            // chunk ahead of the gathers), then a fixed tree
            prefetch_idx(k + 1);
            double s = 0.0;
            int64_t e = nb + tid;
            uint32_t u[UL];
            if (e + (UL - 1) * kThr < ne) {
#pragma unroll
                for (int j = 0; j < UL; ++j) u[j] = ld_col(a.col + e + j * kThr);
            }
            if (pend) finish_pending();  // the staged tile, under the first chunk's index loads
            for (; e + (UL - 1) * kThr < ne; e += UL * kThr) {
                double v[UL];
#pragma unroll
                for (int j = 0; j < UL; ++j) v[j] = __ldg(a.share_in + u[j]);
                if (e + UL * kThr + (UL - 1) * kThr < ne) {
#pragma unroll
                    for (int j = 0; j < UL; ++j) u[j] = ld_col(a.col + e + UL * kThr + j * kThr);
                }
#pragma unroll
                for (int j = 0; j < UL; ++j) s = dadd(s, v[j]);
            }
            for (; e < ne; e += kThr) s = dadd(s, __ldg(a.share_in + ld_col(a.col + e)));
            s = warp_sum(s);
            if (lane == 0) s_row[k & 1][warp] = s;
            __syncthreads();
            if (tid == 0) {
                if (pend) take_partials();
                double y = s_row[k & 1][0];
#pragma unroll
                for (int w = 1; w < kW; ++w) y = dadd(y, s_row[k & 1][w]);
                const uint32_t d = __ldg(a.deg + rb);
                if (st.has_spread) y = dadd(y, st.spread);  // graph.cpp:265-268
                if (a.y_out) a.y_out[rb] = y;
                if (a.acc) {
                    const double f = dadd(a.acc[rb], y);  // cpi.cpp:50
                    if (a.out) a.out[rb] = a.stranger ? dadd(dmul(a.scale, f), a.stranger[rb]) : dmul(f, a.scale);
                    else a.acc[rb] = f;
                }
                if (a.share_out) {
                    const double sv = d ? ddiv(dmul(a.keep, y), (double)d) : 0.0;  // graph.cpp:222
                    a.share_out[kRanked ? a.rank[rb] : rb] = sv;
                    for (uint32_t q = 0; q < M.peers.n; ++q) M.peers.p[q][rb] = sv;
                }
                // the item's partial: K2's tree over |y| in thread 0 and zeros elsewhere is |y|
                const double tl1 = fabs(y);
                if (tl1 != 0.0) fx_add(l1h, l1l, tl1);
                if (want_dm && d == 0 && y != 0.0) fx_add(dmh, dml, dadd(0.0, y));
            }
            pend = false;
        }
    }
    if (pend) {
        finish_pending();
        __syncthreads();
        if (tid == 0) take_partials();
    }
    // only thread 0 takes the ticket: the rest of the CTA leaves now instead
    // of waiting out the fence + atomic round trip
    if (tid != 0) return;
    if (l1h | l1l) fx_atomic_add(&M.fx[0], &M.fx[1], l1h, l1l);
    if (dmh | dml) fx_atomic_add(&M.fx[2], &M.fx[3], dmh, dml);
    __threadfence();
    if (atomicAdd(a.done_cnt, 1u) != gridDim.x - 1) return;
    __threadfence();
    // exact 128-bit sums (order-free)
    const unsigned long long h0 = atomicAdd(&M.fx[0], 0ull), l0 = atomicAdd(&M.fx[1], 0ull);
    const unsigned long long h1 = atomicAdd(&M.fx[2], 0ull), l1 = atomicAdd(&M.fx[3], 0ull);
    if (M.limbs) {
        // a partition's totals: all-reduced, then k_part_finalize advances the state
        fx_to_limbs(h0, l0, M.limbs);
        fx_to_limbs(h1, l1, M.limbs + 3);
        for (uint32_t k = 0; k < M.peers.n; ++k) {
            auto* pl = reinterpret_cast<unsigned long long*>(M.peers.p[k] + M.limb_off);
            fx_to_limbs(h0, l0, pl);
            fx_to_limbs(h1, l1, pl + 3);
        }
    } else {
        // last CTA: cpi.cpp:73-80
        a.state_out[0] = advance_state(st, fx_decode(h0, l0), fx_decode(h1, l1), a);
    }
    for (int k = 0; k < 4 * kMvFxSlots; ++k) M.fx[k] = 0ull;
    *a.done_cnt = 0;
}

// Partition mode, after the all-reduce of every partition's limbs: the same
// state on every GPU.  init: x⁽⁰⁾'s state (k_init_finish's role).
__global__ void k_part_finalize(const unsigned long long* __restrict__ limbs, StepArgs a, int init, int active0) {
    unsigned long long h0, l0, h1, l1;
    limbs_to_fx(limbs, h0, l0);
    limbs_to_fx(limbs + 3, h1, l1);
    const double res = fx_decode(h0, l0), dmt = fx_decode(h1, l1);
    if (init) {
        ColState s;
        s.residual = res;
        s.iters = 0;
        s.active = active0;
        s.converged = 0;
        s.has_spread = a.policy == kUniform && dmt != 0.0;
        s.spread = s.has_spread ? ddiv(dmul(a.keep, dmt), (double)a.n) : 0.0;
        a.state_out[0] = s;
        return;
    }
    const ColState st = a.state_in[0];
    a.state_out[0] = st.active ? advance_state(st, res, dmt, a) : st;
}

}  // namespace tpa
