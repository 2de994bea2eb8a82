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
//     to k_part_finalize;
//   * on large grids a CTA takes several tiles (kMulti): the per-tile partials
//     meet in the CTA's exact totals in shared memory, and the total atomics,
//     the fence and the ticket are paid once per CTA.
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
    uint32_t per_cta;                        // items per CTA, gridDim.x apart
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

// Items per CTA (gridDim.x apart): up to kMvItemsPerCta while the grid keeps
// >= 64 CTAs per SM.  Measured per C4 PageRank sweep (ms; 408 k items, one
// ticket + one set of total atomics per CTA instead of per tile):
//   1: 2.853   3: 2.577   4: 2.538   6: 2.504   8: 2.494   10: 2.489
// C3 (65 k items): 1: 0.403   3: 0.362   6: 0.351   8: 0.353;  C2 (16 k items):
// one item per CTA stays best (0.096 ms; 3: 0.099).
constexpr uint32_t kMvItemsPerCta = 8;
inline uint32_t mv_items_per_cta(uint32_t n_items, int num_sms) {
    const uint32_t t = n_items / (uint32_t)(num_sms * 64);
    return t < 1u ? 1u : (t > kMvItemsPerCta ? kMvItemsPerCta : t);
}
constexpr int kMvFxSlots = 1;  // [4 x slots] fixed-point accumulators (w.fx, B = 1)
// Consecutive sweeps are chained by programmatic dependent launch (C1 65.4 ->
// 68.3 GTEPS: launch-bound sweeps); only thread 0 of a finished CTA takes the
// ticket (0.1102 -> 0.1097 ms per C2 sweep).  The default register
// allocation (no minimum-blocks bound) measured best in both forms.
// kMulti: the CTA takes M.per_cta items (48 registers, 56 with the index
// look-ahead of the 128-thread shape); otherwise exactly one (40 registers,
// 12 CTAs per SM: the better form when the grid is small).
template <bool kRanked, int kThr, int kNnz, int kRows, bool kMulti>
__global__ void __launch_bounds__(kThr) k_step_spmv2(MvArgs M) {
    const StepArgs& a = M.s;
    // the tile's staging in dynamic shared memory (kMvDynSmem bytes): values,
    // row pointers, row sums
    extern __shared__ __align__(16) unsigned char s_mv[];
    double* s_vals = reinterpret_cast<double*>(s_mv);
    int* s_rp = reinterpret_cast<int*>(s_vals + kNnz);  // row starts - nb
    double* s_y = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(s_rp) + mv_rp_bytes<kRows>());
    __shared__ double s_red[kThr / 32], s_l1[kThr / 32], s_dm[kThr / 32];
    __shared__ unsigned long long s_fx[4];  // the CTA's exact totals (thread 0 only)

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // a CTA takes M.per_cta items, gridDim.x apart (the longest rows, first in
    // the item list, stay spread over the grid): one ticket and one set of
    // total atomics per CTA instead of per tile
    // programmatic dependent launch: the next sweep's CTAs may start once
    // every CTA of this one has; they wait below for this grid to finish
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    uint2 it = a.items[blockIdx.x];  // the tiling is static: read before the wait
    longlong2 nr = M.item_nnz[blockIdx.x];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous sweep's shares, acc, state
    const ColState st = a.state_in[0];

    if (!st.active) {
        // column stopped earlier: only a pending combine remains (tpa.cpp:73)
        if (a.out)
            for (uint32_t item = blockIdx.x; item < a.n_items; item += gridDim.x) {
                const uint2 ii = a.items[item];
                for (uint32_t v = ii.x + tid; v < (ii.y & ~kLongFlag); v += kThr) combine_only(a, v, 0, 1, v);
            }
        if (blockIdx.x == 0 && tid == 0) {
            a.state_out[0] = st;
            if (M.limbs)
                for (int k = 0; k < 6; ++k) M.limbs[k] = 0ull;
        }
        return;
    }
    if (kMulti && tid == 0) s_fx[0] = s_fx[1] = s_fx[2] = s_fx[3] = 0ull;
  uint32_t item = blockIdx.x, t = 0;
  // kMulti: a tile's column indices are requested before the barrier that ends
  // the previous tile, so that round trip overlaps the wait for its slowest warp
  // (the 128-thread shape only: C4 2.488 -> 2.449 ms; the 256-thread shape of C5
  // loses a resident CTA to the longer-lived registers, 33.5 -> 35.1 ms)
  constexpr bool kAhead = kMulti && kThr == 128;
  uint32_t u[kNnz / kThr];
  auto prefetch_idx = [&](const uint2& ii, const longlong2& rr) {
      if (ii.y & kLongFlag) return;  // a long row streams its own indices
      const int nnz = (int)(rr.y - rr.x);
#pragma unroll
      for (int j = 0; j < kNnz / kThr; ++j) {
          const int k = tid + j * kThr;
          u[j] = k < nnz ? ld_col(a.col + rr.x + k) : 0u;
      }
  };
  if constexpr (kAhead) prefetch_idx(it, nr);
  do {
    if (kMulti && !kAhead && t) {
        it = a.items[item];
        nr = M.item_nnz[item];
    }
    const uint32_t rb = it.x, re = it.y & ~kLongFlag;
    const bool is_long = (it.y & kLongFlag) != 0;
    const int64_t nb = nr.x, ne = nr.y;
    const bool want_dm = a.policy == kUniform;
    double my_l1 = 0.0, my_dm = 0.0;
    auto add_row = [&](double y, bool dangling) {
        my_l1 = dadd(my_l1, fabs(y));
        if (want_dm && dangling) my_dm = dadd(my_dm, y);
    };

    if (!is_long) {
        const uint32_t nrows = re - rb;
        const int nnz = (int)(ne - nb);
        constexpr int U = kNnz / kThr;
        constexpr int RPT = kRows / kThr;  // rows per thread
        // ---- round trip 1: indices, row pointers, degrees, accumulators ----
        if constexpr (!kAhead) prefetch_idx(it, nr);
        for (uint32_t r = tid; r <= nrows; r += kThr) s_rp[r] = (int)(__ldg(a.row_ptr + rb + r) - nb);
        uint32_t dg[RPT], so[RPT];
        double ac[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const uint32_t r = tid + q * kThr;
            dg[q] = r < nrows ? __ldg(a.deg + rb + r) : 0u;
            if constexpr (kRanked) so[q] = r < nrows ? __ldg(a.rank + rb + r) : 0u;  // share slot
            else so[q] = rb + r;
            ac[q] = (r < nrows && a.acc) ? a.acc[rb + r] : 0.0;
        }
        // ---- round trip 2: gathers ----
        double v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int k = tid + j * kThr;
            v[j] = k < nnz ? __ldg(a.share_in + u[j]) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int k = tid + j * kThr;
            if (k < nnz) s_vals[k] = v[j];
        }
        __syncthreads();
        // short rows: one thread, ascending-source sequential sum (reference order)
        for (uint32_t r = tid; r < nrows; r += kThr) {
            const int lo = s_rp[r], hi = s_rp[r + 1];
            if (hi - lo <= kMvShortRow) {
                // four loads ahead of their (still strictly sequential) adds
                double s = 0.0;
                int k = lo;
                for (; k + 4 <= hi; k += 4) {
                    const double a0 = s_vals[k], a1 = s_vals[k + 1], a2 = s_vals[k + 2], a3 = s_vals[k + 3];
                    s = dadd(dadd(dadd(dadd(s, a0), a1), a2), a3);
                }
                for (; k < hi; ++k) s = dadd(s, s_vals[k]);
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
        // a thread's rows r = tid + q * kThr were summed by itself (short rows)
        // or by its own warp (r / 32 % (kThr / 32) == warp): no CTA barrier
        __syncwarp();
        // epilogue with the prefetched degree / accumulator of each row
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const uint32_t r = tid + q * kThr;
            if (r >= nrows) continue;
            const uint32_t vtx = rb + r;
            double y = s_y[r];
            if (st.has_spread) y = dadd(y, st.spread);  // graph.cpp:265-268
            if (a.y_out) a.y_out[vtx] = y;
            if (a.acc) {
                const double f = dadd(ac[q], y);  // cpi.cpp:50
                if (a.out) {
                    a.out[vtx] = a.stranger ? dadd(dmul(a.scale, f), a.stranger[vtx]) : dmul(f, a.scale);
                } else {
                    a.acc[vtx] = f;
                }
            }
            if (a.share_out) {
                const double sv = dg[q] ? ddiv(dmul(a.keep, y), (double)dg[q]) : 0.0;
                a.share_out[so[q]] = sv;
                for (uint32_t k = 0; k < M.peers.n; ++k) M.peers.p[k][vtx] = sv;
            }
            add_row(y, dg[q] == 0);
        }
    } else {
        // one long row: every thread sums a fixed strided subset, then a fixed tree
        double s = 0.0;
        constexpr int U = 8;
        int64_t e = nb + tid;
        for (; e + (U - 1) * kThr < ne; e += U * kThr) {
            uint32_t u[U];
            double v[U];
#pragma unroll
            for (int j = 0; j < U; ++j) u[j] = ld_col(a.col + e + j * kThr);
#pragma unroll
            for (int j = 0; j < U; ++j) v[j] = __ldg(a.share_in + u[j]);
#pragma unroll
            for (int j = 0; j < U; ++j) s = dadd(s, v[j]);
        }
        for (; e < ne; e += kThr) s = dadd(s, __ldg(a.share_in + ld_col(a.col + e)));
        s = warp_sum(s);
        if (lane == 0) s_red[warp] = s;
        __syncthreads();
        if (tid == 0) {
            const uint32_t d = __ldg(a.deg + rb);
            double y = s_red[0];  // the fixed tree: warp butterflies, then the warps in order
#pragma unroll
            for (int k = 1; k < kThr / 32; ++k) y = dadd(y, s_red[k]);
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
                for (uint32_t k = 0; k < M.peers.n; ++k) M.peers.p[k][rb] = sv;
            }
            add_row(y, d == 0);
        }
    }
    {
        // tile partials (fixed tree: warp butterflies, then the warps in order)
        // -> exact fixed-point totals across tiles; one barrier, thread 0 adds
        // (a long row's partials are thread 0's alone: the tree adds zeros)
        my_l1 = warp_sum(my_l1);
        if (want_dm) my_dm = warp_sum(my_dm);
        if (lane == 0) {
            s_l1[warp] = my_l1;
            s_dm[warp] = my_dm;
        }
        if constexpr (kAhead) {
            if (t + 1 < M.per_cta && item + gridDim.x < a.n_items) {
                it = a.items[item + gridDim.x];
                nr = M.item_nnz[item + gridDim.x];
                prefetch_idx(it, nr);
            }
        }
        __syncthreads();
        if (tid == 0) {
            double tl1 = s_l1[0], tdm = s_dm[0];
#pragma unroll
            for (int k = 1; k < kThr / 32; ++k) {
                tl1 = dadd(tl1, s_l1[k]);
                tdm = dadd(tdm, s_dm[k]);
            }
            if constexpr (kMulti) {
                if (tl1 != 0.0) fx_add(s_fx[0], s_fx[1], tl1);
                if (want_dm && tdm != 0.0) fx_add(s_fx[2], s_fx[3], tdm);
            } else {
                unsigned long long h = 0, l = 0;
                if (tl1 != 0.0) {
                    fx_add(h, l, tl1);
                    fx_atomic_add(&M.fx[0], &M.fx[1], h, l);
                }
                if (want_dm && tdm != 0.0) {
                    h = l = 0;
                    fx_add(h, l, tdm);
                    fx_atomic_add(&M.fx[2], &M.fx[3], h, l);
                }
            }
        }
    }
    if constexpr (!kMulti) break;
    ++t;
    item += gridDim.x;
  } while (t < M.per_cta && item < a.n_items);  // the CTA's items
    // only thread 0 takes the ticket: the rest of the CTA leaves now instead
    // of waiting out the fence + atomic round trip
    if (tid != 0) return;
    if constexpr (kMulti) {
        if (s_fx[0] | s_fx[1]) fx_atomic_add(&M.fx[0], &M.fx[1], s_fx[0], s_fx[1]);
        if (s_fx[2] | s_fx[3]) fx_atomic_add(&M.fx[2], &M.fx[3], s_fx[2], s_fx[3]);
    }
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
