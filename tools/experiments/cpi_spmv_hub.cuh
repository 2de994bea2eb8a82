// EXPERIMENT, not part of libtpa_gpu.so (profiles/r02_experiments.md, "K2h").
// Include after csrc/cpi_spmv2.cuh; launch one CTA per SM with
// mvh_dyn_smem<...>() bytes of dynamic shared memory over the ranked layout.
// Bitwise K2, measured slower or equal at every hub size.
//
// cpi_spmv_hub.cuh -- K2h: the B = 1 sweep over the ranked share layout with
// the hub slice of the share vector staged in shared memory.
//
// K2 (cpi_spmv2.cuh) is bound by the SM's L1 -> L2 request path: every random
// 8-byte gather of a share is one sector request (0.7 per clock per SM,
// profiles/r02_experiments.md).  In the ranked layout slot k of the share
// vector belongs to the node with the k-th largest out-degree, so the first
// kHub slots are the sources of a third (R-MAT 24) to two thirds (R-MAT 20) of
// all nonzeros.  One persistent CTA per SM copies those kHub shares into
// shared memory once per sweep; its kGroups groups of kThr threads then claim
// K2's tiles from one counter and gather shares below kHub from shared memory
// and only the rest through L2.
//
// The tiles, the thread -> row / nonzero mapping inside a tile, every row's
// summation order and the per-tile residual tree are K2's, and tile totals
// meet in exact fixed point, so the sweep is bitwise K2's whichever group
// takes which tile (graph.cpp:211-270, cpi.cpp:43-83 semantics unchanged).
#pragma once

#include "cpi_spmv2.cuh"

namespace tpa {

// K2h pays a hub copy per CTA per sweep: used from this many tiles / edges up
// (below, K2 over the unranked layout)
#ifndef TPA_MVH_MIN_ITEMS
#define TPA_MVH_MIN_ITEMS 4096
#endif
constexpr uint32_t kMvHubMinItems = TPA_MVH_MIN_ITEMS;
constexpr uint64_t kMvHubMinEdges = 4ull << 20;

#ifndef TPA_MVH_GATHER_NA
#define TPA_MVH_GATHER_NA 0
#endif
__device__ __forceinline__ double mvh_gather(const double* p) {
#if TPA_MVH_GATHER_NA
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
#else
    return __ldg(p);
#endif
}

template <int kThr>
__device__ __forceinline__ void grp_bar(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(kThr) : "memory");
}

// per-group staging: values, row offsets, row sums, reduction slots, claim slot
template <int kThr, int kNnz, int kRows>
__host__ __device__ constexpr size_t mvh_group_bytes() {
    return mv_dyn_smem<kNnz, kRows>() + (size_t)3 * (kThr / 32) * 8 + 16;
}
template <int kThr, int kNnz, int kRows, int kGroups, int kHub>
__host__ __device__ constexpr size_t mvh_dyn_smem() {
    return (size_t)kHub * 8 + (size_t)kGroups * mvh_group_bytes<kThr, kNnz, kRows>();
}

struct MvHubArgs {
    MvArgs m;
    uint32_t* next_item;  // tile counter, zero between launches
    uint32_t chunk;       // tiles per claim
    uint32_t hub;         // shares staged: min(kHub, n)
};

template <int kThr, int kNnz, int kRows, int kGroups, int kHub>
__global__ void __launch_bounds__(kThr* kGroups, 1) k_step_spmv_hub(MvHubArgs H) {
    const MvArgs& M = H.m;
    const StepArgs& a = M.s;
    constexpr int kW = kThr / 32;
    extern __shared__ __align__(16) unsigned char s_all[];
    double* s_hub = reinterpret_cast<double*>(s_all);
    const int grp = threadIdx.x / kThr, tid = threadIdx.x % kThr, lane = tid & 31, warp = tid >> 5;
    const int bar = grp + 1;
    unsigned char* s_grp = s_all + (size_t)kHub * 8 + (size_t)grp * mvh_group_bytes<kThr, kNnz, kRows>();
    double* s_vals = reinterpret_cast<double*>(s_grp);
    int* s_rp = reinterpret_cast<int*>(s_vals + kNnz);
    double* s_y = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(s_rp) + mv_rp_bytes<kRows>());
    double* s_row = s_y + kRows;  // [kW] long-row partials
    double* s_l1 = s_row + kW;    // [kW]
    double* s_dm = s_l1 + kW;     // [kW]
    uint32_t* s_claim = reinterpret_cast<uint32_t*>(s_dm + kW);

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous sweep's shares, acc, state, counters
    const ColState st = a.state_in[0];
    const uint32_t n_items = a.n_items;

    if (!st.active) {
        // column stopped earlier: only a pending combine remains (tpa.cpp:73)
        if (a.out)
            for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < a.n; v += gridDim.x * blockDim.x)
                combine_only(a, v, 0, 1, v);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            a.state_out[0] = st;
            if (M.limbs)
                for (int k = 0; k < 6; ++k) M.limbs[k] = 0ull;
        }
        return;
    }
    // first claim in flight while the hub slice loads
    uint32_t nxt = 0;
    if (tid == 0) nxt = atomicAdd(H.next_item, H.chunk);
    {
        const uint32_t hub2 = H.hub / 2;
        const double2* src = reinterpret_cast<const double2*>(a.share_in);
        double2* dst = reinterpret_cast<double2*>(s_hub);
        for (uint32_t k = threadIdx.x; k < hub2; k += kThr * kGroups) dst[k] = __ldg(src + k);
        if ((H.hub & 1) && threadIdx.x == 0) s_hub[H.hub - 1] = __ldg(a.share_in + H.hub - 1);
    }
    __syncthreads();
    const uint32_t hub = H.hub;
    const bool want_dm = a.policy == kUniform;
    // the group's exact totals (thread 0)
    unsigned long long l1h = 0, l1l = 0, dmh = 0, dml = 0;

    for (;;) {
        if (tid == 0) *s_claim = nxt;
        grp_bar<kThr>(bar);
        const uint32_t cur = *s_claim;
        if (cur >= n_items) break;
        if (tid == 0) nxt = atomicAdd(H.next_item, H.chunk);  // the next claim's round trip hides behind this one's tiles
        const uint32_t cend = min(cur + H.chunk, n_items);
        for (uint32_t item = cur; item < cend; ++item) {
            const uint2 it = a.items[item];
            const uint32_t rb = it.x, re = it.y & ~kLongFlag;
            const bool is_long = (it.y & kLongFlag) != 0;
            const longlong2 nr = M.item_nnz[item];
            const int64_t nb = nr.x, ne = nr.y;
            double my_l1 = 0.0, my_dm = 0.0;
            auto add_row = [&](double y, bool dangling) {
                my_l1 = dadd(my_l1, fabs(y));
                if (want_dm && dangling) my_dm = dadd(my_dm, y);
            };
            if (!is_long) {
                const uint32_t nrows = re - rb;
                const int nnz = (int)(ne - nb);
                constexpr int U = kNnz / kThr;
                constexpr int RPT = kRows / kThr;
                // ---- round trip 1: indices, row pointers, degrees, accumulators ----
                uint32_t u[U];
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int k = tid + j * kThr;
                    u[j] = k < nnz ? ld_col(a.col + nb + k) : 0u;
                }
                for (uint32_t r = tid; r <= nrows; r += kThr) s_rp[r] = (int)(__ldg(a.row_ptr + rb + r) - nb);
                uint32_t dg[RPT], so[RPT];
                double ac[RPT];
#pragma unroll
                for (int q = 0; q < RPT; ++q) {
                    const uint32_t r = tid + q * kThr;
                    dg[q] = r < nrows ? __ldg(a.deg + rb + r) : 0u;
                    so[q] = r < nrows ? __ldg(a.rank + rb + r) : 0u;  // share slot
                    ac[q] = (r < nrows && a.acc) ? a.acc[rb + r] : 0.0;
                }
                // ---- round trip 2: gathers (hub slots from shared memory) ----
                double v[U];
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int k = tid + j * kThr;
                    v[j] = 0.0;
                    if (k < nnz && u[j] >= hub) v[j] = mvh_gather(a.share_in + u[j]);
                }
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int k = tid + j * kThr;
                    if (k < nnz && u[j] < hub) v[j] = s_hub[u[j]];
                }
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const int k = tid + j * kThr;
                    if (k < nnz) s_vals[k] = v[j];
                }
                grp_bar<kThr>(bar);
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
                grp_bar<kThr>(bar);
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
                        const double sv = dg[q] ? ddiv(dmul(a.keep, y), (double)dg[q]) : 0.0;  // graph.cpp:222
                        a.share_out[so[q]] = sv;
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
                    for (int j = 0; j < U; ++j) {
                        v[j] = 0.0;
                        if (u[j] >= hub) v[j] = mvh_gather(a.share_in + u[j]);
                    }
#pragma unroll
                    for (int j = 0; j < U; ++j)
                        if (u[j] < hub) v[j] = s_hub[u[j]];
#pragma unroll
                    for (int j = 0; j < U; ++j) s = dadd(s, v[j]);
                }
                for (; e < ne; e += kThr) {
                    const uint32_t c = ld_col(a.col + e);
                    s = dadd(s, c < hub ? s_hub[c] : mvh_gather(a.share_in + c));
                }
                s = warp_sum(s);
                if (lane == 0) s_row[warp] = s;
                grp_bar<kThr>(bar);
                if (tid == 0) {
                    double y = s_row[0];
#pragma unroll
                    for (int k = 1; k < kW; ++k) y = dadd(y, s_row[k]);
                    const uint32_t d = __ldg(a.deg + rb);
                    if (st.has_spread) y = dadd(y, st.spread);  // graph.cpp:265-268
                    if (a.y_out) a.y_out[rb] = y;
                    if (a.acc) {
                        const double f = dadd(a.acc[rb], y);  // cpi.cpp:50
                        if (a.out) a.out[rb] = a.stranger ? dadd(dmul(a.scale, f), a.stranger[rb]) : dmul(f, a.scale);
                        else a.acc[rb] = f;
                    }
                    if (a.share_out) a.share_out[a.rank[rb]] = d ? ddiv(dmul(a.keep, y), (double)d) : 0.0;
                    add_row(y, d == 0);
                }
            }
            // tile partials (K2's fixed tree) into the group's exact totals
            my_l1 = warp_sum(my_l1);
            if (want_dm) my_dm = warp_sum(my_dm);
            if (lane == 0) {
                s_l1[warp] = my_l1;
                s_dm[warp] = my_dm;
            }
            grp_bar<kThr>(bar);
            if (tid == 0) {
                double tl1 = s_l1[0], tdm = s_dm[0];
#pragma unroll
                for (int k = 1; k < kW; ++k) {
                    tl1 = dadd(tl1, s_l1[k]);
                    tdm = dadd(tdm, s_dm[k]);
                }
                if (tl1 != 0.0) fx_add(l1h, l1l, tl1);
                if (want_dm && tdm != 0.0) fx_add(dmh, dml, tdm);
            }
        }
    }
    if (tid == 0) {
        if (l1h | l1l) fx_atomic_add(&M.fx[0], &M.fx[1], l1h, l1l);
        if (dmh | dml) fx_atomic_add(&M.fx[2], &M.fx[3], dmh, dml);
        __threadfence();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    __threadfence();
    if (atomicAdd(a.done_cnt, 1u) != gridDim.x - 1) return;
    __threadfence();
    const unsigned long long h0 = atomicAdd(&M.fx[0], 0ull), l0 = atomicAdd(&M.fx[1], 0ull);
    const unsigned long long h1 = atomicAdd(&M.fx[2], 0ull), l1 = atomicAdd(&M.fx[3], 0ull);
    if (M.limbs) {
        fx_to_limbs(h0, l0, M.limbs);
        fx_to_limbs(h1, l1, M.limbs + 3);
    } else {
        a.state_out[0] = advance_state(st, fx_decode(h0, l0), fx_decode(h1, l1), a);  // cpi.cpp:73-80
    }
    for (int k = 0; k < 4; ++k) M.fx[k] = 0ull;
    *H.next_item = 0;
    *a.done_cnt = 0;
}

}  // namespace tpa
