// cpi_spmm_tma.cuh -- EXPERIMENT (not built into the library): the dense
// B = 32 sweep of a seed batch with the share-row gathers on the Tensor Memory
// Accelerator (sm_100a tile::gather4).  Measured bitwise equal to K3 and 10x
// slower (C4 sweep 4: 154 ms vs 14 ms): the single producer warp per SM walks
// a dependent index -> frontier-bit -> issue chain per 32-position window
// (~1.4 us each, 112 k windows per SM at C4); see profiles/r02_experiments.md.
// It was wired into tpa_gpu.cu's launch_step for B = 32 (with a `tma` flag in
// Mm4Args telling K3 to leave the dense sweeps) at commit "TMA gather4 SpMM
// kernel k_mm_tma".
//
// K3 (cpi_spmm5.cuh) gathers every 256-byte share row with one LDG per lane
// (lane = column): ~14 warp instructions per nonzero, 64 registers, 32 warps
// per SM -- latency-bound with half the issue slots busy (profiles/r02_ncu_c4.md).
// Here the gathers leave the register file:
//   * one PRODUCER warp per CTA claims work items (long-row segments, then
//     <= 8-row blocks, the K3 schedule), reads each 32-position window's
//     column indices and frontier bits, and issues one
//     cp.async.bulk.tensor.2d...tile::gather4 per four live sources into a
//     ring of 32-row slots in shared memory (mbarrier complete_tx);
//   * C CONSUMER warps take the items round robin and sum the slots' rows in
//     position order -- lane = column, one LDS + one DADD per live nonzero,
//     the same strictly sequential per-row order as K3 (bitwise its result)
//     -- then run K3's epilogue (acc, share_out, bitmaps, fixed-point
//     residual, the fused combine of the last sweep).
// Full / empty mbarriers per slot and per item-queue entry; no CTA barrier in
// the loop.  Dense sweeps only (the sparse ones stay on K3); the kernel exits
// at once when the frontier marking chose a sparse pull.
#pragma once

#include <cuda.h>

#include "cpi_spmm5.cuh"

namespace tpa {

struct MmT {
    static constexpr int B = 32;
    static constexpr int RB = 8;          // rows per block item (blocks_w[1])
    static constexpr int C = 7;           // consumer warps
    static constexpr int NT = 32 * (C + 1);
    static constexpr int S = 20;          // ring slots (32 rows x 256 B each)
    static constexpr int Q = 16;          // item queue entries
    static constexpr int TS = B + 2;      // acc tile row stride (doubles)
    static constexpr size_t kSlotBytes = 32 * B * 8;
    static constexpr size_t kRing = S * kSlotBytes;
    static constexpr size_t kConsBytes = RB * B * 8 + RB * TS * 8;  // yb + acc tile per consumer
    static constexpr size_t kDynSmem = kRing + C * kConsBytes;
};

struct TmaItem {
    uint32_t kind;   // 0 block, 1 segment, 2 end
    uint32_t id;     // segment id (kind 1)
    uint32_t r0, nrows;
    int64_t e0, e1;
    uint32_t seq0;   // ring sequence number of the first window
    uint32_t pad;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* tm, uint32_t r0, uint32_t r1, uint32_t r2,
                                            uint32_t r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar))
        : "memory");
}

template <bool kLast>
__global__ void __launch_bounds__(MmT::NT, 1) k_mm_tma(const __grid_constant__ CUtensorMap tm, Mm4Args P) {
    constexpr int B = MmT::B, RB = MmT::RB, C = MmT::C, S = MmT::S, Q = MmT::Q, TS = MmT::TS;
    const MmArgs& A = P.m;
    const StepArgs& a = A.s;
    extern __shared__ __align__(1024) unsigned char s_dyn[];
    __shared__ uint64_t full[S], empty[S], ifull[Q], iempty[Q];
    __shared__ uint32_t live_of[S];
    __shared__ TmaItem items[Q];
    __shared__ uint32_t s_u[32];
    __shared__ unsigned long long s_fx[4 * B];
    __shared__ uint32_t s_ticket;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // a sparse sweep (frontier marking chose the pull over marked windows) stays on K3
    const bool dense = P.rowflag == nullptr || *P.dense != 0;
    if (!dense) return;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int q = 0; q < Q; ++q) {
            mbar_init(&ifull[q], 1);
            mbar_init(&iempty[q], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < 4 * B; i += MmT::NT) s_fx[i] = 0ull;
    __syncthreads();

    const uint32_t total = A.n_segs + P.n_blocks_rb;
    double* ring = reinterpret_cast<double*>(s_dyn);

    if (wid == 0) {
        // ------------------------------ producer ------------------------------
        const uint32_t* __restrict__ nz = A.nz_in;
        uint32_t seq = 0, qn = 0, n_end = 0;
        uint32_t item = blockIdx.x;  // first item by CTA id, then the global counter
        const uint32_t n_ctas = gridDim.x;
        for (;;) {
            TmaItem it{};
            if (item >= total) {
                it.kind = 2;
            } else if (item < A.n_segs) {
                it.kind = 1;
                it.id = item;
                it.r0 = A.seg_row[item];
                it.nrows = 1;
                it.e0 = A.seg_lo[item];
                it.e1 = min(it.e0 + (int64_t)kLong, (int64_t)__ldg(a.row_ptr + it.r0 + 1));
            } else {
                const uint2 blk = P.blocks_rb[item - A.n_segs];
                it.kind = 0;
                it.r0 = blk.x;
                it.nrows = blk.y;
                it.e0 = __ldg(a.row_ptr + blk.x);
                it.e1 = __ldg(a.row_ptr + blk.x + blk.y);
            }
            it.seq0 = seq;
            const int qs = (int)(qn % Q);
            mbar_wait(&iempty[qs], ((qn / Q) & 1) ^ 1);
            if (lane == 0) {
                items[qs] = it;
                mbar_arrive(&ifull[qs]);
            }
            ++qn;
            if (it.kind == 2) {
                // C end markers: one lands in every consumer's residue class
                if (++n_end == C) break;
                continue;
            }
            // the item's windows: 32 positions each, live sources gathered 4 per request
            for (int64_t wb = it.e0; wb < it.e1; wb += 32) {
                const int s = (int)(seq % S);
                mbar_wait(&empty[s], ((seq / S) & 1) ^ 1);
                const int64_t e = wb + lane;
                const uint32_t u = e < it.e1 ? __ldg(a.col + e) : 0u;
                const bool lv = e < it.e1 && (!nz || ((__ldg(nz + (u >> 5)) >> (u & 31)) & 1u));
                const uint32_t live = __ballot_sync(0xffffffffu, lv);
                const int cnt = __popc(live);
                if (lv) s_u[__popc(live & ((1u << lane) - 1u))] = u;
                __syncwarp();
                const int nreq = (cnt + 3) >> 2;
                if (lane == 0) {
                    live_of[s] = live;
                    mbar_arrive_tx(&full[s], (uint32_t)(nreq * 4 * B * 8));
                }
                __syncwarp();
                if (lane < nreq) {
                    const int k = lane * 4;
                    const uint32_t z = A.zero_row;
                    tma_gather4(ring + ((size_t)s * 32 + k) * B, &tm, s_u[k], k + 1 < cnt ? s_u[k + 1] : z,
                                k + 2 < cnt ? s_u[k + 2] : z, k + 3 < cnt ? s_u[k + 3] : z, &full[s]);
                }
                __syncwarp();
                ++seq;
            }
            if (lane == 0) item = n_ctas + atomicAdd(A.work_cnt, 1u);
            item = __shfl_sync(0xffffffffu, item, 0);
        }
    } else {
        // ------------------------------ consumers -----------------------------
        const int cw = wid - 1;
        double (*yb)[B] = reinterpret_cast<double (*)[B]>(s_dyn + MmT::kRing + (size_t)cw * MmT::kConsBytes);
        double* tile = reinterpret_cast<double*>(s_dyn + MmT::kRing + (size_t)cw * MmT::kConsBytes + RB * B * 8);
        const int c0 = lane;
        const ColState st = a.state_in[c0];
        const bool want_dm = a.policy == kUniform;
        unsigned long long fx[4] = {0ull, 0ull, 0ull, 0ull};
        for (uint32_t qn = cw;; qn += C) {
            const int qs = (int)(qn % Q);
            mbar_wait(&ifull[qs], (qn / Q) & 1);
            const TmaItem it = items[qs];
            __syncwarp();
            if (lane == 0) mbar_arrive(&iempty[qs]);
            if (it.kind == 2) break;
            const bool is_seg = it.kind == 1;
            const uint32_t r0 = it.r0;
            const int nrows = (int)it.nrows;
            const int64_t e0 = it.e0, e1 = it.e1;
            int64_t rpl;
            if (is_seg) rpl = lane == 0 ? e0 : e1;
            else rpl = lane <= nrows ? __ldg(a.row_ptr + r0 + lane) : 0;
            const uint32_t av = (A.acc_valid && a.acc) ? __ldcg(A.acc_valid + (r0 >> 5)) : 0u;
            const uint32_t dl = lane < nrows ? __ldg(a.deg + r0 + lane) : 0u;
            if (!is_seg && a.acc)
                for (int k = 0; k < nrows; ++k)
                    if ((av >> ((r0 + k) & 31)) & 1u) cp_async_acc<1>(tile + k * TS + c0, a.acc + (size_t)(r0 + k) * B + c0, L2Pol{});
            asm volatile("cp.async.commit_group;\n" ::: "memory");
            const int64_t rpn = __shfl_down_sync(0xffffffffu, rpl, 1);
            const bool starts = !is_seg && lane >= 1 && lane < nrows && rpn > rpl && rpl > e0;
            const uint32_t ne_mask = __ballot_sync(0xffffffffu, lane < nrows && rpn > rpl);
            int cur = ne_mask ? __ffs(ne_mask) - 1 : 0;
            for (int k = 0; k < nrows; ++k) yb[k][c0] = 0.0;
            double s = 0.0;
            uint32_t seq = it.seq0;
            for (int64_t wb = e0; wb < e1; wb += 32, ++seq) {
                const int sl = (int)(seq % S);
                mbar_wait(&full[sl], (seq / S) & 1);
                const uint32_t live = live_of[sl];
                const double* rows = ring + (size_t)sl * 32 * B;
                const int64_t p = rpl - wb;
                uint32_t smask = __ballot_sync(0xffffffffu, starts && p >= 0 && p < 32);
                int rk = 0;
                const int lim = (int)(e1 - wb < 32 ? e1 - wb : 32);
                for (int j = 0; j < lim; ++j) {
                    if (smask & 1u) {  // a row starts at position j (warp-uniform)
                        const int kn = __ffs(__ballot_sync(0xffffffffu, starts && p == j)) - 1;
                        yb[cur][c0] = s;
                        s = 0.0;
                        cur = kn;
                    }
                    smask >>= 1;
                    if ((live >> j) & 1u) s = dadd(s, rows[(size_t)(rk++) * B + c0]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[sl]);
            }
            if (is_seg) {
                A.seg_part[(size_t)it.id * B + c0] = s;
                __threadfence();
                __syncwarp();
                const uint32_t li = A.seg_long[it.id];
                uint32_t t = 0;
                if (lane == 0) t = atomicAdd(A.long_cnt + li, 1u);
                t = __shfl_sync(0xffffffffu, t, 0);
                if (t != A.long_nseg[li] - 1) continue;
                __threadfence();
                const uint32_t f0 = A.long_first[li], ns = A.long_nseg[li];
                yb[0][c0] = seg_sum(A.seg_part + (size_t)f0 * B + c0, B, ns);
                if (lane == 0) A.long_cnt[li] = 0;
                if (a.acc && ((av >> (r0 & 31)) & 1u)) cp_async_acc<1>(tile + c0, a.acc + (size_t)r0 * B + c0, L2Pol{});
                asm volatile("cp.async.commit_group;\n" ::: "memory");
            } else if (ne_mask) {
                yb[cur][c0] = s;
            }
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            __syncwarp();
            // ---- K3's block epilogue (cpi_spmm5.cuh): rows r0 .. r0+nrows-1 ----
            double bl1 = 0.0, bdm = 0.0;
            uint32_t nzw = 0, avw = 0;
            for (int k = 0; k < nrows; ++k) {
                const uint32_t r = r0 + k;
                const uint32_t d = __shfl_sync(0xffffffffu, dl, k);
                const bool valid = (av >> (r & 31)) & 1u;
                double yy = yb[k][c0];
                if (st.has_spread) yy = dadd(yy, st.spread);  // graph.cpp:265-268
                if (!st.active) yy = 0.0;
                const double ao = valid ? tile[k * TS + c0] : 0.0;
                const bool row_nz = __ballot_sync(0xffffffffu, yy != 0.0) != 0;
                if (!kLast && !row_nz) continue;
                const size_t ix = (size_t)r * B + c0;
                if (!st.active) {
                    if (kLast) tile[k * TS + c0] = combine_value(a, ao, r);
                    else if (!valid) a.acc[ix] = 0.0;
                } else {
                    const double f = dadd(ao, yy);  // cpi.cpp:50
                    if (kLast) {
                        tile[k * TS + c0] = combine_value(a, f, r);  // tpa.cpp:73-74
                    } else {
                        a.acc[ix] = f;
                        a.share_out[ix] = d ? ddiv(dmul(a.keep, yy), (double)d) : 0.0;  // graph.cpp:222
                    }
                    bl1 = dadd(bl1, fabs(yy));
                    if (want_dm && d == 0) bdm = dadd(bdm, yy);
                }
                nzw |= (row_nz ? 1u : 0u) << (r & 31);
                avw |= 1u << (r & 31);
            }
            if (kLast) {
                __syncwarp();
                if (a.out_node_major) {
                    for (int k = 0; k < nrows; ++k)
                        if (c0 < (int)a.b_valid) a.out[(size_t)(r0 + k) * B + c0] = tile[k * TS + c0];
                } else {
                    const int k = lane % RB;
                    for (uint32_t b = lane / RB; b < a.b_valid; b += 32 / RB)
                        if (k < nrows) a.out[(size_t)b * a.n + r0 + k] = tile[k * TS + b];
                }
                __syncwarp();
            }
            if (bl1 != 0.0) fx_add(fx[0], fx[1], bl1);
            if (bdm != 0.0) fx_add(fx[2], fx[3], bdm);
            if (lane == 0 && !kLast) {
                if (A.nz_out && nzw) atomicOr(A.nz_out + (r0 >> 5), nzw);
                if (A.acc_valid && avw) atomicOr(A.acc_valid + (r0 >> 5), avw);
            }
            __syncwarp();
        }
        if (fx[0] | fx[1]) fx_atomic_add(&s_fx[4 * c0 + 0], &s_fx[4 * c0 + 1], fx[0], fx[1]);
        if (fx[2] | fx[3]) fx_atomic_add(&s_fx[4 * c0 + 2], &s_fx[4 * c0 + 3], fx[2], fx[3]);
    }
    // residual / dangling mass: exact integer sums; the last CTA advances the states
    __syncthreads();
    for (int b = tid; b < B; b += MmT::NT) {
        if (s_fx[4 * b + 0] | s_fx[4 * b + 1])
            fx_atomic_add(&A.fx[4 * b + 0], &A.fx[4 * b + 1], s_fx[4 * b + 0], s_fx[4 * b + 1]);
        if (s_fx[4 * b + 2] | s_fx[4 * b + 3])
            fx_atomic_add(&A.fx[4 * b + 2], &A.fx[4 * b + 3], s_fx[4 * b + 2], s_fx[4 * b + 3]);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_ticket = atomicAdd(a.done_cnt, 1u);
    __syncthreads();
    if (s_ticket != gridDim.x - 1) return;
    __threadfence();
    for (int b = tid; b < B; b += MmT::NT) {
        ColState sc = a.state_in[b];
        const unsigned long long h0 = atomicAdd(&A.fx[4 * b + 0], 0ull), l0 = atomicAdd(&A.fx[4 * b + 1], 0ull);
        const unsigned long long h1 = atomicAdd(&A.fx[4 * b + 2], 0ull), l1 = atomicAdd(&A.fx[4 * b + 3], 0ull);
        if (sc.active) {
            const double res = fx_decode(h0, l0);
            const double dm = fx_decode(h1, l1);
            sc.residual = res;
            sc.iters = a.step;
            sc.converged = res < a.eps;
            sc.active = !sc.converged && (a.terminal < 0 || (int64_t)a.step < a.terminal);
            sc.has_spread = (a.policy == kUniform && dm != 0.0);
            sc.spread = sc.has_spread ? ddiv(dmul(a.keep, dm), (double)a.n) : 0.0;
        }
        a.state_out[b] = sc;
        A.fx[4 * b + 0] = A.fx[4 * b + 1] = A.fx[4 * b + 2] = A.fx[4 * b + 3] = 0ull;
    }
    if (tid == 0) {
        *A.work_cnt = 0;
        *a.done_cnt = 0;
    }
}

}  // namespace tpa
