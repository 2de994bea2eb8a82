// cpi_spmm3.cuh -- K3 v3: the SpMM sweep for B = 32 / 64 with the gathers
// staged through a per-warp shared-memory ring by cp.async.
//
// Same contract, work items, bitmaps, epilogue and reduction as v2
// (cpi_spmm.cuh).  What changes is how the sources' B-wide share rows reach
// the warp: instead of loads into registers (register-bound depth), every
// position of the item's stream is copied global -> shared with
// cp.async.cg (16 B per lane; a dead source is a zero-fill with src-size 0,
// no memory traffic), kRing positions ahead of the sequential summation.  In
// flight data therefore costs no registers, and each warp keeps kRing rows
// (kRing x B x 8 bytes) of gathers outstanding while it sums.
#pragma once

#include "cpi_spmm.cuh"

namespace tpa {

constexpr int kC3 = 16;     // positions per pipeline stage (one commit group)

template <int B>
struct Mm3Shape {
    static_assert(B == 32 || B == 64, "v3 handles warp-wide rows");
    static constexpr int CPL = B / 32;             // columns per lane
    static constexpr int NGRP = 4;                 // warps per CTA
    static constexpr int NT = NGRP * 32;
    static constexpr int RPI = 512 / (B * 8);      // rows per cp.async instruction (2 or 1)
    static constexpr int PPR = 32 / RPI;           // lanes per row
    static constexpr int RING = 16384 / (B * 8);   // positions in flight per warp (16 KiB)
    static constexpr size_t kRingBytes = (size_t)RING * B * 8;
    static constexpr size_t kYBytes = (size_t)kMmRows * B * 8;
    static constexpr size_t kGrpBytes = kRingBytes + 2 * kYBytes;  // ring | ybuf | abuf
    static constexpr size_t kDynSmem = NGRP * kGrpBytes;
};

__device__ __forceinline__ void cp_async16_zfill(void* dst_smem, const void* src, bool live) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst_smem);
    const uint32_t n = live ? 16u : 0u;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Raw source indices + one live bit per position (group = warp).
__device__ __forceinline__ bool stage_raw(const MmArgs& A, int64_t lo, int nnz, int padded, int lane,
                                          uint32_t* sidx, uint32_t* lbits) {
    constexpr int PER = 8;
    const uint32_t* __restrict__ col = A.s.col;
    const uint32_t* __restrict__ nz = A.nz_in;
    uint32_t any = 0;
    for (int p0 = 0; p0 < padded; p0 += PER * 32) {
        uint32_t u[PER], w[PER];
#pragma unroll
        for (int t = 0; t < PER; ++t) {
            const int e = p0 + t * 32 + lane;
            u[t] = e < nnz ? ld_stream_u32(col + lo + e) : 0u;
        }
#pragma unroll
        for (int t = 0; t < PER; ++t) {
            const int e = p0 + t * 32 + lane;
            w[t] = (nz && e < nnz) ? __ldg(nz + (u[t] >> 5)) : 0xffffffffu;
        }
#pragma unroll
        for (int t = 0; t < PER; ++t) {
            const int e0 = p0 + t * 32;
            if (e0 >= padded) break;
            const int e = e0 + lane;
            const bool live = e < nnz && ((w[t] >> (u[t] & 31)) & 1u);
            sidx[e] = u[t];
            const uint32_t bits = __ballot_sync(0xffffffffu, live);
            if (lane == 0) lbits[e0 >> 5] = bits;
            any |= bits;
        }
    }
    __syncwarp();
    return any != 0;
}

template <int B>
__global__ void __launch_bounds__(Mm3Shape<B>::NT) k_step_spmm3(MmArgs A) {
    using Sh = Mm3Shape<B>;
    constexpr int CPL = Sh::CPL, NGRP = Sh::NGRP, NT = Sh::NT, RPI = Sh::RPI, PPR = Sh::PPR;
    constexpr int RING = Sh::RING;
    constexpr int CIN = RING / kC3;  // stages in flight
    const StepArgs& a = A.s;
    extern __shared__ __align__(16) unsigned char s_dyn[];
    __shared__ int64_t s_rp[NGRP][kMmRows + 2];
    __shared__ __align__(16) uint32_t s_idx[NGRP][kBlockNnz];
    __shared__ uint32_t s_lb[NGRP][kBlockNnz / 32];
    __shared__ uint32_t s_rs[NGRP][kBlockNnz / 32 + 2];
    __shared__ int8_t s_nx[NGRP][kMmRows + 1];
    __shared__ ColState s_st[B];
    __shared__ unsigned long long s_fx[4 * B];
    __shared__ uint32_t s_ticket;
    __shared__ int s_any;

    const int tid = threadIdx.x;
    const int grp = tid >> 5, lane = tid & 31;
    const int c0 = lane * CPL;

    if (tid == 0) s_any = 0;
    for (int i = tid; i < 4 * B; i += NT) s_fx[i] = 0ull;
    __syncthreads();
    for (int b = tid; b < B; b += NT) {
        s_st[b] = a.state_in[b];
        if (s_st[b].active) s_any = 1;
    }
    __syncthreads();
    ColState st[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) st[c] = s_st[c0 + c];
    const bool any_active = s_any != 0;

    unsigned long long fx[4][CPL];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < CPL; ++c) fx[q][c] = 0ull;

    unsigned char* gbase = s_dyn + (size_t)grp * Sh::kGrpBytes;
    double (*ring)[B] = reinterpret_cast<double (*)[B]>(gbase);
    double (*yb)[B] = reinterpret_cast<double (*)[B]>(gbase + Sh::kRingBytes);
    double (*ab)[B] = reinterpret_cast<double (*)[B]>(gbase + Sh::kRingBytes + Sh::kYBytes);
    int64_t* rp = s_rp[grp];
    uint32_t* sidx = s_idx[grp];
    uint32_t* lb = s_lb[grp];
    uint32_t* rsb = s_rs[grp];
    const double* __restrict__ share = a.share_in;

    const uint32_t total = A.n_segs + A.n_blocks;
    const bool work = any_active || a.out != nullptr;
    uint32_t next_item = 0;
    if (work && lane == 0) next_item = atomicAdd(A.work_cnt, 1u);
    while (work) {
        const uint32_t item = __shfl_sync(0xffffffffu, next_item, 0);
        if (item >= total) break;
        if (lane == 0) next_item = atomicAdd(A.work_cnt, 1u);
        const bool is_seg = item < A.n_segs;
        uint32_t r0;
        int nrows;
        if (is_seg) {
            r0 = A.seg_row[item];
            nrows = 1;
            if (lane == 0) {
                rp[0] = A.seg_lo[item];
                rp[1] = min(rp[0] + (int64_t)kLong, __ldg(a.row_ptr + r0 + 1));
            }
        } else {
            const uint2 blk = A.blocks[item - A.n_segs];
            r0 = blk.x;
            nrows = (int)blk.y;
            if (lane <= nrows) rp[lane] = __ldg(a.row_ptr + r0 + lane);
        }
        uint32_t deg_lane[1];
        deg_lane[0] = lane < nrows ? __ldg(a.deg + r0 + lane) : 0u;
        __syncwarp();
        const int64_t lo = rp[0];
        const int nnz = (int)(rp[nrows] - lo);
        const int padded = (nnz + kC3 - 1) / kC3 * kC3;
        double s[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) s[c] = 0.0;
        const bool live = any_active && nnz > 0 && stage_raw(A, lo, nnz, padded, lane, sidx, lb);
        if (!is_seg) {
            for (int k = lane; k < (nnz + 31) / 32 + 1; k += 32) rsb[k] = 0u;
            for (int k = 0; k < nrows; ++k)
#pragma unroll
                for (int c = 0; c < CPL; ++c) yb[k][c0 + c] = 0.0;
            if (lane == 0) {
                int nx = nrows;
                for (int k = nrows - 1; k >= 0; --k) {
                    s_nx[grp][k] = (int8_t)nx;
                    if (rp[k + 1] > rp[k]) nx = k;
                }
                s_nx[grp][kMmRows] = (int8_t)nx;
            }
            __syncwarp();
            if (lane >= 1 && lane < nrows) {
                const int p = (int)(rp[lane] - lo);
                if (rp[lane + 1] > rp[lane] && p > 0) atomicOr(&rsb[p >> 5], 1u << (p & 31));
            }
        }
        __syncwarp();
        if (live) {
            const int nst = padded / kC3;
            auto stage_live = [&](int c) {
                const uint32_t w = lb[(c * kC3) >> 5];
                return ((w >> ((c * kC3) & 31)) & ((1u << kC3) - 1u)) != 0u;
            };
            // issue stage c: kC3 positions, RPI rows per instruction
            auto issue = [&](int c) {
                if (c < nst && stage_live(c)) {
#pragma unroll
                    for (int i = 0; i < kC3 / RPI; ++i) {
                        const int p = c * kC3 + i * RPI + lane / PPR;
                        const int q = lane % PPR;  // 16-byte piece of the row
                        const bool lv = (lb[p >> 5] >> (p & 31)) & 1u;
                        cp_async16_zfill(&ring[p & (RING - 1)][2 * q], share + (size_t)sidx[p] * B + 2 * q, lv);
                    }
                }
                cp_async_commit();
            };
            const int8_t* nxt = s_nx[grp];
            int cur = is_seg ? 0 : nxt[kMmRows];
#pragma unroll
            for (int c = 0; c < CIN; ++c) issue(c);
            for (int c = 0; c < nst; ++c) {
                cp_async_wait<CIN - 1>();
                __syncwarp();
                const int base = c * kC3;
                const uint32_t rs = is_seg ? 0u : (rsb[base >> 5] >> (base & 31)) & ((1u << kC3) - 1u);
                if (stage_live(c)) {
                    double v[kC3][CPL];
#pragma unroll
                    for (int j = 0; j < kC3; ++j) {
                        const double* src = &ring[(base + j) & (RING - 1)][c0];
                        if constexpr (CPL == 1) {
                            v[j][0] = *src;
                        } else {
                            const double2 t = *reinterpret_cast<const double2*>(src);
                            v[j][0] = t.x;
                            v[j][1] = t.y;
                        }
                    }
#pragma unroll
                    for (int j = 0; j < kC3; ++j) {
                        const bool nb = (rs >> j) & 1u;
#pragma unroll
                        for (int c2 = 0; c2 < CPL; ++c2) {
                            const double fin = s[c2];
                            const double t = dadd(s[c2], v[j][c2]);
                            s[c2] = nb ? v[j][c2] : t;  // a new row starts from 0.0 + v == v
                            if (nb) yb[cur][c0 + c2] = fin;
                        }
                        if (nb) cur = nxt[cur];
                    }
                } else {
                    uint32_t m = rs;
                    while (m) {
                        m &= m - 1;
#pragma unroll
                        for (int c2 = 0; c2 < CPL; ++c2) {
                            yb[cur][c0 + c2] = s[c2];
                            s[c2] = 0.0;
                        }
                        cur = nxt[cur];
                    }
                }
                __syncwarp();
                issue(c + CIN);
            }
            cp_async_wait<0>();
            if (!is_seg && nnz > 0)
#pragma unroll
                for (int c2 = 0; c2 < CPL; ++c2) yb[cur][c0 + c2] = s[c2];
        }
        if (is_seg) {
#pragma unroll
            for (int c = 0; c < CPL; ++c) A.seg_part[(size_t)item * B + c0 + c] = s[c];
            __threadfence();
            __syncwarp();
            const uint32_t li = A.seg_long[item];
            uint32_t t = 0;
            if (lane == 0) t = atomicAdd(A.long_cnt + li, 1u);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t != A.long_nseg[li] - 1) continue;
            __threadfence();
            const uint32_t f0 = A.long_first[li], ns = A.long_nseg[li];
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const double y = seg_sum(A.seg_part + (size_t)f0 * B + c0 + c, B, ns);
                yb[0][c0 + c] = y;
            }
            if (lane == 0) A.long_cnt[li] = 0;
        }
        __syncwarp();
        mm_epilogue_rows<B>(A, st, r0, nrows, yb, ab, deg_lane, lane, c0, fx);
        __syncwarp();
    }

#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int b = c0 + c;
        if (fx[0][c] | fx[1][c]) fx_atomic_add(&s_fx[4 * b + 0], &s_fx[4 * b + 1], fx[0][c], fx[1][c]);
        if (fx[2][c] | fx[3][c]) fx_atomic_add(&s_fx[4 * b + 2], &s_fx[4 * b + 3], fx[2][c], fx[3][c]);
    }
    __syncthreads();
    for (int b = tid; b < B; b += NT) {
        if (s_fx[4 * b + 0] | s_fx[4 * b + 1]) fx_atomic_add(&A.fx[4 * b + 0], &A.fx[4 * b + 1], s_fx[4 * b + 0], s_fx[4 * b + 1]);
        if (s_fx[4 * b + 2] | s_fx[4 * b + 3]) fx_atomic_add(&A.fx[4 * b + 2], &A.fx[4 * b + 3], s_fx[4 * b + 2], s_fx[4 * b + 3]);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_ticket = atomicAdd(a.done_cnt, 1u);
    __syncthreads();
    if (s_ticket != gridDim.x - 1) return;
    __threadfence();
    for (int b = tid; b < B; b += NT) {
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
