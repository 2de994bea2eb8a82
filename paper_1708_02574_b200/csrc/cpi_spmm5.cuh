// cpi_spmm5.cuh -- K3 v5: the B-seed sweep (B = 32, 64) as ONE lean kernel.
//
// v4's gather stream (lane = column, 16 gathers in flight, strictly
// sequential per-row sums) with the epilogue folded back in, without the
// per-warp register weight that capped v2 at 16 warps/SM:
//   * at block start the block's accumulator rows are copied global -> shared
//     by cp.async (they arrive while the gathers run: no exposed round trip);
//   * a closing row only stores its B sums to a small shared buffer;
//   * after the stream the warp walks the block's <= 16 rows in a rolled
//     loop: acc += y, share_out = keep*y/deg (mid sweeps) or the combine
//     out = (1+nsf)*acc + stranger staged in the same shared tile and written
//     transposed (256-byte contiguous stores into the seed-major output);
//   * bitmaps and the fixed-point residual as in v2/v4.
// No Y round trip through HBM, one launch per sweep.
#pragma once

#include "cpi_frontier.cuh"

namespace tpa {

// B = 16 ("paired" form): a 128-byte share row is one half-warp's load, so
// every gather instruction fetches TWO consecutive positions of the block's
// nonzero stream (lanes 0-15 the even one, 16-31 the odd one), and a
// shfl_xor(16) hands each half the other's value; both halves then add the
// two terms in position order, so every lane holds its column's sum in the
// reference's strictly sequential order (bitwise as B = 32 / 64) and the
// halves stay in lockstep (no divergence).  32 positions per window in
// flight per warp = 4 KB, as B = 32.
template <int B, int RB_>
struct Mm5 {
    static_assert(B == 16 || B == 32 || B == 64, "v5: one warp per row group");
    static_assert(RB_ == 4 || RB_ == 8 || RB_ == 16, "rows per block");
    static constexpr bool PAIR = B == 16;
    static constexpr int CPL = PAIR ? 1 : B / 32;  // columns per lane
    static constexpr int U = PAIR ? 32 : 16 / CPL;  // positions per gather group (PAIR: 16 loads / lane)
    static constexpr int RB = RB_;             // rows per block (the host's block window)
    static constexpr int NW = 4;               // warps per CTA
    static constexpr int NT = NW * 32;
    static constexpr int TS = B + 2;           // padded row stride (doubles) of the tile
    static constexpr size_t kYBytes = (size_t)RB * B * 8;
    static constexpr size_t kTBytes = (size_t)RB * TS * 8;
    static constexpr size_t kWarpBytes = kYBytes + kTBytes;
    static constexpr size_t kDynSmem = NW * kWarpBytes;
};

template <int CPL>
__device__ __forceinline__ void cp_async_acc(double* dst_smem, const double* src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst_smem);
    if constexpr (CPL == 1)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}

template <int B, bool kLast, int RB>
__global__ void __launch_bounds__(Mm5<B, RB>::NT, 8) k_mm_fused(Mm4Args P) {
    using Sh = Mm5<B, RB>;
    constexpr int CPL = Sh::CPL, U = Sh::U, TS = Sh::TS;
    constexpr bool PAIR = Sh::PAIR;
    const MmArgs& A = P.m;
    const StepArgs& a = A.s;
    extern __shared__ __align__(16) unsigned char s_dyn[];
    // column states read straight from global memory and the CTA's
    // fixed-point totals aliased onto the (by then idle) dynamic tile:
    // 2 KB less static shared memory per CTA, left to the L1
    unsigned long long* s_fx = reinterpret_cast<unsigned long long*>(s_dyn);
    __shared__ uint32_t s_ticket;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int c0 = PAIR ? (lane & 15) : lane * CPL;
    const int half = lane >> 4;  // PAIR: which position of a pair this lane loads
    double (*yb)[B] = reinterpret_cast<double (*)[B]>(s_dyn + (size_t)wid * Sh::kWarpBytes);
    double* tile = reinterpret_cast<double*>(s_dyn + (size_t)wid * Sh::kWarpBytes + Sh::kYBytes);

    __syncthreads();
    ColState st[CPL];
    bool any_active = false;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        st[c] = a.state_in[c0 + c];
        any_active = any_active || st[c].active;
    }
    any_active = __any_sync(0xffffffffu, any_active);
    const bool want_dm = a.policy == kUniform;
    unsigned long long fx[4][CPL];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < CPL; ++c) fx[q][c] = 0ull;

    const uint32_t* __restrict__ col = a.col;
    const uint32_t* __restrict__ nz = A.nz_in;
    const double* __restrict__ share = a.share_in;
    const bool use_mask = P.rowflag != nullptr && *P.dense == 0;
    // sparse sweep: the items are the long-row segments + the marked windows
    const bool by_window = use_mask && P.wl != nullptr;
    const uint32_t n_seg_items = by_window ? *P.sl_cnt : A.n_segs;
    const uint32_t total = n_seg_items + (by_window ? *P.wl_cnt : P.n_blocks_rb);
    const bool work = any_active || kLast;

    // first item by warp id, later ones from the shared counter (offset by the
    // warp count): a sparse sweep with fewer items than warps costs no atomics
    const uint32_t n_warps = gridDim.x * Sh::NW;
    uint32_t next_item = blockIdx.x * Sh::NW + wid;
    uint32_t pb = 0, pe = 0;  // blocks of the current window still to do (warp-uniform)
    while (work) {
        uint32_t item = 0;
        bool is_seg = false;
        if (pb >= pe) {
            item = __shfl_sync(0xffffffffu, next_item, 0);
            if (item >= total) break;
            if (lane == 0) next_item = n_warps + atomicAdd(A.work_cnt, 1u);
            is_seg = item < n_seg_items;
            if (is_seg) {
                if (by_window) item = P.sl[item];  // -> segment id
            } else {
                if (by_window) {
                    const uint32_t wdx = P.wl[item - n_seg_items];
                    pb = P.win_blk[wdx];
                    pe = P.win_blk[wdx + 1];
                    if (pb >= pe) continue;
                } else {
                    pb = item - A.n_segs;
                    pe = pb + 1;
                }
            }
        }
        uint32_t r0;
        int nrows;
        if (is_seg) {
            r0 = A.seg_row[item];
            nrows = 1;
        } else {
            const uint2 blk = P.blocks_rb[pb++];
            r0 = blk.x;
            nrows = (int)blk.y;
        }
        // sparse sweep: skip items none of whose rows the frontier reaches
        // (unless a combine still has to produce them)
        if (use_mask && !kLast) {
            const bool mk = lane < nrows && P.rowflag[r0 + lane];
            if (!__any_sync(0xffffffffu, mk)) continue;
        }
        int64_t rpl;
        if (is_seg) {
            const int64_t lo = A.seg_lo[item];
            const int64_t hi = min(lo + (int64_t)kLong, (int64_t)__ldg(a.row_ptr + r0 + 1));
            rpl = lane == 0 ? lo : hi;
        } else {
            rpl = lane <= nrows ? __ldg(a.row_ptr + r0 + lane) : 0;
        }
        // block epilogue inputs, fetched now so they land during the gathers
        const uint32_t av = (A.acc_valid && a.acc) ? __ldcg(A.acc_valid + (r0 >> 5)) : 0u;
        const uint32_t dl = lane < nrows ? __ldg(a.deg + r0 + lane) : 0u;
        if (!is_seg && a.acc) {
            // PAIR: each half-warp fetches the rows its epilogue takes
            for (int k = PAIR ? half : 0; k < nrows; k += PAIR ? 2 : 1)
                if ((av >> ((r0 + k) & 31)) & 1u)
                    cp_async_acc<CPL>(tile + k * TS + c0, a.acc + (size_t)(r0 + k) * B + c0);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");

        const int64_t e0 = __shfl_sync(0xffffffffu, rpl, 0);
        const int64_t e1 = __shfl_sync(0xffffffffu, rpl, nrows);
        const int64_t rpn = __shfl_down_sync(0xffffffffu, rpl, 1);
        const bool starts = !is_seg && lane >= 1 && lane < nrows && rpn > rpl && rpl > e0;
        const uint32_t ne_mask = __ballot_sync(0xffffffffu, lane < nrows && rpn > rpl);
        int cur = ne_mask ? __ffs(ne_mask) - 1 : 0;
        double s[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) s[c] = 0.0;
        for (int k = 0; k < nrows; ++k)
#pragma unroll
            for (int c = 0; c < CPL; ++c) yb[k][c0 + c] = 0.0;
        // PAIR: only the lower half-warp's sums are in position order (the
        // upper half adds the same two terms the other way round), so only
        // the lower half stores them
        const bool keeper = !PAIR || half == 0;
        auto close_row = [&](int k_next) {
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                if (keeper) yb[cur][c0 + c] = s[c];
                s[c] = 0.0;
            }
            cur = k_next;
        };
        // indices 32 at a time (every lane), two windows ahead of use; the
        // U-wide gather groups take their sources from the window by shuffle
        auto idx32 = [&](int64_t base) -> uint32_t {
            const int64_t e = base + lane;
            return e < e1 ? ld_col(col + e) : 0u;
        };
        auto bits32 = [&](uint32_t u, int64_t base) -> uint32_t {
            return (nz && base + lane < e1) ? __ldg(nz + (u >> 5)) : 0xffffffffu;
        };
        if (any_active && e1 > e0) {
            uint32_t i0 = idx32(e0), i1 = idx32(e0 + 32);
            uint32_t w0 = bits32(i0, e0);
            for (int64_t wbase = e0; wbase < e1; wbase += 32) {
                const uint32_t i2 = idx32(wbase + 64);
                const uint32_t w1 = bits32(i1, wbase + 32);
                const uint32_t live32 =
                    __ballot_sync(0xffffffffu, ((w0 >> (i0 & 31)) & 1u) && wbase + lane < e1);
#pragma unroll 1
                for (int h = 0; h < 32 / U; ++h) {
                    const int64_t base = wbase + h * U;
                    if (base >= e1) break;  // warp-uniform
                    const uint32_t lmask = U == 32 ? live32 : (live32 >> (h * U)) & ((1u << (U & 31)) - 1u);
                    const int64_t p = rpl - base;
                    const uint32_t smask = __ballot_sync(0xffffffffu, starts && p >= 0 && p < U);
                    if (PAIR && lmask) {
                        // 16 loads per lane: position 2*jp + half of the window
                        double v[U / 2];
#pragma unroll
                        for (int jp = 0; jp < U / 2; ++jp) {
                            const int pp = 2 * jp + half;
                            const uint32_t u = __shfl_sync(0xffffffffu, i0, h * U + pp);
                            v[jp] = ((lmask >> pp) & 1u) ? __ldg(share + (size_t)u * B + c0) : 0.0;
                        }
                        // the term of position j: the lower half holds 2j'
                        // and receives 2j'+1 from the upper half, so its sum
                        // runs in position order (the upper half's is unused)
                        double od = 0.0;
                        auto term = [&](int j) -> double {
                            if (j & 1) return od;
                            const double x = v[j >> 1];
                            od = __shfl_xor_sync(0xffffffffu, x, 16);
                            return x;
                        };
                        if (smask == 0) {
#pragma unroll
                            for (int j = 0; j < U; ++j) s[0] = dadd(s[0], term(j));
                        } else {
                            uint32_t m = smask;
                            int k_next = __ffs(m) - 1;
                            m &= m - 1;
                            int pos_next = (int)__shfl_sync(0xffffffffu, p, k_next);
#pragma unroll
                            for (int j = 0; j < U; ++j) {
                                const double t = term(j);
                                if (j == pos_next) {  // warp-uniform
                                    close_row(k_next);
                                    if (m) {
                                        k_next = __ffs(m) - 1;
                                        m &= m - 1;
                                        pos_next = (int)__shfl_sync(0xffffffffu, p, k_next);
                                    } else {
                                        pos_next = U;
                                    }
                                }
                                s[0] = dadd(s[0], t);
                            }
                        }
                    } else if (!PAIR && lmask) {
                        double v[U][CPL];
#pragma unroll
                        for (int j = 0; j < U; ++j) {
                            const uint32_t u = __shfl_sync(0xffffffffu, i0, h * U + j);
                            if ((lmask >> j) & 1u) {
                                ld_cols<CPL>(share + (size_t)u * B + c0, v[j]);
                            } else {
#pragma unroll
                                for (int c = 0; c < CPL; ++c) v[j][c] = 0.0;
                            }
                        }
                        if (smask == 0) {
#pragma unroll
                            for (int j = 0; j < U; ++j)
#pragma unroll
                                for (int c = 0; c < CPL; ++c) s[c] = dadd(s[c], v[j][c]);
                        } else {
                            uint32_t m = smask;
                            int pos_next = U, k_next = 0;
                            if (m) {
                                k_next = __ffs(m) - 1;
                                m &= m - 1;
                                pos_next = (int)__shfl_sync(0xffffffffu, p, k_next);
                            }
#pragma unroll
                            for (int j = 0; j < U; ++j) {
                                if (j == pos_next) {  // warp-uniform
                                    close_row(k_next);
                                    if (m) {
                                        k_next = __ffs(m) - 1;
                                        m &= m - 1;
                                        pos_next = (int)__shfl_sync(0xffffffffu, p, k_next);
                                    } else {
                                        pos_next = U;
                                    }
                                }
#pragma unroll
                                for (int c = 0; c < CPL; ++c) s[c] = dadd(s[c], v[j][c]);
                            }
                        }
                    } else if (smask) {
                        uint32_t m = smask;
                        while (m) {
                            const int k = __ffs(m) - 1;
                            m &= m - 1;
                            close_row(k);
                        }
                    }
                }
                i0 = i1;
                i1 = i2;
                w0 = w1;
            }
        }
        if (is_seg) {
            // publish the segment; the last one of the row combines in order
#pragma unroll
            for (int c = 0; c < CPL; ++c)
                if (keeper) A.seg_part[(size_t)item * B + c0 + c] = s[c];
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
            if (a.acc && ((av >> (r0 & 31)) & 1u)) cp_async_acc<CPL>(tile + c0, a.acc + (size_t)r0 * B + c0);
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        } else if (ne_mask) {
#pragma unroll
            for (int c = 0; c < CPL; ++c)
                if (keeper) yb[cur][c0 + c] = s[c];
        }
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();

        // ---- block epilogue: rows r0 .. r0+nrows-1 ----
        double bl1[CPL], bdm[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) bl1[c] = bdm[c] = 0.0;
        uint32_t nzw = 0, avw = 0;
        // PAIR: the half-warps take alternate rows (16 lanes = 16 columns each)
        constexpr int KS = PAIR ? 2 : 1;
        const uint32_t hmask = PAIR ? (0xffffu << (16 * half)) : 0xffffffffu;
        for (int k0 = 0; k0 < nrows; k0 += KS) {
            const int k = k0 + (PAIR ? half : 0);
            const bool kin = k < nrows;
            const uint32_t r = r0 + k;
            const uint32_t d = __shfl_sync(0xffffffffu, dl, kin ? k : 0);
            const bool valid = kin && ((av >> (r & 31)) & 1u);
            double yy[CPL], ao[CPL];
            bool nzc = false;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                yy[c] = kin ? yb[k][c0 + c] : 0.0;
                if (st[c].has_spread) yy[c] = dadd(yy[c], st[c].spread);  // graph.cpp:265-268
                if (!st[c].active) yy[c] = 0.0;
                ao[c] = valid ? tile[k * TS + c0 + c] : 0.0;
                nzc = nzc || yy[c] != 0.0;
            }
            const bool row_nz = (__ballot_sync(0xffffffffu, nzc) & hmask) != 0;
            if (!kin || (!kLast && !row_nz)) continue;  // nothing changes for this row
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const size_t ix = (size_t)r * B + c0 + c;
                if (!st[c].active) {
                    if (kLast) tile[k * TS + c0 + c] = combine_value(a, ao[c], r);
                    else if (!valid) a.acc[ix] = 0.0;  // the row becomes valid below
                    continue;
                }
                const double f = dadd(ao[c], yy[c]);  // cpi.cpp:50
                if (kLast) {
                    tile[k * TS + c0 + c] = combine_value(a, f, r);  // tpa.cpp:73-74
                } else {
                    const double sh = d ? ddiv(dmul(a.keep, yy[c]), (double)d) : 0.0;  // graph.cpp:222
                    a.acc[ix] = f;
                    a.share_out[ix] = sh;
                }
                bl1[c] = dadd(bl1[c], fabs(yy[c]));
                if (want_dm && d == 0) bdm[c] = dadd(bdm[c], yy[c]);
            }
            nzw |= (row_nz ? 1u : 0u) << (r & 31);
            avw |= 1u << (r & 31);
        }
        if (PAIR) {
            nzw |= __shfl_xor_sync(0xffffffffu, nzw, 16);
            avw |= __shfl_xor_sync(0xffffffffu, avw, 16);
        }
        if (kLast) {
            __syncwarp();
            if (a.out_node_major) {
                for (int k = 0; k < nrows; ++k)
#pragma unroll
                    for (int c = 0; c < CPL; ++c)
                        if (c0 + c < (int)a.b_valid) a.out[(size_t)(r0 + k) * B + c0 + c] = tile[k * TS + c0 + c];
            } else {
                // transposed: RB lanes x 8 B contiguous of one seed's vector per store
                const int k = lane % RB;
                for (uint32_t b = lane / RB; b < a.b_valid; b += 32 / RB)
                    if (k < nrows) a.out[(size_t)b * a.n + r0 + k] = tile[k * TS + b];
            }
            __syncwarp();
        }
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            if (bl1[c] != 0.0) fx_add(fx[0][c], fx[1][c], bl1[c]);
            if (bdm[c] != 0.0) fx_add(fx[2][c], fx[3][c], bdm[c]);
        }
        if (lane == 0 && !kLast) {
            if (A.nz_out && nzw) atomicOr(A.nz_out + (r0 >> 5), nzw);
            if (A.acc_valid && avw) atomicOr(A.acc_valid + (r0 >> 5), avw);
        }
        __syncwarp();
    }

    // residual / dangling mass: exact integer sums; the last CTA advances state
    __syncthreads();  // every warp is done with its tile: s_fx may overlay it
    for (int i = tid; i < 4 * B; i += Sh::NT) s_fx[i] = 0ull;
    __syncthreads();
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int b = c0 + c;
        if (fx[0][c] | fx[1][c]) fx_atomic_add(&s_fx[4 * b + 0], &s_fx[4 * b + 1], fx[0][c], fx[1][c]);
        if (fx[2][c] | fx[3][c]) fx_atomic_add(&s_fx[4 * b + 2], &s_fx[4 * b + 3], fx[2][c], fx[3][c]);
    }
    __syncthreads();
    for (int b = tid; b < B; b += Sh::NT) {
        if (s_fx[4 * b + 0] | s_fx[4 * b + 1]) fx_atomic_add(&A.fx[4 * b + 0], &A.fx[4 * b + 1], s_fx[4 * b + 0], s_fx[4 * b + 1]);
        if (s_fx[4 * b + 2] | s_fx[4 * b + 3]) fx_atomic_add(&A.fx[4 * b + 2], &A.fx[4 * b + 3], s_fx[4 * b + 2], s_fx[4 * b + 3]);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_ticket = atomicAdd(a.done_cnt, 1u);
    __syncthreads();
    if (s_ticket != gridDim.x - 1) return;
    __threadfence();
    for (int b = tid; b < B; b += Sh::NT) {
        ColState sc = a.state_in[b];
        const unsigned long long h0 = atomicAdd(&A.fx[4 * b + 0], 0ull), l0 = atomicAdd(&A.fx[4 * b + 1], 0ull);
        const unsigned long long h1 = atomicAdd(&A.fx[4 * b + 2], 0ull), l1 = atomicAdd(&A.fx[4 * b + 3], 0ull);
        if (A.limbs_out) {  // a partition's totals: summed over partitions by k_part_finalize_b
            fx_to_limbs(h0, l0, A.limbs_out + 6 * b);
            fx_to_limbs(h1, l1, A.limbs_out + 6 * b + 3);
            A.fx[4 * b + 0] = A.fx[4 * b + 1] = A.fx[4 * b + 2] = A.fx[4 * b + 3] = 0ull;
            continue;
        }
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
