// cpi_spmm4.cuh -- K3 v4: the B-seed sweep as two lean kernels (B = 32, 64).
//
// Measured on the B200 (tools/gather_micro.cu): random 256-B row gathers run at
// 0.73 ms per 16.6 M gathers with 16 warps/SM but 0.35 ms with 48 warps/SM
// (~12 TB/s through L2), whatever the bytes per gather.  The fused sweep (v2)
// holds too much per-warp state for that occupancy, so v4 splits it:
//
//   k_mm_gather<B>  y[v][:] = sum over in-neighbours u (ascending) of share[u][:]
//                   -- lane = column, 16 gathers in flight per warp, a flat nnz
//                   stream per work item with indices loaded two chunks ahead
//                   and frontier words one chunk ahead, strictly sequential
//                   per-row sums (bitwise the reference's scatter order for
//                   rows <= kLong; longer rows: kLong-nnz segments combined in
//                   order by the last one), ~40 registers.  Rows whose sums are
//                   zero in every column are not written; ybits marks the rest.
//   k_mm_epi<B>     per (row, column), fully coalesced: + Uniform spread,
//                   acc += y, share_out = keep*y/deg, or the fused combine
//                   out = (1+nsf)*acc + stranger; frontier / acc_valid bitmaps;
//                   fixed-point residual + dangling mass; last CTA advances the
//                   per-column state (cpi.cpp:73-80).
#pragma once

#include "cpi_spmm.cuh"

namespace tpa {

template <int B>
struct Mm4 {
    static_assert(B == 32 || B == 64, "v4: one warp per row group");
    static constexpr int CPL = B / 32;
    static constexpr int U = 16 / CPL;   // gathers in flight per lane (16 x 256 B per warp)
    static constexpr int RB = 32;        // rows per block window (one bitmap word)
    static constexpr int NT = 256;
};

struct Mm4Args {
    MmArgs m;               // graph, state, bitmaps, segments, reduction (reused)
    double* __restrict__ Y; // [n][B] row sums
    uint32_t* __restrict__ ybits;  // rows of Y written (nonzero), pre-zeroed
    const uint8_t* __restrict__ rowflag;   // rows that can be nonzero (sparse sweeps), or null
    const int* dense;                      // set by k_mark_out when the frontier is too big
    const uint2* __restrict__ blocks_rb;   // v5: blocks of <= Mm5<B>::RB rows
    uint32_t n_blocks_rb;
    // v5 sparse sweeps: the RB-row windows holding a marked row (appended by
    // k_mark_out) and each window's first block (prefix, n_windows + 1)
    const uint32_t* __restrict__ wl;
    const uint32_t* wl_cnt;
    const uint32_t* __restrict__ win_blk;
    const uint32_t* __restrict__ sl;  // segments of the marked long rows
    const uint32_t* sl_cnt;
};

// Direction-optimised sparse sweeps.  A frontier row is a row of share_in
// that is not all-zero (nz bitmap).  k_frontier_cost sums the frontier's
// out-degrees; if the push would touch at most `limit` edges, k_mark_out sets
// rowflag[v] = 1 for every out-neighbour v of the frontier (plain byte stores:
// idempotent, no atomics), otherwise it flags the sweep dense.  A row left
// unmarked has no live in-neighbour, so its pull sum is exactly zero and the
// gather kernel skips it.  One warp per 32-row frontier word.
__global__ void __launch_bounds__(256) k_frontier_cost(const uint32_t* __restrict__ nz, uint32_t n_words,
                                                       const uint64_t* __restrict__ out_off,
                                                       unsigned long long* cost, const ColState* __restrict__ st,
                                                       int B, unsigned long long limit) {
    const int lane = threadIdx.x & 31;
    // a Uniform spread reaches every row (graph.cpp:265-268): no sparse pull then
#ifndef TPA_NO_SPREAD_GUARD  // (A/B only: reproduces the unguarded decision)
    if (blockIdx.x == 0 && (int)threadIdx.x < B && st[threadIdx.x].active && st[threadIdx.x].has_spread)
        atomicAdd(cost, 1ull << 62);
#endif
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    unsigned long long c = 0;
    uint32_t k = 0;
    for (uint32_t w = gw; w < n_words; w += nw, ++k) {
        // a dense frontier: stop once the running total is past the limit
        if ((k & 7) == 7) {
            const int over = lane == 0 && *reinterpret_cast<volatile unsigned long long*>(cost) > limit;
            if (__shfl_sync(0xffffffffu, over, 0)) break;  // warp-uniform
        }
        const uint32_t bits = __ldg(nz + w);
        if ((bits >> lane) & 1u) {
            const uint32_t u = w * 32 + lane;
            c += __ldg(out_off + u + 1) - __ldg(out_off + u);
        }
        if ((k & 7) == 7) {  // publish the partial total every 8 words
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if (lane == 0 && c) atomicAdd(cost, c);
            c = 0;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0 && c) atomicAdd(cost, c);
}

struct MarkArgs {
    const uint32_t* __restrict__ nz;
    uint32_t n_words;
    const uint64_t* __restrict__ out_off;
    const uint32_t* __restrict__ out_tgt;
    const unsigned long long* cost;
    unsigned long long limit;
    uint8_t* rowflag;
    int* dense;
    uint32_t* wbits;    // marked windows (bitmap), zeroed
    uint32_t* wl;       // marked windows (list), or null: no list
    uint32_t* wl_cnt;
    int rb_shift;       // window = row >> rb_shift
    ulonglong2* chunks;   // edge ranges [lo, hi) of <= kMarkChunk out-edges of big frontier rows
    uint32_t* chunk_cnt;  // zeroed
};

constexpr uint32_t kMarkInline = 32;   // frontier rows with more out-edges are chunked
constexpr uint32_t kMarkChunk = 128;   // one warp, 4 loads per lane in flight
// chunk list capacity for a graph of m edges (any push limit <= m)
__host__ __device__ constexpr size_t mark_chunk_cap(uint64_t m) { return m / kMarkChunk + m / kMarkInline + 2; }

__device__ __forceinline__ void mark_row(const MarkArgs& M, uint32_t t) {
    M.rowflag[t] = 1;
    if (M.wl) {  // the first marker of a window appends it to the work list
        const uint32_t wdx = t >> M.rb_shift, bit = 1u << (wdx & 31);
        if (!(__ldcg(M.wbits + (wdx >> 5)) & bit) && !(atomicOr(M.wbits + (wdx >> 5), bit) & bit))
            M.wl[atomicAdd(M.wl_cnt, 1u)] = wdx;
    }
}

// Marks the out-neighbours of frontier rows with <= kMarkInline out-edges
// (one warp per frontier word, one edge per lane) and cuts the edge lists of
// the others into kMarkChunk-edge chunks for k_mark_big, which spreads them
// over all warps of its grid (a hub's 100k out-edges no longer serialise on
// one warp).
__global__ void __launch_bounds__(256) k_mark_out(MarkArgs M) {
    if (*M.cost > M.limit) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *M.dense = 1;
        return;
    }
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w = gw; w < M.n_words; w += nw) {
        uint32_t bits = __ldg(M.nz + w);
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const uint32_t u = w * 32 + b;
            const uint64_t lo = __ldg(M.out_off + u), hi = __ldg(M.out_off + u + 1);
            if (hi - lo > kMarkInline) {
                const uint32_t nch = (uint32_t)((hi - lo + kMarkChunk - 1) / kMarkChunk);
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(M.chunk_cnt, nch);
                base = __shfl_sync(0xffffffffu, base, 0);
                for (uint32_t c = lane; c < nch; c += 32)
                    M.chunks[base + c] = make_ulonglong2(lo + (uint64_t)c * kMarkChunk,
                                                         min(hi, lo + (uint64_t)(c + 1) * kMarkChunk));
                continue;
            }
            if (lo + lane < hi) mark_row(M, __ldg(M.out_tgt + lo + lane));
        }
    }
}

// Sparse sweep work list, part 2: the segments of every marked long row.
__global__ void __launch_bounds__(256) k_long_list(MarkArgs M, const uint32_t* __restrict__ seg_row,
                                                   const uint32_t* __restrict__ long_first,
                                                   const uint32_t* __restrict__ long_nseg, uint32_t n_long,
                                                   uint32_t* sl, uint32_t* sl_cnt) {
    if (*M.cost > M.limit) return;
    for (uint32_t li = blockIdx.x * blockDim.x + threadIdx.x; li < n_long; li += gridDim.x * blockDim.x) {
        const uint32_t f = long_first[li];
        if (!M.rowflag[seg_row[f]]) continue;
        const uint32_t ns = long_nseg[li];
        const uint32_t base = atomicAdd(sl_cnt, ns);
        for (uint32_t j = 0; j < ns; ++j) sl[base + j] = f + j;
    }
}

// The chunked edge lists: one warp per chunk, 4 loads per lane in flight.
__global__ void __launch_bounds__(256) k_mark_big(MarkArgs M) {
    if (*M.cost > M.limit) return;
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nc = *M.chunk_cnt;
    for (uint32_t q = gw; q < nc; q += nw) {
        const ulonglong2 r = M.chunks[q];
        uint32_t t[kMarkChunk / 32];
#pragma unroll
        for (int j = 0; j < (int)(kMarkChunk / 32); ++j) {
            const uint64_t e = r.x + j * 32 + lane;
            t[j] = e < r.y ? __ldg(M.out_tgt + e) : 0xffffffffu;
        }
#pragma unroll
        for (int j = 0; j < (int)(kMarkChunk / 32); ++j)
            if (t[j] != 0xffffffffu) mark_row(M, t[j]);
    }
}

template <int B>
__global__ void __launch_bounds__(Mm4<B>::NT, 5) k_mm_gather(Mm4Args P) {
    constexpr int CPL = Mm4<B>::CPL, U = Mm4<B>::U;
    const MmArgs& A = P.m;
    const StepArgs& a = A.s;
    const int lane = threadIdx.x & 31;
    const int c0 = lane * CPL;
    const uint32_t* __restrict__ col = a.col;
    const uint32_t* __restrict__ nz = A.nz_in;
    const double* __restrict__ share = a.share_in;
    const uint32_t total = A.n_segs + A.n_blocks;

    const bool use_mask = P.rowflag != nullptr && *P.dense == 0;
    uint32_t next_item = 0;
    if (lane == 0) next_item = atomicAdd(A.work_cnt, 1u);
    for (;;) {
        const uint32_t item = __shfl_sync(0xffffffffu, next_item, 0);
        if (item >= total) break;
        if (lane == 0) next_item = atomicAdd(A.work_cnt, 1u);
        const bool is_seg = item < A.n_segs;
        uint32_t r0;
        int nrows;
        int64_t rpl;  // lane k: row_ptr[r0 + k] (k <= nrows)
        if (use_mask) {
            // sparse sweep: skip items whose rows cannot receive anything
            // (a long row is marked or not as a whole, so either all of its
            // segments run -- and the last one finishes it -- or none does)
            const uint32_t rr = is_seg ? A.seg_row[item] : A.blocks[item - A.n_segs].x;
            const uint32_t nrr = is_seg ? 1u : A.blocks[item - A.n_segs].y;
            const bool mk = lane < (int)nrr && P.rowflag[rr + lane];
            if (!__any_sync(0xffffffffu, mk)) continue;
        }
        if (is_seg) {
            r0 = A.seg_row[item];
            nrows = 1;
            const int64_t lo = A.seg_lo[item];
            const int64_t hi = min(lo + (int64_t)kLong, (int64_t)__ldg(a.row_ptr + r0 + 1));
            rpl = lane == 0 ? lo : hi;
        } else {
            const uint2 blk = A.blocks[item - A.n_segs];
            r0 = blk.x;
            nrows = (int)blk.y;
            rpl = lane <= nrows ? __ldg(a.row_ptr + r0 + lane) : 0;
        }
        const int64_t e0 = __shfl_sync(0xffffffffu, rpl, 0);
        const int64_t e1 = __shfl_sync(0xffffffffu, rpl, nrows);
        // next non-empty row start of every row boundary, as stream positions:
        // lane k (1 <= k < nrows) starts a non-empty row at rp[k] if rp[k+1] > rp[k]
        const int64_t rpn = __shfl_down_sync(0xffffffffu, rpl, 1);
        const bool starts = !is_seg && lane >= 1 && lane < nrows && rpn > rpl && rpl > e0;
        double s[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) s[c] = 0.0;
        // current (non-empty) row: the first row with rp[k+1] > e0
        const uint32_t ne_mask = __ballot_sync(0xffffffffu, lane < nrows && rpn > rpl);
        int cur = ne_mask ? __ffs(ne_mask) - 1 : 0;
        uint32_t ybits_w = 0;  // rows of this block written to Y
        bool any_live = false;

        auto idx_at = [&](int64_t base) -> uint32_t {
            const int64_t e = base + lane;
            return (lane < U && e < e1) ? ld_stream_u32(col + e) : 0u;
        };
        auto bits_at = [&](uint32_t u, int64_t base) -> uint32_t {
            return (nz && lane < U && base + lane < e1) ? __ldg(nz + (u >> 5)) : 0xffffffffu;
        };
        auto close_row = [&](int k_next) {
            // y of row `cur` is final: write it if nonzero in any column
            bool nzc = false;
#pragma unroll
            for (int c = 0; c < CPL; ++c) nzc = nzc || s[c] != 0.0;
            if (__any_sync(0xffffffffu, nzc)) {
                double* dst = P.Y + (size_t)(r0 + cur) * B + c0;
                if constexpr (CPL == 1) {
                    dst[0] = s[0];
                } else {
                    *reinterpret_cast<double2*>(dst) = make_double2(s[0], s[1]);
                }
                ybits_w |= 1u << ((r0 + cur) & 31);
            }
#pragma unroll
            for (int c = 0; c < CPL; ++c) s[c] = 0.0;
            cur = k_next;
        };

        if (e1 > e0) {
            uint32_t i0 = idx_at(e0), i1 = idx_at(e0 + U);
            uint32_t w0 = bits_at(i0, e0);
            for (int64_t base = e0; base < e1; base += U) {
                const uint32_t i2 = idx_at(base + 2 * U);  // two chunks ahead
                const uint32_t w1 = bits_at(i1, base + U);  // one chunk ahead
                const bool live = (w0 >> (i0 & 31)) & 1u;
                const uint32_t lmask = __ballot_sync(0xffffffffu, live && lane < U && base + lane < e1);
                // row starts inside [base, base+U): positions p = rp[k] - base
                const int64_t p = rpl - base;
                const uint32_t smask =
                    __ballot_sync(0xffffffffu, starts && p >= 0 && p < U);  // lanes k whose row starts here
                if (lmask) {
                    any_live = true;
                    double v[U][CPL];
#pragma unroll
                    for (int j = 0; j < U; ++j) {
                        const uint32_t u = __shfl_sync(0xffffffffu, i0, j);
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
                        // positions of the starts, in order (rows start at
                        // increasing positions, one row per start)
                        uint32_t m = smask;
                        int pos_next = 0, k_next = 0;
                        auto next_start = [&] {
                            if (m) {
                                k_next = __ffs(m) - 1;
                                m &= m - 1;
                                pos_next = (int)(__shfl_sync(0xffffffffu, p, k_next));
                            } else {
                                pos_next = U;
                            }
                        };
                        next_start();
#pragma unroll
                        for (int j = 0; j < U; ++j) {
                            if (j == pos_next) {  // warp-uniform
                                close_row(k_next);
                                next_start();
                            }
#pragma unroll
                            for (int c = 0; c < CPL; ++c) s[c] = dadd(s[c], v[j][c]);
                        }
                    }
                } else if (smask) {
                    // dead chunk: sums unchanged (+0.0); only row ends happen
                    uint32_t m = smask;
                    while (m) {
                        const int k = __ffs(m) - 1;
                        m &= m - 1;
                        close_row(k);
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
                s[c] = y;
            }
            if (lane == 0) A.long_cnt[li] = 0;
            cur = 0;
            close_row(0);
        } else if (any_live && ne_mask) {
            close_row(0);  // the block's last non-empty row
        }
        if (lane == 0 && ybits_w) atomicOr(P.ybits + (r0 >> 5), ybits_w);
    }
    // last warp out resets the work counter for the next sweep
    __syncwarp();
    if (lane == 0) {
        __threadfence();
        const uint32_t nw = gridDim.x * (blockDim.x >> 5);
        if (atomicAdd(a.done_cnt, 1u) == nw - 1) {
            *A.work_cnt = 0;
            *a.done_cnt = 0;
        }
    }
}

// Epilogue: one warp per 32-row window, lane = column; rows of the window in
// order, loads batched 4 rows deep.  Writes only what changes.
template <int B>
__global__ void __launch_bounds__(Mm4<B>::NT) k_mm_epi(Mm4Args P) {
    constexpr int CPL = Mm4<B>::CPL;
    constexpr int TP = B + 1;  // padded tile row (doubles): 2-way bank pattern
    const MmArgs& A = P.m;
    const StepArgs& a = A.s;
    // seed-major combine output is staged per 32-row window and written
    // transposed: each store instruction then writes 256 contiguous bytes
    extern __shared__ __align__(16) double s_tile[];
    __shared__ ColState s_st[B];
    __shared__ unsigned long long s_fx[4 * B];
    __shared__ uint32_t s_ticket;
    const int tid = threadIdx.x, lane = tid & 31;
    const int c0 = lane * CPL;
    for (int i = tid; i < 4 * B; i += blockDim.x) s_fx[i] = 0ull;
    for (int b = tid; b < B; b += blockDim.x) s_st[b] = a.state_in[b];
    __syncthreads();
    ColState st[CPL];
    bool any_spread = false;
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        st[c] = s_st[c0 + c];
        any_spread = any_spread || (st[c].active && st[c].has_spread);
    }
    any_spread = __any_sync(0xffffffffu, any_spread);
    const bool want_dm = a.policy == kUniform;
    const bool write_acc = a.acc != nullptr && a.out == nullptr;
    unsigned long long fx[4][CPL];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < CPL; ++c) fx[q][c] = 0ull;

    const bool stage_out = a.out != nullptr && !a.out_node_major;
    double* tile = s_tile + (size_t)(tid >> 5) * 32 * TP;
    const uint32_t nwin = (a.n + 31) / 32;
    const uint32_t gw = (blockIdx.x * blockDim.x + tid) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t wdx = gw; wdx < nwin; wdx += nwarps) {
        const uint32_t r0 = wdx * 32;
        const int nr = (int)min(32u, a.n - r0);
        const uint32_t yb = __ldg(P.ybits + wdx);
        const uint32_t av = A.acc_valid ? A.acc_valid[wdx] : 0xffffffffu;
        // rows that need work: a written y, a spread, or a pending combine
        uint32_t todo = (any_spread || a.out) ? (nr == 32 ? 0xffffffffu : ((1u << nr) - 1u)) : yb;
        const uint32_t dl = lane < nr ? __ldg(a.deg + r0 + lane) : 0u;
        double bl1[CPL], bdm[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) bl1[c] = bdm[c] = 0.0;
        uint32_t nzw = 0, avw = 0;
        while (todo) {
            // up to 4 rows per round: all loads first
            int ks[4];
            double yv[4][CPL], ao[4][CPL];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                ks[q] = todo ? __ffs(todo) - 1 : -1;
                if (todo) todo &= todo - 1;
                if (ks[q] >= 0) {
                    const size_t ix = (size_t)(r0 + ks[q]) * B + c0;
                    const bool hy = (yb >> ks[q]) & 1u;
                    const bool va = a.acc && ((av >> ks[q]) & 1u);
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        yv[q][c] = hy ? P.Y[ix + c] : 0.0;
                        ao[q][c] = va ? a.acc[ix + c] : 0.0;
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = ks[q];
                if (k < 0) continue;
                const uint32_t r = r0 + k;
                const uint32_t d = __shfl_sync(0xffffffffu, dl, k);
                bool row_nz = false;
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    const uint32_t b = c0 + c;
                    const size_t ix = (size_t)r * B + b;
                    if (!st[c].active) {
                        if (a.out) {
                            const double o = combine_value(a, ao[q][c], r);
                            if (stage_out) tile[k * TP + b] = o;
                            else if (b < a.b_valid) a.out[ix] = o;
                        } else if (write_acc && !((av >> k) & 1u)) {
                            a.acc[ix] = 0.0;  // row becomes valid below: keep the column's zero
                        }
                        continue;
                    }
                    double yy = yv[q][c];
                    if (st[c].has_spread) yy = dadd(yy, st[c].spread);  // graph.cpp:265-268
                    row_nz = row_nz || yy != 0.0;
                    if (a.acc) {
                        const double f = dadd(ao[q][c], yy);  // cpi.cpp:50
                        if (a.out) {
                            const double o = combine_value(a, f, r);
                            if (stage_out) tile[k * TP + b] = o;
                            else if (b < a.b_valid) a.out[ix] = o;
                        } else {
                            a.acc[ix] = f;
                        }
                    }
                    if (a.share_out) a.share_out[ix] = d ? ddiv(dmul(a.keep, yy), (double)d) : 0.0;  // graph.cpp:222
                    bl1[c] = dadd(bl1[c], fabs(yy));
                    if (want_dm && d == 0) bdm[c] = dadd(bdm[c], yy);
                }
                const bool rn = __any_sync(0xffffffffu, row_nz);
                nzw |= (rn ? 1u : 0u) << k;
                avw |= 1u << k;
            }
        }
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            if (bl1[c] != 0.0) fx_add(fx[0][c], fx[1][c], bl1[c]);
            if (bdm[c] != 0.0) fx_add(fx[2][c], fx[3][c], bdm[c]);
        }
        if (stage_out) {
            __syncwarp();
            if (lane < nr)
                for (uint32_t b = 0; b < a.b_valid; ++b) a.out[(size_t)b * a.n + r0 + lane] = tile[lane * TP + b];
            __syncwarp();
        }
        if (lane == 0) {
            if (A.nz_out) A.nz_out[wdx] = nzw;                   // whole word: this warp owns it
            if (A.acc_valid && write_acc) A.acc_valid[wdx] = av | avw;
        }
    }
    // residual / dangling mass: exact integer sums, then the last CTA decides
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int b = c0 + c;
        if (fx[0][c] | fx[1][c]) fx_atomic_add(&s_fx[4 * b + 0], &s_fx[4 * b + 1], fx[0][c], fx[1][c]);
        if (fx[2][c] | fx[3][c]) fx_atomic_add(&s_fx[4 * b + 2], &s_fx[4 * b + 3], fx[2][c], fx[3][c]);
    }
    __syncthreads();
    for (int b = tid; b < B; b += blockDim.x) {
        if (s_fx[4 * b + 0] | s_fx[4 * b + 1]) fx_atomic_add(&A.fx[4 * b + 0], &A.fx[4 * b + 1], s_fx[4 * b + 0], s_fx[4 * b + 1]);
        if (s_fx[4 * b + 2] | s_fx[4 * b + 3]) fx_atomic_add(&A.fx[4 * b + 2], &A.fx[4 * b + 3], s_fx[4 * b + 2], s_fx[4 * b + 3]);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_ticket = atomicAdd(a.done_cnt, 1u);
    __syncthreads();
    if (s_ticket != gridDim.x - 1) return;
    __threadfence();
    for (int b = tid; b < B; b += blockDim.x) {
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
    if (tid == 0) *a.done_cnt = 0;
}

}  // namespace tpa
