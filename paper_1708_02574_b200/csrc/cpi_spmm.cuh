// cpi_spmm.cuh -- K3 v2: fused CPI sweep over B seeds (SpMM), persistent.
//
// Replaces, for B independent single-seed series at once, the reference's
// propagation_sweep + l1_sum + add_into + run_series step (graph.cpp:211-270,
// cpi.cpp:43-83) and the query combine (tpa.cpp:70-74).
//
// Layout: iterate (as shares, see cpi_kernels.cuh) row-major [n][B] fp64, so a
// gather of source u is B*8 contiguous bytes; lane = column (G = min(B,32)
// lanes per row group, CPL = B/G columns per lane).
//
// Work: a persistent grid; every group of G lanes pulls work items from one
// atomic counter: first the segments of long rows (in-degree > kLong, longest
// first), then blocks of consecutive short rows (<= 16 rows inside one aligned
// 16-row window, <= kBlockNnz nnz), so no item is much longer than another.  Inside a block the group walks the nnz of its
// rows as ONE flat stream in chunks of U (so gathers stay U-deep whatever the
// row lengths), with the chunk's indices loaded two chunks ahead and the
// frontier-bitmap words one chunk ahead (software pipeline).  Per column,
// every row <= kLong is summed strictly sequentially in ascending source
// order: bitwise the reference's scatter order.  Long rows: fixed kLong-nnz
// segments, each sequential, combined in segment order by the last segment
// to finish.
//
// Sparse frontier (query batches): nz_in marks rows of share_in that are not
// all-zero; gathers of zero rows are skipped (adding +0.0 is the identity, so
// results are unchanged).  Rows whose new value is zero in every column write
// nothing; nz_out / acc_valid bitmaps record what was written, so x^(0) needs
// no dense zero-fill and early (sparse) sweeps move only the frontier's bytes.
//
// Residual L1 and dangling mass: per lane 128-bit fixed-point accumulators
// (exact integer adds, so the total does not depend on which group handled
// which block) -> one atomic per CTA per column -> the last CTA decodes them
// and advances the per-column state (cpi.cpp:73-80).
#pragma once

#include "cpi_kernels.cuh"

namespace tpa {

constexpr int kMmRows = 16;  // a block lies inside one aligned kMmRows-row window
constexpr int kLong = 512;      // rows above: cut into kLong-nnz segments
constexpr int kBlockNnz = 512;  // nnz cap of a block (bounds the longest work item)
constexpr int kU = 8;           // stream chunk (positions); gathers per chunk = kU

struct MmArgs {
    StepArgs s;                           // shared fields (graph, buffers, state)
    const uint32_t* __restrict__ nz_in;   // bitmap over share_in rows, or null (dense)
    uint32_t* __restrict__ nz_out;        // bitmap over share_out rows (pre-zeroed), or null
    uint32_t* __restrict__ acc_valid;     // rows of acc holding data, or null (acc dense)
    // long rows
    const uint32_t* __restrict__ seg_row;     // [n_segs] row of the segment
    const int64_t* __restrict__ seg_lo;       // [n_segs] nnz begin (end = min(lo+kLong, row end))
    const uint32_t* __restrict__ seg_long;    // [n_segs] long-row index
    const uint32_t* __restrict__ long_first;  // [n_long] first segment index
    const uint32_t* __restrict__ long_nseg;   // [n_long]
    uint32_t* __restrict__ long_cnt;          // [n_long] arrival counters (zero between launches)
    double* __restrict__ seg_part;            // [n_segs][B]
    const uint2* __restrict__ blocks;         // [n_blocks] {first row, row count}
    uint32_t n_segs;
    uint32_t n_blocks;
    uint32_t zero_row;                        // = n: an all-zero row of every share buffer
    // scheduling / reduction
    uint32_t* work_cnt;       // zero between launches
    unsigned long long* fx;   // [4B]: l1 hi/lo, dm hi/lo per column; zero between launches
    // row partition (tpa_part.cuh): the last CTA publishes the sweep's exact
    // totals as limbs [B][6] here and leaves the state to k_part_finalize_b
    unsigned long long* limbs_out;
};

// ---- 128-bit fixed point (value = hi*2^-56 + lo*2^-120), for y in [0, 2^7) --
__device__ __forceinline__ void fx_add(unsigned long long& hi, unsigned long long& lo, double y) {
    double t = dmul(fabs(y), 0x1p56);
    t = fmin(t, 0x1p62);
    const unsigned long long h = __double2ull_rz(t);
    const double r = t - (double)h;  // exact
    const unsigned long long l = __double2ull_rz(dmul(r, 0x1p64));
    lo += l;
    hi += h + (lo < l ? 1ull : 0ull);
}

// Sum of a long row's segment partials p[0], p[stride], ... in segment order
// (the fixed combine order), with 8 L2 loads in flight instead of a chain of
// dependent round trips (a 40k-nnz row has ~80 segments).
__device__ __forceinline__ double seg_sum(const double* p, size_t stride, uint32_t ns) {
    double y = __ldcg(p);
    uint32_t j = 1;
    for (; j + 8 <= ns; j += 8) {
        double t[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) t[k] = __ldcg(p + (size_t)(j + k) * stride);
#pragma unroll
        for (int k = 0; k < 8; ++k) y = dadd(y, t[k]);
    }
    for (; j < ns; ++j) y = dadd(y, __ldcg(p + (size_t)j * stride));
    return y;
}

// 128-bit fixed-point totals as three limbs each (hi, lo >> 32, lo & 2^32-1):
// limb-wise integer sums over up to 2^31 partitions cannot overflow, and
// limbs_to_fx restores the exact 128-bit total (NCCL all-reduce of uint64).
__device__ __forceinline__ void fx_to_limbs(unsigned long long hi, unsigned long long lo, unsigned long long* L) {
    L[0] = hi;
    L[1] = lo >> 32;
    L[2] = lo & 0xffffffffull;
}
__device__ __forceinline__ void limbs_to_fx(const unsigned long long* L, unsigned long long& hi,
                                            unsigned long long& lo) {
    const unsigned long long t2 = L[2];
    const unsigned long long t1 = L[1] + (t2 >> 32);
    lo = ((t1 & 0xffffffffull) << 32) | (t2 & 0xffffffffull);
    hi = L[0] + (t1 >> 32);
}

__device__ __forceinline__ double fx_decode(unsigned long long hi, unsigned long long lo) {
    return dadd((double)hi * 0x1p-56, (double)lo * 0x1p-120);
}

__device__ __forceinline__ void fx_atomic_add(unsigned long long* p_hi, unsigned long long* p_lo,
                                              unsigned long long hi, unsigned long long lo) {
    const unsigned long long old = atomicAdd(p_lo, lo);
    const unsigned long long carry = (old + lo < old) ? 1ull : 0ull;
    if (hi + carry) atomicAdd(p_hi, hi + carry);
}

// Exact warp total of per-lane 128-bit fixed-point values (every lane gets it).
__device__ __forceinline__ void fx_warp_sum(unsigned long long& hi, unsigned long long& lo) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long oh = __shfl_xor_sync(0xffffffffu, hi, o);
        const unsigned long long ol = __shfl_xor_sync(0xffffffffu, lo, o);
        const unsigned long long l2 = lo + ol;
        hi += oh + (l2 < lo ? 1ull : 0ull);
        lo = l2;
    }
}

// CTA total of per-thread (l1, dm) fixed-point pairs added into the global
// fx[4] (warp shuffles, then one thread; no shared-memory atomics).  Every
// thread of the CTA must call it.  s_w: >= 4 * (blockDim.x / 32) words.
__device__ __forceinline__ void fx_cta_flush(unsigned long long f0, unsigned long long f1, unsigned long long f2,
                                             unsigned long long f3, unsigned long long* s_w,
                                             unsigned long long* fx) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    fx_warp_sum(f0, f1);
    fx_warp_sum(f2, f3);
    if (lane == 0) {
        s_w[4 * w + 0] = f0;
        s_w[4 * w + 1] = f1;
        s_w[4 * w + 2] = f2;
        s_w[4 * w + 3] = f3;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long h0 = 0, l0 = 0, h1 = 0, l1 = 0;
        for (int k = 0; k < nw; ++k) {
            unsigned long long t = l0 + s_w[4 * k + 1];
            h0 += s_w[4 * k + 0] + (t < l0 ? 1ull : 0ull);
            l0 = t;
            t = l1 + s_w[4 * k + 3];
            h1 += s_w[4 * k + 2] + (t < l1 ? 1ull : 0ull);
            l1 = t;
        }
        if (fx) {
            if (h0 | l0) fx_atomic_add(&fx[0], &fx[1], h0, l0);
            if (h1 | l1) fx_atomic_add(&fx[2], &fx[3], h1, l1);
        } else {  // no target: the CTA totals stay in s_w[0..3] (thread 0)
            s_w[0] = h0;
            s_w[1] = l0;
            s_w[2] = h1;
            s_w[3] = l1;
        }
    }
}


template <int B>
struct MmShape {
    static constexpr int G = MmVec<B>::G, CPL = MmVec<B>::CPL;
    static constexpr int NGRP = 8;            // row groups per CTA
    static constexpr int NT = NGRP * G;       // CTA size (64 / 128 / 256 threads)
    static constexpr int IPL = kU > G ? kU / G : 1;  // chunk indices held per lane
    static constexpr int DPL = (kMmRows + G - 1) / G;  // row degrees held per lane
    // per group: row sums (kMmRows x B) + a work area shared by the staged
    // indices (stream phase) and the prefetched accumulator rows (epilogue)
    static constexpr size_t kYBytes = (size_t)kMmRows * B * sizeof(double);
    static constexpr size_t kWBytes = kYBytes > kBlockNnz * 4 ? kYBytes : (size_t)kBlockNnz * 4;
    static constexpr size_t kDynSmem = (size_t)NGRP * (kYBytes + kWBytes);
};

// Lanes of this lane's group (G consecutive lanes).  Groups of one warp may be
// at different points of their work, so every warp-level primitive below
// names only the group's lanes.
template <int G>
__device__ __forceinline__ uint32_t group_mask() {
    if constexpr (G == 32) {
        return 0xffffffffu;
    } else {
        return ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
    }
}

template <int G>
__device__ __forceinline__ uint32_t gshfl(uint32_t v, int src) {
    return __shfl_sync(group_mask<G>(), v, src, G);
}

// Stages the item's source indices into shared memory.  A source whose row
// is all-zero in nz_in is replaced by zero_row (an all-zero row kept at index
// n of every share buffer), so the gather loop needs no predication; the
// stream is padded with zero_row to a multiple of kU.  chunk_live gets one bit
// per kU-chunk that holds any live source.  Returns "any live" (group-uniform).
template <int G>
__device__ __forceinline__ bool stage_indices(const MmArgs& A, int64_t lo, int nnz, int gl, uint32_t* sidx,
                                              uint32_t* chunk_live) {
    constexpr int PER = 8;  // positions per lane per pass: index loads, then frontier loads
    const uint32_t* __restrict__ col = A.s.col;
    const uint32_t* __restrict__ nz = A.nz_in;
    const uint32_t gm = group_mask<G>();
    const int lane_base = (threadIdx.x & 31) & ~(G - 1);
    const int padded = (nnz + kU - 1) / kU * kU;
    if (gl < 2) chunk_live[gl] = 0u;
    __syncwarp(gm);
    uint32_t any = 0;
    for (int p0 = 0; p0 < padded; p0 += PER * G) {
        uint32_t u[PER], wbits[PER];
#pragma unroll
        for (int t = 0; t < PER; ++t) {
            const int e = p0 + t * G + gl;
            u[t] = e < nnz ? ld_stream_u32(col + lo + e) : 0u;
        }
#pragma unroll
        for (int t = 0; t < PER; ++t) {
            const int e = p0 + t * G + gl;
            wbits[t] = (nz && e < nnz) ? __ldg(nz + (u[t] >> 5)) : 0xffffffffu;
        }
#pragma unroll
        for (int t = 0; t < PER; ++t) {
            const int e0 = p0 + t * G;
            if (e0 >= padded) break;  // group-uniform
            const int e = e0 + gl;
            const bool live = e < nnz && ((wbits[t] >> (u[t] & 31)) & 1u);
            if (e < padded) sidx[e] = live ? u[t] : A.zero_row;
            const uint32_t bits =
                (__ballot_sync(gm, live) >> lane_base) & (G == 32 ? 0xffffffffu : ((1u << G) - 1u));
            any |= bits;
            if (gl == 0 && bits) {
#pragma unroll
                for (int q = 0; q < (G + kU - 1) / kU; ++q) {
                    const uint32_t part = G >= kU ? (bits >> (q * kU)) & ((1u << kU) - 1u) : bits;
                    if (part) {
                        const int ci = (e0 + q * kU) / kU;
                        chunk_live[ci >> 5] |= 1u << (ci & 31);
                    }
                }
            }
        }
    }
    __syncwarp(gm);
    return any != 0;
}

// Sequential per-row sums over the staged stream.  rs_bits has a bit at every
// position where a new non-empty row starts; close(fin, nb) runs (with nb set)
// before such an element is added.  Per column the additions run in stream
// order = ascending source order, each row starting from 0.0 + first.  The
// gathers of chunk k+1 are issued before chunk k is summed (two chunks in
// flight per group).
template <int B, bool kRows, class Close>
__device__ __forceinline__ void consume_staged(const double* __restrict__ share, const uint32_t* sidx,
                                               const uint32_t* chunk_live, const uint32_t* rs_bits, int nnz,
                                               int c0, double (&s)[MmShape<B>::CPL], Close&& close) {
    constexpr int CPL = MmShape<B>::CPL;
    const int nch = (nnz + kU - 1) / kU;
    auto live = [&](int ci) { return ci < nch && ((chunk_live[ci >> 5] >> (ci & 31)) & 1u); };
    auto issue = [&](int ci, double (&v)[kU][CPL]) {
        if (!live(ci)) return;
        uint32_t w[kU];
        const uint4* p4 = reinterpret_cast<const uint4*>(sidx + ci * kU);
#pragma unroll
        for (int q = 0; q < kU / 4; ++q) {
            const uint4 t = p4[q];
            w[4 * q + 0] = t.x;
            w[4 * q + 1] = t.y;
            w[4 * q + 2] = t.z;
            w[4 * q + 3] = t.w;
        }
#pragma unroll
        for (int j = 0; j < kU; ++j) ld_cols<CPL>(share + (size_t)w[j] * B + c0, v[j]);
    };
    auto consume = [&](int ci, const double (&v)[kU][CPL]) {
        const int base = ci * kU;
        const uint32_t rs = kRows ? (rs_bits[base >> 5] >> (base & 31)) & ((1u << kU) - 1u) : 0u;
        if (!live(ci)) {
            // no live source: sums unchanged (+0.0 each); only row ends happen
            if (kRows) {
                uint32_t m = rs;
                while (m) {
                    m &= m - 1;
                    double fin[CPL];
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        fin[c] = s[c];
                        s[c] = 0.0;
                    }
                    close(fin, true);
                }
            }
            return;
        }
#pragma unroll
        for (int j = 0; j < kU; ++j) {
            if (kRows) {
                const bool nb = (rs >> j) & 1u;
                double fin[CPL];
#pragma unroll
                for (int c = 0; c < CPL; ++c) {
                    fin[c] = s[c];
                    const double t = dadd(s[c], v[j][c]);
                    s[c] = nb ? v[j][c] : t;  // a new row starts from 0.0 + v == v
                }
                close(fin, nb);
            } else {
#pragma unroll
                for (int c = 0; c < CPL; ++c) s[c] = dadd(s[c], v[j][c]);
            }
        }
    };
    // double-buffered chunks: chunk ci+1's gathers are in flight while ci sums
    double va[kU][CPL], vb[kU][CPL];
    issue(0, va);
    for (int ci = 0; ci < nch; ci += 2) {
        issue(ci + 1, vb);
        consume(ci, va);
        if (ci + 1 < nch) {
            issue(ci + 2, va);
            consume(ci + 1, vb);
        }
    }
}

__device__ __forceinline__ double combine_value(const StepArgs& a, double f, uint32_t r) {
    return a.stranger ? dadd(dmul(a.scale, f), a.stranger[r])  // tpa.cpp:73-74
                      : dmul(f, a.scale);                     // tpa.cpp:84
}

// cp.async of one lane's CPL accumulator values (8 or 16 bytes) into smem.
template <int CPL>
__device__ __forceinline__ void cp_async_cols(double* dst_smem, const double* src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst_smem);
    if constexpr (CPL == 1) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
    } else {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
    }
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Epilogue for rows r0 .. r0+nrows-1 (inside one aligned 16-row window) whose
// per-column sums sit in ybuf.
// Phase 1 decides which rows must be written and starts cp.async copies of
// their accumulator rows (all in flight together); phase 2 is one rolled loop.
template <int B>
__device__ __forceinline__ void mm_epilogue_rows(const MmArgs& A, const ColState (&st)[MmShape<B>::CPL],
                                              uint32_t r0, int nrows, const double (*ybuf)[B],
                                              double (*abuf)[B], const uint32_t (&deg_lane)[MmShape<B>::DPL],
                                              int gl, int c0,
                                              unsigned long long (&fx)[4][MmShape<B>::CPL]) {
    constexpr int G = MmShape<B>::G, CPL = MmShape<B>::CPL;
    const StepArgs& a = A.s;
    const uint32_t gm = group_mask<G>();
    const bool want_dm = a.policy == kUniform;
    const bool write_acc = a.acc != nullptr && a.out == nullptr;
    const uint32_t av_word = A.acc_valid ? __ldcg(A.acc_valid + (r0 >> 5)) : 0xffffffffu;
    uint32_t live_rows = 0;
    for (int k = 0; k < nrows; ++k) {
        const uint32_t r = r0 + k;
        bool nzc = false;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            double yy = ybuf[k][c0 + c];
            if (st[c].has_spread) yy = dadd(yy, st[c].spread);
            nzc = nzc || (st[c].active && yy != 0.0);
        }
        // a row with no nonzero column writes nothing unless a combine must output it
        if (__any_sync(gm, nzc) || a.out != nullptr) {
            live_rows |= 1u << k;
            if (a.acc && ((av_word >> (r & 31)) & 1u)) cp_async_cols<CPL>(&abuf[k][c0], a.acc + (size_t)r * B + c0);
        }
    }
    cp_async_wait_all();
    __syncwarp(gm);
    uint32_t nz_bits = 0, av_bits = 0;
    double bl1[CPL], bdm[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) bl1[c] = bdm[c] = 0.0;
    for (int k = 0; k < nrows; ++k) {
        if (!((live_rows >> k) & 1u)) continue;
        const uint32_t r = r0 + k;
        const bool valid = a.acc && ((av_word >> (r & 31)) & 1u);
        uint32_t d = 0;  // prefetched at item start: lane k % G holds row k
#pragma unroll
        for (int t = 0; t < MmShape<B>::DPL; ++t) {
            const uint32_t dt = __shfl_sync(gm, deg_lane[t], k % G, G);
            if (k / G == t) d = dt;
        }
        bool row_nz = false;
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            const uint32_t b = c0 + c;
            const size_t ix = (size_t)r * B + b;
            const double acc_old = valid ? abuf[k][b] : 0.0;
            if (!st[c].active) {
                // stopped column: acc stays; a pending combine still outputs it
                if (a.out) {
                    if (b < a.b_valid) a.out[a.out_node_major ? ix : (size_t)b * a.n + r] = combine_value(a, acc_old, r);
                } else if (write_acc) {
                    a.acc[ix] = acc_old;
                }
                continue;
            }
            double yy = ybuf[k][b];
            if (st[c].has_spread) yy = dadd(yy, st[c].spread);  // graph.cpp:265-268
            row_nz = row_nz || yy != 0.0;
            if (a.acc) {
                const double f = dadd(acc_old, yy);  // cpi.cpp:50
                if (a.out) {
                    if (b < a.b_valid) a.out[a.out_node_major ? ix : (size_t)b * a.n + r] = combine_value(a, f, r);
                } else {
                    a.acc[ix] = f;
                }
            }
            if (a.share_out) a.share_out[ix] = d ? ddiv(dmul(a.keep, yy), (double)d) : 0.0;  // graph.cpp:222
            bl1[c] = dadd(bl1[c], fabs(yy));  // block partials in row order,
            if (want_dm && d == 0) bdm[c] = dadd(bdm[c], yy);  // converted once below
        }
        if (write_acc) av_bits |= 1u << (r & 31);
        nz_bits |= (row_nz ? 1u : 0u) << (r & 31);
    }
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        // exact integer accumulation across blocks: order-independent totals
        if (bl1[c] != 0.0) fx_add(fx[0][c], fx[1][c], bl1[c]);
        if (bdm[c] != 0.0) fx_add(fx[2][c], fx[3][c], bdm[c]);
    }
    if (A.nz_out || (A.acc_valid && write_acc)) {
        uint32_t bits = nz_bits;
#pragma unroll
        for (int o = 1; o < G; o <<= 1) bits |= __shfl_xor_sync(gm, bits, o, G);
        if (gl == 0) {
            if (A.nz_out && bits) atomicOr(A.nz_out + (r0 >> 5), bits);
            if (A.acc_valid && write_acc && av_bits) atomicOr(A.acc_valid + (r0 >> 5), av_bits);
        }
    }
}

template <int B>
__global__ void __launch_bounds__(MmShape<B>::NT, 1) k_step_spmm2(MmArgs A) {
    using Sh = MmShape<B>;
    constexpr int G = Sh::G, CPL = Sh::CPL, NGRP = Sh::NGRP, NT = Sh::NT;
    const StepArgs& a = A.s;
    // per group: kMmRows x B row sums + kMmRows x B accumulator rows (dynamic)
    extern __shared__ __align__(16) unsigned char s_dyn[];
    __shared__ int64_t s_rp[NGRP][kMmRows + 2];
    __shared__ uint32_t s_rs[NGRP][kBlockNnz / 32 + 2];
    __shared__ uint32_t s_cl[NGRP][2];
    __shared__ int8_t s_nx[NGRP][kMmRows + 1];
    __shared__ ColState s_st[B];
    __shared__ unsigned long long s_fx[4 * B];
    __shared__ uint32_t s_ticket;
    __shared__ int s_any;

    const int tid = threadIdx.x;
    const int grp = tid / G, gl = tid % G;
    const int c0 = gl * CPL;
    const uint32_t gm = group_mask<G>();

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

    unsigned long long fx[4][CPL];  // l1 hi, l1 lo, dm hi, dm lo
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < CPL; ++c) fx[q][c] = 0ull;

    const uint32_t total = A.n_segs + A.n_blocks;
    const bool work = any_active || a.out != nullptr;  // all stopped: only a pending combine
    unsigned char* gbase = s_dyn + (size_t)grp * (Sh::kYBytes + Sh::kWBytes);
    double (*yb)[B] = reinterpret_cast<double (*)[B]>(gbase);
    double (*ab)[B] = reinterpret_cast<double (*)[B]>(gbase + Sh::kYBytes);  // epilogue view
    uint32_t* sidx = reinterpret_cast<uint32_t*>(gbase + Sh::kYBytes);      // stream view
    int64_t* rp = s_rp[grp];
    uint32_t next_item = 0;
    if (work && gl == 0) next_item = atomicAdd(A.work_cnt, 1u);
    while (work) {
        const uint32_t item = gshfl<G>(next_item, 0);
        if (item >= total) break;
        if (gl == 0) next_item = atomicAdd(A.work_cnt, 1u);  // overlap the next fetch
        const bool is_seg = item < A.n_segs;
        uint32_t r0;
        int nrows;
        if (is_seg) {
            // one kLong-nnz segment of a long row: a single run, no row ends inside
            r0 = A.seg_row[item];
            nrows = 1;
            if (gl == 0) {
                rp[0] = A.seg_lo[item];
                rp[1] = min(rp[0] + (int64_t)kLong, __ldg(a.row_ptr + r0 + 1));
            }
        } else {
            const uint2 blk = A.blocks[item - A.n_segs];
            r0 = blk.x;
            nrows = (int)blk.y;
            for (int k = gl; k <= nrows; k += G) rp[k] = __ldg(a.row_ptr + r0 + k);
        }
        // degrees of the item's rows: lane l holds rows l, l+G, ...
        uint32_t deg_lane[Sh::DPL];
#pragma unroll
        for (int t = 0; t < Sh::DPL; ++t) {
            const int k = t * G + gl;
            deg_lane[t] = k < nrows ? __ldg(a.deg + r0 + k) : 0u;
        }
        __syncwarp(gm);
        // ---- stage indices (+ frontier) and row starts, then stream -------
        const int64_t lo = rp[0];
        const int nnz = (int)(rp[nrows] - lo);
        uint32_t* rsb = s_rs[grp];
        uint32_t* clive = s_cl[grp];
        double s[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) s[c] = 0.0;
        const bool live = any_active && stage_indices<G>(A, lo, nnz, gl, sidx, clive);
        if (!is_seg) {
            for (int k = gl; k < (nnz + 31) / 32 + 1; k += G) rsb[k] = 0u;
            for (int k = 0; k < nrows; ++k)
#pragma unroll
                for (int c = 0; c < CPL; ++c) yb[k][c0 + c] = 0.0;
            if (gl == 0) {
                // next non-empty row after k (nrows if none)
                int nx = nrows;
                for (int k = nrows - 1; k >= 0; --k) {
                    s_nx[grp][k] = (int8_t)nx;
                    if (rp[k + 1] > rp[k]) nx = k;
                }
                s_nx[grp][kMmRows] = (int8_t)nx;  // first non-empty row
            }
            __syncwarp(gm);
            for (int k = 1 + gl; k < nrows; k += G) {
                const int p = (int)(rp[k] - lo);
                if (rp[k + 1] > rp[k] && p > 0) atomicOr(&rsb[p >> 5], 1u << (p & 31));
            }
        }
        __syncwarp(gm);
        if (live) {
            if (is_seg) {
                consume_staged<B, false>(a.share_in, sidx, clive, nullptr, nnz, c0, s, [](const double*, bool) {});
            } else {
                const int8_t* nxt = s_nx[grp];
                int cur = nxt[kMmRows];
                consume_staged<B, true>(a.share_in, sidx, clive, rsb, nnz, c0, s, [&](const double* fin, bool nb) {
                    if (nb) {
#pragma unroll
                        for (int c = 0; c < CPL; ++c) yb[cur][c0 + c] = fin[c];
                        cur = nxt[cur];
                    }
                });
                if (nnz > 0)
#pragma unroll
                    for (int c = 0; c < CPL; ++c) yb[cur][c0 + c] = s[c];
            }
        }
        if (is_seg) {
            // publish the segment; the last of the row's segments finishes it
#pragma unroll
            for (int c = 0; c < CPL; ++c) A.seg_part[(size_t)item * B + c0 + c] = s[c];
            __threadfence();
            __syncwarp(gm);
            const uint32_t li = A.seg_long[item];
            uint32_t t = 0;
            if (gl == 0) t = atomicAdd(A.long_cnt + li, 1u);
            t = gshfl<G>(t, 0);
            if (t != A.long_nseg[li] - 1) continue;
            __threadfence();
            const uint32_t f0 = A.long_first[li], ns = A.long_nseg[li];
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const double y = seg_sum(A.seg_part + (size_t)f0 * B + c0 + c, B, ns);
                yb[0][c0 + c] = y;
            }
            if (gl == 0) A.long_cnt[li] = 0;
        }
        __syncwarp(gm);
        mm_epilogue_rows<B>(A, st, r0, nrows, yb, ab, deg_lane, gl, c0, fx);
        __syncwarp(gm);
    }

    // ---- residual / dangling-mass reduction: exact 128-bit integer sums, so
    // the result is independent of which group processed which rows.
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
    // last CTA: cpi.cpp:73-80 for every column, then reset the counters
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
