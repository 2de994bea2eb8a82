// cpi_frontier.cuh -- arguments of the fused B-seed sweep (cpi_spmm5.cuh) and
// the direction-optimised sparse sweeps of a seed batch: frontier cost, push
// marking of the rows a small frontier reaches (byte flags, hub out-lists cut
// into chunks), the marked row windows and long-row segments the pull visits.
#pragma once

#include "cpi_spmm.cuh"

namespace tpa {

struct Mm4Args {
    MmArgs m;               // graph, state, bitmaps, segments, reduction (reused)
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
    if (blockIdx.x == 0 && (int)threadIdx.x < B && st[threadIdx.x].active && st[threadIdx.x].has_spread)
        atomicAdd(cost, 1ull << 62);
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

}  // namespace tpa
