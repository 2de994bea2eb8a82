// tpa_topk.cuh -- top_k_nodes (metrics.cpp:25-36) on the device, for B score
// vectors at once: a query batch then returns B·k results
// instead of B·n doubles.
//
// Order (the reference's comparator): score descending, equal scores by
// ascending node id.  Every node gets a distinct 96-bit key
//   K = order_key(score) << 32 | ~id
// (order_key: the IEEE bits made unsigned-monotone, -0.0 folded onto +0.0
// since the reference compares values), so the k largest keys are exactly
// the reference's top k, and a radix select over K needs no tie handling.
//   * digits of 12 bits from the top; per digit: a histogram of the
//     still-matching elements, a select (the bin holding the k-th key), and
//     an emit of the elements above it, merged into the next histogram pass;
//   * the first two digits scan the whole vector, the second also compacts
//     the bin's elements into a candidate list that later digits scan;
//   * the k emitted ids are finally ordered by two stable segmented radix
//     sorts (id ascending, then order_key descending).
// Included at the end of tpa_gpu.cu.
#pragma once

#include <cub/device/device_segmented_radix_sort.cuh>

namespace tpa {

constexpr int kTkBits = 12, kTkBins = 1 << kTkBits, kTkDigits = 96 / kTkBits;

struct TopkState {
    unsigned long long pfx_hi, pfx_lo;  // resolved digits (96-bit, high-aligned) after the last select
    unsigned long long old_hi, old_lo;  // ... before it (what the emit of that digit matches)
    uint32_t k_rem;                     // keys still to take from the selected bin onwards
    uint32_t t;                         // selected bin of the last select
    uint32_t take_all;                  // the selected bin is taken whole: finished after its emit
    uint32_t done;                      // finished (all k emitted)
    uint32_t n_out;                     // emitted so far
    uint32_t n_cand;                    // candidate list length
};

__device__ __forceinline__ unsigned long long order_key(double x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(x == 0.0 ? 0.0 : x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// 96-bit key as (hi 64, lo 32): hi = order_key, lo = ~id.  Digit d covers
// key bits [95 - 12d, 84 - 12d].
__device__ __forceinline__ uint32_t tk_digit(unsigned long long hi, uint32_t lo, int d) {
    const int sh = 84 - kTkBits * d;  // position of the digit's lowest bit
    if (sh >= 32) return (uint32_t)(hi >> (sh - 32)) & (kTkBins - 1);
    if (sh + kTkBits <= 32) return (lo >> sh) & (kTkBins - 1);
    // d = 5 (key bits 35..24) straddles: 4 bits of hi, 8 of lo
    return (uint32_t)(((hi << (32 - sh)) | (lo >> sh)) & (kTkBins - 1));
}

// key's top 12d bits equal the prefix's (d = 0: always)
__device__ __forceinline__ bool tk_match(unsigned long long hi, uint32_t lo, unsigned long long p_hi,
                                         unsigned long long p_lo, int d) {
    const int nb = kTkBits * d;  // resolved bits
    if (nb == 0) return true;
    if (nb <= 64) {
        const unsigned long long m = nb == 64 ? ~0ull : ~((1ull << (64 - nb)) - 1);
        return (hi & m) == (p_hi & m);
    }
    if (hi != p_hi) return false;
    const int lb = nb - 64;  // bits of the low 32 resolved
    const uint32_t m = lb >= 32 ? 0xffffffffu : ~((1u << (32 - lb)) - 1);
    return (lo & m) == ((uint32_t)p_lo & m);
}

__device__ __forceinline__ void tk_set_digit(unsigned long long& p_hi, unsigned long long& p_lo, int d, uint32_t v) {
    const int sh = 84 - kTkBits * d;
    if (sh >= 32) {
        p_hi |= (unsigned long long)v << (sh - 32);
    } else if (sh + kTkBits <= 32) {
        p_lo |= (unsigned long long)v << sh;
    } else {  // straddles (d = 5)
        p_hi |= (unsigned long long)v >> (32 - sh);
        p_lo |= ((unsigned long long)v << sh) & 0xffffffffull;
    }
}

struct TkArgs {
    const double* scores;  // [B][n]
    uint32_t n, k;
    TopkState* st;         // [B]
    uint32_t* hist;        // [B][kTkBins], zero between passes
    uint32_t* cand;        // [B][n]
    uint32_t* out_ids;     // [B][k] (unordered until the final sort)
};

// One pass over vector b's elements (all of them, or its candidate list):
// emit the keys above the last selected bin (digit d-1), compact the bin's
// keys (when `compact`), and histogram digit d of the keys in the bin (d < 8).
__global__ void __launch_bounds__(256) k_topk_pass(TkArgs A, int d, int from_cand, int compact) {
    __shared__ uint32_t s_hist[kTkBins];
    const uint32_t b = blockIdx.y;
    TopkState& S = A.st[b];
    if (S.done) return;
    const bool do_hist = d < kTkDigits && !S.take_all;
    if (do_hist)
        for (int i = threadIdx.x; i < kTkBins; i += blockDim.x) s_hist[i] = 0;
    __syncthreads();
    const uint32_t cnt = from_cand ? S.n_cand : A.n;
    const double* sc = A.scores + (size_t)b * A.n;
    const uint32_t* cl = A.cand + (size_t)b * A.n;
    const unsigned long long o_hi = S.old_hi, o_lo = S.old_lo, p_hi = S.pfx_hi, p_lo = S.pfx_lo;
    const uint32_t t = S.t;
    const bool take_all = S.take_all;
    // 8 independent loads in flight per thread (the scan is HBM-bound)
    constexpr int U = 8;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < cnt; i0 += U * stride) {
      uint32_t ids[U];
      double vals[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
          const uint32_t i = i0 + u * stride;
          ids[u] = i < cnt ? (from_cand ? cl[i] : i) : 0xffffffffu;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) vals[u] = ids[u] != 0xffffffffu ? __ldcs(sc + ids[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t id = ids[u];
        if (id == 0xffffffffu) continue;
        const unsigned long long hi = order_key(vals[u]);
        const uint32_t lo = ~id;
        bool in_bin = true;  // still a candidate for digit d
        if (d > 0) {
            in_bin = false;
            if (tk_match(hi, lo, o_hi, o_lo, d - 1)) {
                const uint32_t dg = tk_digit(hi, lo, d - 1);
                if (dg > t || (take_all && dg == t)) {
                    A.out_ids[(size_t)b * A.k + atomicAdd(&S.n_out, 1u)] = id;
                } else if (dg == t) {
                    in_bin = true;
                    if (compact) A.cand[(size_t)b * A.n + atomicAdd(&S.n_cand, 1u)] = id;
                }
            }
        }
        if (do_hist && in_bin && tk_match(hi, lo, p_hi, p_lo, d)) atomicAdd(&s_hist[tk_digit(hi, lo, d)], 1u);
      }
    }
    if (!do_hist) return;
    __syncthreads();
    uint32_t* gh = A.hist + (size_t)b * kTkBins;
    for (int i = threadIdx.x; i < kTkBins; i += blockDim.x)
        if (s_hist[i]) atomicAdd(gh + i, s_hist[i]);
}

// The bin of digit d holding the k_rem-th largest key; one CTA per vector.
__global__ void __launch_bounds__(1024) k_topk_select(TkArgs A, int d) {
    __shared__ uint32_t s_sum[1024];
    const uint32_t b = blockIdx.x;
    TopkState& S = A.st[b];
    if (S.done) return;
    if (S.take_all) {  // finished by the emit of the previous pass
        if (threadIdx.x == 0) S.done = 1;
        return;
    }
    const uint32_t k = S.k_rem;  // read before the scan's barriers; the winner rewrites it
    uint32_t* gh = A.hist + (size_t)b * kTkBins;
    constexpr int per = kTkBins / 1024;
    // thread j owns bins [kTkBins - per(j+1), kTkBins - per j): descending order
    uint32_t c[per], tot = 0;
#pragma unroll
    for (int q = 0; q < per; ++q) {
        c[q] = gh[kTkBins - 1 - (threadIdx.x * per + q)];
        tot += c[q];
    }
    s_sum[threadIdx.x] = tot;
    __syncthreads();
    // inclusive scan (Hillis-Steele) of the per-thread totals
    for (int o = 1; o < 1024; o <<= 1) {
        const uint32_t v = threadIdx.x >= (unsigned)o ? s_sum[threadIdx.x - o] : 0u;
        __syncthreads();
        s_sum[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t above = threadIdx.x ? s_sum[threadIdx.x - 1] : 0u;
    if (above < k && k <= s_sum[threadIdx.x]) {
#pragma unroll
        for (int q = 0; q < per; ++q) {
            if (above < k && k <= above + c[q]) {
                const uint32_t bin = kTkBins - 1 - (threadIdx.x * per + q);
                S.old_hi = S.pfx_hi;
                S.old_lo = S.pfx_lo;
                tk_set_digit(S.pfx_hi, S.pfx_lo, d, bin);
                S.t = bin;
                S.k_rem = k - above;
                S.take_all = (above + c[q] == k) || d == kTkDigits - 1;
            }
            above += c[q];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kTkBins; i += 1024) gh[i] = 0;
}

// Digits 3..7 (and the last emit) over the candidate list, one CTA per vector
// with the state and the histogram in shared memory: the candidate list is
// short unless many keys share their top 24 bits, and one launch replaces
// twelve.
__global__ void __launch_bounds__(1024) k_topk_finish(TkArgs A) {
    __shared__ uint32_t s_hist[kTkBins];
    __shared__ uint32_t s_sum[1024];
    __shared__ TopkState S;
    const uint32_t b = blockIdx.x, tid = threadIdx.x;
    if (tid == 0) S = A.st[b];
    __syncthreads();
    if (S.done) return;
    const uint32_t* cl = A.cand + (size_t)b * A.n;
    const double* sc = A.scores + (size_t)b * A.n;
    const uint32_t cnt = S.n_cand;
    constexpr int per = kTkBins / 1024;
    for (int d = 3; d <= kTkDigits; ++d) {
        const bool do_hist = d < kTkDigits && !S.take_all;
        if (do_hist)
            for (int i = tid; i < kTkBins; i += 1024) s_hist[i] = 0;
        const unsigned long long o_hi = S.old_hi, o_lo = S.old_lo, p_hi = S.pfx_hi, p_lo = S.pfx_lo;
        const uint32_t t = S.t;
        const bool take_all = S.take_all;
        __syncthreads();
        for (uint32_t i = tid; i < cnt; i += 1024) {
            const uint32_t id = cl[i];
            const unsigned long long hi = order_key(sc[id]);
            const uint32_t lo = ~id;
            if (!tk_match(hi, lo, o_hi, o_lo, d - 1)) continue;
            const uint32_t dg = tk_digit(hi, lo, d - 1);
            if (dg > t || (take_all && dg == t)) {
                A.out_ids[(size_t)b * A.k + atomicAdd(&S.n_out, 1u)] = id;
                continue;
            }
            if (dg == t && do_hist && tk_match(hi, lo, p_hi, p_lo, d)) atomicAdd(&s_hist[tk_digit(hi, lo, d)], 1u);
        }
        __syncthreads();
        if (!do_hist) break;  // take_all emitted or the last digit
        // select (as k_topk_select)
        const uint32_t k = S.k_rem;
        uint32_t c[per], tot = 0;
#pragma unroll
        for (int q = 0; q < per; ++q) {
            c[q] = s_hist[kTkBins - 1 - (tid * per + q)];
            tot += c[q];
        }
        s_sum[tid] = tot;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            const uint32_t v = tid >= (unsigned)o ? s_sum[tid - o] : 0u;
            __syncthreads();
            s_sum[tid] += v;
            __syncthreads();
        }
        uint32_t above = tid ? s_sum[tid - 1] : 0u;
        if (above < k && k <= s_sum[tid]) {
#pragma unroll
            for (int q = 0; q < per; ++q) {
                if (above < k && k <= above + c[q]) {
                    const uint32_t bin = kTkBins - 1 - (tid * per + q);
                    S.old_hi = S.pfx_hi;
                    S.old_lo = S.pfx_lo;
                    tk_set_digit(S.pfx_hi, S.pfx_lo, d, bin);
                    S.t = bin;
                    S.k_rem = k - above;
                    S.take_all = (above + c[q] == k) || d == kTkDigits - 1;
                }
                above += c[q];
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        S.done = 1;
        A.st[b] = S;
    }
}

__global__ void k_topk_init(TopkState* st, uint32_t B, uint32_t k) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    TopkState s{};
    s.k_rem = k;
    st[b] = s;
}

__global__ void k_topk_keys(TkArgs A, uint32_t B, unsigned long long* keys, const uint32_t* ids_sorted,
                            double* out_scores) {
    const uint64_t total = (uint64_t)B * A.k;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = (uint32_t)(i / A.k);
        const uint32_t id = ids_sorted ? ids_sorted[i] : A.out_ids[i];
        const double v = A.scores[(size_t)b * A.n + id];
        if (keys) keys[i] = order_key(v);
        if (out_scores) out_scores[i] = v;
    }
}

// Final order for k <= kTkSmall: one CTA per vector, bitonic sort in shared
// memory by (order_key descending, id ascending), scores re-read exactly.
constexpr uint32_t kTkSmall = 2048;

__global__ void __launch_bounds__(1024) k_topk_sort_small(TkArgs A, uint32_t* out_ids, double* out_scores) {
    __shared__ unsigned long long s_key[kTkSmall];
    __shared__ uint32_t s_id[kTkSmall];
    const uint32_t b = blockIdx.x, k = A.k;
    uint32_t P = 1;
    while (P < k) P <<= 1;
    const double* sc = A.scores + (size_t)b * A.n;
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        if (i < k) {
            const uint32_t id = A.out_ids[(size_t)b * k + i];
            s_key[i] = order_key(sc[id]);
            s_id[i] = id;
        } else {
            s_key[i] = 0ull;  // below every real key (order_key sets the top bit of non-negatives)
            s_id[i] = 0xffffffffu;
        }
    }
    __syncthreads();
    // "before" = (key greater) or (key equal and id smaller)
    for (uint32_t size = 2; size <= P; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
                const uint32_t j = i ^ stride;
                if (j > i) {
                    const bool desc_block = (i & size) == 0;  // this block sorts "before"-first
                    const unsigned long long ki = s_key[i], kj = s_key[j];
                    const uint32_t ii = s_id[i], ij = s_id[j];
                    const bool j_before_i = kj > ki || (kj == ki && ij < ii);
                    if (j_before_i == desc_block) {
                        s_key[i] = kj;
                        s_key[j] = ki;
                        s_id[i] = ij;
                        s_id[j] = ii;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
        out_ids[(size_t)b * k + i] = s_id[i];
        if (out_scores) out_scores[(size_t)b * k + i] = sc[s_id[i]];
    }
}

__global__ void k_seg_offsets(int* off, uint32_t B, uint32_t k) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b <= B) off[b] = (int)(b * k);
}

// top-k of B device-resident vectors [B][n] into device ids / scores [B][k].
// `scratch` (optional, >= B * n * 4 bytes): a dead device buffer to hold the
// candidate lists instead of the handle's own (the query path passes the
// batch's accumulator, free once its last sweep has combined).
static void topk_device(tpa_graph* g, const double* scores, uint32_t B, uint32_t k, uint32_t* d_ids,
                        double* d_scores, void* scratch = nullptr, size_t scratch_bytes = 0) {
    cudaStream_t s = g->stream;
    const uint32_t n = g->n;
    auto& W = g->topk;
    DevBuf &st = W.st, &hist = W.hist, &cand = W.cand, &ids = W.ids;
    st.ensure((size_t)B * sizeof(TopkState), g->stream);
    if (hist.bytes < (size_t)B * kTkBins * 4) {
        hist.ensure((size_t)B * kTkBins * 4, g->stream);
        CK(cudaMemsetAsync(hist.p, 0, hist.bytes, s));  // the selects leave it zeroed
    }
    uint32_t* cand_p = nullptr;
    if (scratch && scratch_bytes >= (size_t)B * n * 4) {
        cand_p = static_cast<uint32_t*>(scratch);
    } else {
        cand.ensure((size_t)B * n * 4, g->stream);
        cand_p = cand.as<uint32_t>();
    }
    ids.ensure((size_t)B * k * 4, g->stream);
    k_topk_init<<<(B + 127) / 128, 128, 0, s>>>(st.as<TopkState>(), B, k);
    TkArgs A{scores, n, k, st.as<TopkState>(), hist.as<uint32_t>(), cand_p, ids.as<uint32_t>()};
    // a few CTAs per vector, each over >= 16k elements: the per-CTA histogram
    // zeroing / flushing (4096 bins) must stay small against the scan
    const uint32_t full_x = (uint32_t)grid_for(n, 256 * 64, std::max(1, (int)(8 * g->num_sms / std::max<uint32_t>(B, 1))));
    const uint32_t cand_x = (uint32_t)std::max(1, std::min<int>(grid_for(n, 256 * 8, 1 << 20), g->num_sms));
    int launches = 1;
    // digits 0, 1 and the compaction scan the whole vectors; digits 3.. the candidates
    for (int d = 0; d <= 2; ++d) {
        k_topk_pass<<<dim3(full_x, B), 256, 0, s>>>(A, d, 0, d == 2 ? 1 : 0);
        CKL("k_topk_pass");
        k_topk_select<<<B, 1024, 0, s>>>(A, d);
        CKL("k_topk_select");
        launches += 2;
    }
    k_topk_finish<<<B, 1024, 0, s>>>(A);
    CKL("k_topk_finish");
    ++launches;
    (void)cand_x;
    if (k <= kTkSmall) {
        k_topk_sort_small<<<B, 1024, 0, s>>>(A, d_ids, d_scores);
        CKL("k_topk_sort_small");
        g->launches += launches + 1;
        return;
    }
    // larger k: ids ascending, then (stable) keys descending (CUB segmented radix sorts)
    DevBuf keys, keys2, ids2, off, temp;
    keys.ensure((size_t)B * k * 8, g->stream);
    keys2.ensure((size_t)B * k * 8, g->stream);
    ids2.ensure((size_t)B * k * 4, g->stream);
    off.ensure((size_t)(B + 1) * 4, g->stream);
    k_seg_offsets<<<(B + 1 + 127) / 128, 128, 0, s>>>(off.as<int>(), B, k);
    const int nk = (int)(B * k);
    size_t t1 = 0, t2 = 0;
    CK(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, t1, ids.as<uint32_t>(), ids2.as<uint32_t>(), nk, (int)B,
                                               off.as<int>(), off.as<int>() + 1, 0, 32, s));
    CK(cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, t2, keys.as<unsigned long long>(),
                                                          keys2.as<unsigned long long>(), ids2.as<uint32_t>(),
                                                          d_ids, nk, (int)B, off.as<int>(), off.as<int>() + 1,
                                                          0, 64, s));
    temp.ensure(std::max(t1, t2), g->stream);
    CK(cub::DeviceSegmentedRadixSort::SortKeys(temp.p, t1, ids.as<uint32_t>(), ids2.as<uint32_t>(), nk, (int)B,
                                               off.as<int>(), off.as<int>() + 1, 0, 32, s));
    TkArgs A2 = A;
    k_topk_keys<<<grid_for((uint64_t)B * k, 256, 4 * g->num_sms), 256, 0, s>>>(A2, B, keys.as<unsigned long long>(),
                                                                              ids2.as<uint32_t>(), nullptr);
    CK(cub::DeviceSegmentedRadixSort::SortPairsDescending(temp.p, t2, keys.as<unsigned long long>(),
                                                          keys2.as<unsigned long long>(), ids2.as<uint32_t>(),
                                                          d_ids, nk, (int)B, off.as<int>(), off.as<int>() + 1,
                                                          0, 64, s));
    if (d_scores) {
        k_topk_keys<<<grid_for((uint64_t)B * k, 256, 4 * g->num_sms), 256, 0, s>>>(A2, B, nullptr, d_ids, d_scores);
    }
    CKL("k_topk_sort");
    g->launches += launches + 4;
}

}  // namespace tpa

extern "C" {

int tpa_top_k(tpa_graph* g, const double* scores, uint32_t B, uint32_t k, uint32_t* out_ids, double* out_scores,
              int flags) {
    return guard([&] {
        if (!g) throw std::invalid_argument("null graph");
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        require_whole(g, "tpa_top_k");
        const uint32_t n = g->n;
        if (k < 1 || k > n) throw std::out_of_range("k must be in [1, n], got " + std::to_string(k));  // metrics.cpp:26-27
        if (B == 0) return;
        if (!scores || !out_ids) throw std::invalid_argument("null array");
        const bool dev = flags & TPA_DEVICE_PTRS;
        DevBuf in, ids, sc;
        const double* d_in = scores;
        if (!dev) {
            in.ensure((size_t)B * n * 8, g->stream);
            CK(cudaMemcpyAsync(in.p, scores, (size_t)B * n * 8, cudaMemcpyHostToDevice, g->stream));
            d_in = in.as<double>();
            ids.ensure((size_t)B * k * 4, g->stream);
            if (out_scores) sc.ensure((size_t)B * k * 8, g->stream);
        }
        topk_device(g, d_in, B, k, dev ? out_ids : ids.as<uint32_t>(),
                    out_scores ? (dev ? out_scores : sc.as<double>()) : nullptr);
        if (!dev) {
            download(g, out_ids, ids.p, (size_t)B * k * 4);
            if (out_scores) download(g, out_scores, sc.p, (size_t)B * k * 8);
        }
        CK(cudaStreamSynchronize(g->stream));
    });
}

int tpa_query_batch_topk(tpa_graph* g, const tpa_artifact* a, const uint32_t* seeds, uint32_t B, uint32_t S,
                         uint32_t k, uint32_t* out_ids, double* out_scores, int flags) {
    return guard([&] {
        if (!g) throw std::invalid_argument("null graph");
        require_whole(g, "tpa_query_batch_topk");
        std::lock_guard<std::mutex> lk(g->mu);
        DeviceGuard dg(g->device);
        const bool na = flags & TPA_QUERY_NA;
        if (!a) throw std::invalid_argument("null artifact");
        check_query(g, a, S);
        const uint32_t n = g->n;
        if (k < 1 || k > n) throw std::out_of_range("k must be in [1, n], got " + std::to_string(k));
        if (B == 0) return;
        const bool dev = flags & TPA_DEVICE_PTRS;
        const double scale = 1.0 + tpa_neighbor_scale_factor(a->c, S, a->T);  // tpa.cpp:71-72
        DevBuf ids, sc;
        const uint32_t chunk = std::min<uint32_t>(B, 64);
        if (!dev) {
            ids.ensure((size_t)chunk * k * 4, g->stream);
            if (out_scores) sc.ensure((size_t)chunk * k * 8, g->stream);
        }
        for (uint32_t b0 = 0; b0 < B; b0 += chunk) {
            const uint32_t bv = std::min(chunk, B - b0);
            // The combined scores land in the share buffer the batch's last
            // sweep does not touch (sweep i reads share[(i-1)&1] and the last
            // one, i = S-1, writes no shares; with S = 1 no sweep runs and
            // share[1] is idle): no B x n scratch of its own, which is what
            // lets the billion-edge config (B = 16, n = 2^28: 34 GB per
            // buffer) fit one GPU.  Share rows are only ever read through the
            // frontier bitmaps, so the next batch never sees these values.
            Workspace& w = g->workspace(batch_width(bv));
            double* scores = w.share[S == 1 ? 1 : ((S - 1) & 1)].as<double>();
            // seeds are host arrays (tpa_gpu.h); the family parts stay on the device
            run_seed_batch(g, seeds + b0, bv, a->c, a->eps, 0, (int64_t)S - 1, na ? nullptr : a->stranger.as<double>(),
                           scale, true, scores, TPA_DEVICE_PTRS | TPA_ASYNC);
            uint32_t* d_ids = dev ? out_ids + (size_t)b0 * k : ids.as<uint32_t>();
            double* d_sc = out_scores ? (dev ? out_scores + (size_t)b0 * k : sc.as<double>()) : nullptr;
            topk_device(g, scores, bv, k, d_ids, d_sc, w.acc.p, w.acc.bytes);  // acc is dead until the next init
            if (!dev) {
                download(g, out_ids + (size_t)b0 * k, ids.p, (size_t)bv * k * 4);
                if (out_scores) download(g, out_scores + (size_t)b0 * k, sc.p, (size_t)bv * k * 8);
            }
        }
        CK(cudaStreamSynchronize(g->stream));
    });
}

}  // extern "C"
