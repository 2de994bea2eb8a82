// tpa_graph_build.cuh -- the reference Graph constructor (graph.cpp:53-91) on
// the GPU: validate endpoints, sort + dedupe the edges,
// pre-policy dangling list, SelfLoop repair, out-CSR.  The FNV-1a fingerprint
// is a strictly sequential byte chain (graph.cpp:28-31) and stays on the host
// (make_host_graph), over the downloaded arrays.  The result is the same
// tpa_host_graph the host builder makes, byte for byte.
//   * first offending edge in input order (atomicMin over its index) ->
//     out_of_range with the reference's message;
//   * keys (u << 32 | v): CUB radix sort + unique = std::sort + std::unique;
//   * out-degrees by atomics, dangling flags, an exclusive scan of
//     deg + repair -> out_offsets; target of deduped edge i with source u at
//     i + (dangling nodes below u), a repair edge (u, u) at out_offsets[u].
// Included at the end of tpa_gpu.cu.
#pragma once

#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

namespace tpa {

__global__ void k_gb_validate(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t m,
                              uint32_t n, unsigned long long* first_bad) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
        if (src[e] >= n || dst[e] >= n) atomicMin(first_bad, (unsigned long long)e);
}

__global__ void k_gb_keys(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t m,
                          unsigned long long* __restrict__ keys) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
        keys[e] = ((unsigned long long)src[e] << 32) | dst[e];
}

__global__ void k_gb_degrees(const unsigned long long* __restrict__ keys, const unsigned long long* m_ptr,
                             uint32_t* __restrict__ deg) {
    const uint64_t m = *m_ptr;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(deg + (uint32_t)(keys[e] >> 32), 1u);
}

// cnt[u] = deg + SelfLoop repair; dflag[u] = dangling (pre-policy)
__global__ void k_gb_counts(const uint32_t* __restrict__ deg, uint32_t n, int repair,
                            unsigned long long* __restrict__ cnt, uint32_t* __restrict__ dflag) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t d = deg[u];
        dflag[u] = d == 0;
        cnt[u] = d ? d : (repair ? 1u : 0u);
    }
}

__global__ void k_gb_scatter(const unsigned long long* __restrict__ keys, const unsigned long long* m_ptr,
                             const uint32_t* __restrict__ dpre, int repair, uint32_t* __restrict__ tgt) {
    const uint64_t m = *m_ptr;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[e];
        const uint32_t u = (uint32_t)(k >> 32);
        tgt[e + (repair ? dpre[u] : 0u)] = (uint32_t)k;
    }
}

__global__ void k_gb_dangling(const uint32_t* __restrict__ dflag, const uint32_t* __restrict__ dpre, uint32_t n,
                              int repair, const unsigned long long* __restrict__ off, uint32_t* __restrict__ dang,
                              uint32_t* __restrict__ tgt) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x) {
        if (!dflag[u]) continue;
        dang[dpre[u]] = (uint32_t)u;
        if (repair) tgt[off[u]] = (uint32_t)u;  // graph.cpp:72-75
    }
}

struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
    }
};

// Sort + dedupe the m (u << 32 | v) keys in `keys` (graph.cpp:63-64), then the
// degrees, dangling list, SelfLoop repair and out-CSR (graph.cpp:67-82),
// downloaded into a host graph.  Keys equal to kNoEdge (a generator's dropped
// self-loop) sort last and are discarded.  `keys` / `alt` are m-key buffers
// used as the sort's double buffer (no third copy: 2 x 8m bytes at most).
constexpr unsigned long long kNoEdge = ~0ull;

__global__ void k_gb_drop_noedge(const unsigned long long* __restrict__ keys, unsigned long long* m_ptr) {
    const unsigned long long m = *m_ptr;
    if (m && keys[m - 1] == kNoEdge) *m_ptr = m - 1;
}

static tpa_host_graph* graph_from_keys(uint32_t n, DevBuf& keys, DevBuf& alt, uint64_t m, int policy, cudaStream_t s,
                                       int blocks) {
    std::vector<uint64_t> off(n + 1ull);
    std::vector<uint32_t> tgt, dang;
    DevBuf d_m, d_deg, d_cnt, d_off, d_flag, d_pre, d_tgt, d_dang, temp;
    d_m.ensure(8, s);
    int bits = 1;
    while (bits < 32 && (1ull << bits) < n) ++bits;
    // bits [0, 32 + bits) order every real key; kNoEdge (all ones there)
    // still sorts after all of them (v < n <= 2^31, so no real key ties it)
    const int end_bit = 32 + bits;
    DevBuf* cur = &keys;
    DevBuf* oth = &alt;
    if (m) {
        cub::DoubleBuffer<unsigned long long> db(keys.as<unsigned long long>(), alt.as<unsigned long long>());
        size_t t1 = 0;
        CK(cub::DeviceRadixSort::SortKeys(nullptr, t1, db, (int64_t)m, 0, end_bit, s));
        temp.ensure(t1, s);
        CK(cub::DeviceRadixSort::SortKeys(temp.p, t1, db, (int64_t)m, 0, end_bit, s));
        if (db.Current() != keys.as<unsigned long long>()) std::swap(cur, oth);
        size_t t2 = 0;
        CK(cub::DeviceSelect::Unique(nullptr, t2, cur->as<unsigned long long>(), oth->as<unsigned long long>(),
                                     d_m.as<unsigned long long>(), (int64_t)m, s));
        temp.ensure(t2, s);
        CK(cub::DeviceSelect::Unique(temp.p, t2, cur->as<unsigned long long>(), oth->as<unsigned long long>(),
                                     d_m.as<unsigned long long>(), (int64_t)m, s));
        std::swap(cur, oth);
        k_gb_drop_noedge<<<1, 1, 0, s>>>(cur->as<unsigned long long>(), d_m.as<unsigned long long>());
        CKL("k_gb_drop_noedge");
        oth->release();  // the unsorted / duplicate-carrying copy is dead
        temp.release();
    } else {
        CK(cudaMemsetAsync(d_m.p, 0, 8, s));
    }
    const unsigned long long* K = m ? cur->as<unsigned long long>() : nullptr;
    // graph.cpp:67-82: degrees, dangling, repair, offsets, targets
    const int repair = policy == TPA_SELFLOOP;
    d_cnt.ensure((n + 1ull) * 8, s);
    d_off.ensure((n + 1ull) * 8, s);
    d_flag.ensure((n + 1ull) * 4, s);
    d_pre.ensure((n + 1ull) * 4, s);
    d_deg.ensure((size_t)n * 4, s);
    size_t t3 = 0, t4 = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, t3, d_cnt.as<unsigned long long>(), d_off.as<unsigned long long>(),
                                     (int64_t)n + 1, s));
    CK(cub::DeviceScan::ExclusiveSum(nullptr, t4, d_flag.as<uint32_t>(), d_pre.as<uint32_t>(), (int64_t)n + 1, s));
    temp.ensure(std::max(t3, t4), s);
    CK(cudaMemsetAsync(d_deg.p, 0, (size_t)n * 4, s));
    if (m) {
        k_gb_degrees<<<blocks, 256, 0, s>>>(K, d_m.as<unsigned long long>(), d_deg.as<uint32_t>());
        CKL("k_gb_degrees");
    }
    CK(cudaMemsetAsync(d_cnt.as<unsigned long long>() + n, 0, 8, s));
    CK(cudaMemsetAsync(d_flag.as<uint32_t>() + n, 0, 4, s));
    k_gb_counts<<<blocks, 256, 0, s>>>(d_deg.as<uint32_t>(), n, repair, d_cnt.as<unsigned long long>(),
                                       d_flag.as<uint32_t>());
    CKL("k_gb_counts");
    CK(cub::DeviceScan::ExclusiveSum(temp.p, t3, d_cnt.as<unsigned long long>(), d_off.as<unsigned long long>(),
                                     (int64_t)n + 1, s));
    CK(cub::DeviceScan::ExclusiveSum(temp.p, t4, d_flag.as<uint32_t>(), d_pre.as<uint32_t>(), (int64_t)n + 1, s));
    uint32_t n_dang = 0;
    CK(cudaMemcpyAsync(off.data(), d_off.p, (n + 1ull) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&n_dang, d_pre.as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint64_t m_out = off[n];
    d_tgt.ensure(std::max<uint64_t>(m_out, 1) * 4, s);
    d_dang.ensure(std::max<uint32_t>(n_dang, 1) * 4, s);
    if (m) {
        k_gb_scatter<<<blocks, 256, 0, s>>>(K, d_m.as<unsigned long long>(), d_pre.as<uint32_t>(), repair,
                                            d_tgt.as<uint32_t>());
        CKL("k_gb_scatter");
    }
    k_gb_dangling<<<blocks, 256, 0, s>>>(d_flag.as<uint32_t>(), d_pre.as<uint32_t>(), n, repair,
                                         d_off.as<unsigned long long>(), d_dang.as<uint32_t>(), d_tgt.as<uint32_t>());
    CKL("k_gb_dangling");
    tgt.resize(m_out);
    dang.resize(n_dang);
    if (m_out) CK(cudaMemcpyAsync(tgt.data(), d_tgt.p, m_out * 4, cudaMemcpyDeviceToHost, s));
    if (n_dang) CK(cudaMemcpyAsync(dang.data(), d_dang.p, (size_t)n_dang * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return make_host_graph(n, policy, std::move(off), std::move(tgt), std::move(dang));
}

static tpa_host_graph* build_graph_gpu(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t m, int policy,
                                       int device) {
    if (n == 0) throw std::invalid_argument("graph must have at least one node");
    if (policy < 0 || policy > 2) throw std::invalid_argument("unknown dangling policy");
    if (m && (!src || !dst)) throw std::invalid_argument("null edge arrays");
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int blocks = 8 * sms;
    StreamGuard sg{s};  // destroyed after the buffers (their frees are ordered on s)
    DevBuf d_src, d_dst, d_bad, d_keys, d_keys2;
    const size_t mm = std::max<uint64_t>(m, 1);
    d_src.ensure(mm * 4, s);
    d_dst.ensure(mm * 4, s);
    d_bad.ensure(8, s);
    if (m) {
        CK(cudaMemcpyAsync(d_src.p, src, m * 4, cudaMemcpyHostToDevice, s));
        CK(cudaMemcpyAsync(d_dst.p, dst, m * 4, cudaMemcpyHostToDevice, s));
    }
    // graph.cpp:57-61: the first edge (input order) with an endpoint >= n
    CK(cudaMemsetAsync(d_bad.p, 0xff, 8, s));
    k_gb_validate<<<blocks, 256, 0, s>>>(d_src.as<uint32_t>(), d_dst.as<uint32_t>(), m, n,
                                         d_bad.as<unsigned long long>());
    CKL("k_gb_validate");
    unsigned long long bad = 0;
    CK(cudaMemcpyAsync(&bad, d_bad.p, 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (bad < m)
        throw std::out_of_range("edge endpoint out of range: " + std::to_string(src[bad]) + " -> " +
                                std::to_string(dst[bad]));
    d_keys.ensure(mm * 8, s);
    k_gb_keys<<<blocks, 256, 0, s>>>(d_src.as<uint32_t>(), d_dst.as<uint32_t>(), m, d_keys.as<unsigned long long>());
    CKL("k_gb_keys");
    d_src.release();
    d_dst.release();
    d_keys2.ensure(mm * 8, s);
    return graph_from_keys(n, d_keys, d_keys2, m, policy, s, blocks);
}

// ---------------------------------------------------------------------------
// R-MAT generation on the GPU, edge for edge the host generator's
// (host_graph.cpp rmat_edges): edge e comes from the mt19937_64 stream of its
// 2^20-edge chunk, seeded seed*0x9E37..15 + chunk*0xD1B5..03 + 1, one uniform
// double (53 high bits) per level, MSB first, quadrants a | b | c | rest.
// One thread per chunk (each stream is sequential); self-loops become kNoEdge
// keys, dropped after the sort.  mt19937_64: the published MT19937-64
// recurrence (n = 312, m = 156, matrix 0xB5026F5AA96619E9, the standard
// initialisation and tempering), restated here.
// ---------------------------------------------------------------------------
struct Mt64 {
    static constexpr int N = 312, M = 156;
    uint64_t mt[N];
    int idx;
    __device__ void seed(uint64_t s) {
        mt[0] = s;
        for (int i = 1; i < N; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
        idx = N;
    }
    __device__ void twist() {
        constexpr uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, MA = 0xB5026F5AA96619E9ULL;
        for (int i = 0; i < N; ++i) {
            const uint64_t x = (mt[i] & UM) | (mt[(i + 1) % N] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= MA;
            mt[i] = mt[(i + M) % N] ^ xa;
        }
        idx = 0;
    }
    __device__ uint64_t next() {
        if (idx >= N) twist();
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= y >> 43;
        return y;
    }
};

constexpr uint64_t kRmatChunk = 1ull << 20;  // host_graph.cpp rmat_edges kChunk

__global__ void __launch_bounds__(32) k_rmat_keys(uint32_t scale, uint64_t m, double a, double ab, double abc,
                                                  uint64_t seed, unsigned long long* __restrict__ keys) {
    const uint64_t ch = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t e0 = ch * kRmatChunk;
    if (e0 >= m) return;
    const uint64_t e1 = min(m, e0 + kRmatChunk);
    Mt64 rng;
    rng.seed(seed * 0x9E3779B97F4A7C15ULL + ch * 0xD1B54A32D192ED03ULL + 1);
    for (uint64_t e = e0; e < e1; ++e) {
        uint32_t x = 0, y = 0;
        for (uint32_t lvl = 0; lvl < scale; ++lvl) {
            const double r = __dmul_rn((double)(rng.next() >> 11), 0x1.0p-53);
            const uint32_t bit = 1u << (scale - 1 - lvl);
            if (r < a) {
            } else if (r < ab) {
                y |= bit;
            } else if (r < abc) {
                x |= bit;
            } else {
                x |= bit;
                y |= bit;
            }
        }
        keys[e] = x == y ? kNoEdge : (((unsigned long long)x << 32) | y);
    }
}

static tpa_host_graph* rmat_graph_gpu(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                                      uint64_t seed, int policy, int device) {
    if (scale == 0 || scale > 31) throw std::invalid_argument("rmat scale must be in [1, 31]");
    if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0))
        throw std::invalid_argument("rmat probabilities must be non-negative and sum <= 1");
    if (policy < 0 || policy > 2) throw std::invalid_argument("unknown dangling policy");
    const uint64_t n = uint64_t(1) << scale;
    if (n > 0xffffffffULL) throw std::invalid_argument("rmat scale too large for uint32 ids");
    const uint64_t m = n * edge_factor;
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    StreamGuard sg{s};
    DevBuf d_keys, d_keys2;
    const size_t mm = std::max<uint64_t>(m, 1);
    d_keys.ensure(mm * 8, s);
    const uint64_t nch = (m + kRmatChunk - 1) / kRmatChunk;
    if (nch) {
        k_rmat_keys<<<(unsigned)((nch + 31) / 32), 32, 0, s>>>(scale, m, a, a + b, a + b + c, seed,
                                                               d_keys.as<unsigned long long>());
        CKL("k_rmat_keys");
    }
    d_keys2.ensure(mm * 8, s);
    return graph_from_keys((uint32_t)n, d_keys, d_keys2, m, policy, s, 8 * sms);
}

}  // namespace tpa

extern "C" int tpa_host_graph_rmat_gpu(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                                       uint64_t seed, int policy, int device, tpa_host_graph** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output handle");
        *out = rmat_graph_gpu(scale, edge_factor, a, b, c, seed, policy, device);
    });
}

extern "C" int tpa_host_graph_build_gpu(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t m, int policy,
                                        int device, tpa_host_graph** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output handle");
        *out = build_graph_gpu(n, src, dst, m, policy, device);
    });
}
