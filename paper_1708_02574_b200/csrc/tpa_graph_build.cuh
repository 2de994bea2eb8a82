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

static tpa_host_graph* build_graph_gpu(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t m, int policy,
                                       int device) {
    if (n == 0) throw std::invalid_argument("graph must have at least one node");
    if (policy < 0 || policy > 2) throw std::invalid_argument("unknown dangling policy");
    if (m && (!src || !dst)) throw std::invalid_argument("null edge arrays");
    DeviceGuard dg(device);
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    };
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const int blocks = 8 * sms;
    std::vector<uint64_t> off(n + 1ull);
    std::vector<uint32_t> tgt, dang;
    {
        StreamGuard sg{s};  // destroyed after the buffers (their frees are ordered on s)
        DevBuf d_src, d_dst, d_bad, d_keys, d_keys2, d_m, d_deg, d_cnt, d_off, d_flag, d_pre, d_tgt, d_dang, temp;
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
        // graph.cpp:63-64: sort + unique
        d_keys.ensure(mm * 8, s);
        d_keys2.ensure(mm * 8, s);
        d_m.ensure(8, s);
        k_gb_keys<<<blocks, 256, 0, s>>>(d_src.as<uint32_t>(), d_dst.as<uint32_t>(), m,
                                         d_keys.as<unsigned long long>());
        CKL("k_gb_keys");
        d_src.release();
        d_dst.release();
        int bits = 1;
        while (bits < 32 && (1ull << bits) < n) ++bits;
        size_t t1 = 0, t2 = 0, t3 = 0;
        CK(cub::DeviceRadixSort::SortKeys(nullptr, t1, d_keys.as<unsigned long long>(),
                                          d_keys2.as<unsigned long long>(), (int64_t)m, 0, 32 + bits, s));
        CK(cub::DeviceSelect::Unique(nullptr, t2, d_keys2.as<unsigned long long>(), d_keys.as<unsigned long long>(),
                                     d_m.as<unsigned long long>(), (int64_t)m, s));
        d_cnt.ensure((n + 1ull) * 8, s);
        d_off.ensure((n + 1ull) * 8, s);
        d_flag.ensure((n + 1ull) * 4, s);
        d_pre.ensure((n + 1ull) * 4, s);
        CK(cub::DeviceScan::ExclusiveSum(nullptr, t3, d_cnt.as<unsigned long long>(), d_off.as<unsigned long long>(),
                                         (int64_t)n + 1, s));
        size_t t4 = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, t4, d_flag.as<uint32_t>(), d_pre.as<uint32_t>(), (int64_t)n + 1, s));
        temp.ensure(std::max(std::max(t1, t2), std::max(t3, t4)), s);
        if (m) {
            CK(cub::DeviceRadixSort::SortKeys(temp.p, t1, d_keys.as<unsigned long long>(),
                                              d_keys2.as<unsigned long long>(), (int64_t)m, 0, 32 + bits, s));
            CK(cub::DeviceSelect::Unique(temp.p, t2, d_keys2.as<unsigned long long>(), d_keys.as<unsigned long long>(),
                                         d_m.as<unsigned long long>(), (int64_t)m, s));
        } else {
            CK(cudaMemsetAsync(d_m.p, 0, 8, s));
        }
        // graph.cpp:67-82: degrees, dangling, repair, offsets, targets
        const int repair = policy == TPA_SELFLOOP;
        d_deg.ensure((size_t)n * 4, s);
        CK(cudaMemsetAsync(d_deg.p, 0, (size_t)n * 4, s));
        k_gb_degrees<<<blocks, 256, 0, s>>>(d_keys.as<unsigned long long>(), d_m.as<unsigned long long>(),
                                            d_deg.as<uint32_t>());
        CKL("k_gb_degrees");
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
        k_gb_scatter<<<blocks, 256, 0, s>>>(d_keys.as<unsigned long long>(), d_m.as<unsigned long long>(),
                                            d_pre.as<uint32_t>(), repair, d_tgt.as<uint32_t>());
        CKL("k_gb_scatter");
        k_gb_dangling<<<blocks, 256, 0, s>>>(d_flag.as<uint32_t>(), d_pre.as<uint32_t>(), n, repair,
                                             d_off.as<unsigned long long>(), d_dang.as<uint32_t>(),
                                             d_tgt.as<uint32_t>());
        CKL("k_gb_dangling");
        tgt.resize(m_out);
        dang.resize(n_dang);
        if (m_out) CK(cudaMemcpyAsync(tgt.data(), d_tgt.p, m_out * 4, cudaMemcpyDeviceToHost, s));
        if (n_dang) CK(cudaMemcpyAsync(dang.data(), d_dang.p, (size_t)n_dang * 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    return make_host_graph(n, policy, std::move(off), std::move(tgt), std::move(dang));
}

}  // namespace tpa

extern "C" int tpa_host_graph_build_gpu(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t m, int policy,
                                        int device, tpa_host_graph** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output handle");
        *out = build_graph_gpu(n, src, dst, m, policy, device);
    });
}
