// gather_micro.cu -- microbenchmark: random 256-B row gathers (the SpMM's
// access pattern at B = 32 fp64) through three paths, to find which one can
// keep the most requests in flight per SM on the B200.
//   A: LDG into registers (lane = column), U rows in flight per warp
//   B: cp.async.bulk (bulk-copy / TMA engine) of whole rows into a per-warp
//      shared-memory ring, one row per lane per instruction, mbarrier-tracked
//   C: cp.async (LDGSTS) 16 B per lane into the same ring
//   D: TMA tile::gather4 (cp.async.bulk.tensor.2d ... gather4): one request
//      fetches FOUR rows named by four indices (tensor map over [n][32] f64,
//      box 32 x 1); per warp a ring of S stages x 32 rows, lanes 0-7 issue
//      the 8 gather4 requests of a stage
// argv[1] = rows of X (default 2^20: 268 MB, partly L2-resident; 16777216 is
// C4's 4.3 GB share matrix)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_micro tools/gather_micro.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int B = 32;  // doubles per row (256 B)

template <int U>
__global__ void gather_ldg(const double* __restrict__ X, const uint32_t* __restrict__ idx, long long m, double* out) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long per = (m + nw - 1) / nw;
    const long long lo = warp * per, hi = min(m, lo + per);
    double s = 0.0;
    for (long long e = lo; e < hi; e += U) {
        double v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t u = e + j < hi ? __ldg(idx + e + j) : 0u;
            v[j] = __ldg(X + (size_t)u * B + lane);
        }
#pragma unroll
        for (int j = 0; j < U; ++j) s += v[j];
    }
    if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n LAB_WAIT:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra LAB_WAIT;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                     "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                 "r"((uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}

// B: each warp owns a ring of S stages x 32 rows; stage k's 32 rows are issued
// by the 32 lanes (one bulk copy each), completion on mbar[k].
template <int S>
__global__ void gather_bulk(const double* __restrict__ X, const uint32_t* __restrict__ idx, long long m, double* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    double* ring = reinterpret_cast<double*>(smem) + (size_t)w * S * 32 * B;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nwb * S * 32 * B * 8) + w * S;
    if (lane < S) mbar_init(&bars[lane], 1);
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long per = ((m + nw - 1) / nw + 31) / 32 * 32;
    const long long lo = warp * per, hi = min(m, lo + per);
    const long long nst = (hi > lo) ? (hi - lo + 31) / 32 : 0;
    auto issue = [&](long long k) {
        if (k >= nst) return;
        const int slot = (int)(k % S);
        const long long e = lo + k * 32 + lane;
        const int cnt = (int)min(32LL, hi - (lo + k * 32));
        if (lane == 0) mbar_expect_tx(&bars[slot], cnt * B * 8);
        __syncwarp();
        if (lane < cnt) bulk_g2s(ring + ((size_t)slot * 32 + lane) * B, X + (size_t)__ldg(idx + e) * B, B * 8, &bars[slot]);
    };
    for (int k = 0; k < S; ++k) issue(k);
    double s = 0.0;
    for (long long k = 0; k < nst; ++k) {
        const int slot = (int)(k % S);
        mbar_wait(&bars[slot], (uint32_t)((k / S) & 1));
        const int cnt = (int)min(32LL, hi - (lo + k * 32));
        for (int j = 0; j < cnt; ++j) s += ring[((size_t)slot * 32 + j) * B + lane];
        __syncwarp();
        issue(k + S);
    }
    if (s == 12345.678) out[0] = s;
}


// D: TMA gather4
template <int S>
__global__ void gather_g4(const __grid_constant__ CUtensorMap tm, const uint32_t* __restrict__ idx, long long m,
                          double* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    double* ring = reinterpret_cast<double*>(smem) + (size_t)w * S * 32 * B;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nwb * S * 32 * B * 8) + w * S;
    if (lane < S) mbar_init(&bars[lane], 1);
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long per = ((m + nw - 1) / nw + 31) / 32 * 32;
    const long long lo = warp * per, hi = min(m, lo + per);
    const long long nst = (hi > lo) ? (hi - lo + 31) / 32 : 0;
    auto issue = [&](long long k) {
        if (k >= nst) return;
        const int slot = (int)(k % S);
        const long long e = lo + k * 32 + lane;
        const uint32_t myi = e < hi ? __ldg(idx + e) : 0u;  // tail: row 0 (counted, harmless)
        const int q = lane * 4;
        const int r0 = __shfl_sync(0xffffffffu, myi, q & 31), r1 = __shfl_sync(0xffffffffu, myi, (q + 1) & 31);
        const int r2 = __shfl_sync(0xffffffffu, myi, (q + 2) & 31), r3 = __shfl_sync(0xffffffffu, myi, (q + 3) & 31);
        if (lane == 0) mbar_expect_tx(&bars[slot], 32 * B * 8);
        __syncwarp();
        if (lane < 8) {
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(ring + ((size_t)slot * 32 + q) * B);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(d), "l"(&tm), "r"(0), "r"(r0), "r"(r1), "r"(r2),
                "r"(r3), "r"((uint32_t)__cvta_generic_to_shared(&bars[slot]))
                : "memory");
        }
    };
    for (int k = 0; k < S; ++k) issue(k);
    double s = 0.0;
    for (long long k = 0; k < nst; ++k) {
        const int slot = (int)(k % S);
        mbar_wait(&bars[slot], (uint32_t)((k / S) & 1));
        const int cnt = (int)min(32LL, hi - (lo + k * 32));
        for (int j = 0; j < cnt; ++j) s += ring[((size_t)slot * 32 + j) * B + lane];
        __syncwarp();
        issue(k + S);
    }
    if (s == 12345.678) out[0] = s;
}

// C: cp.async 16 B per lane into a per-warp ring of S stages x R rows; lane
// pair (2 rows per instruction: lanes 0-15 row a, 16-31 row b), consumer reads
// lane = column (8 B) per row.
template <int S, int R>
__global__ void gather_ldgsts(const double* __restrict__ X, const uint32_t* __restrict__ idx, long long m, double* out) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double* ring = reinterpret_cast<double*>(smem) + (size_t)w * S * R * B;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long per = ((m + nw - 1) / nw + R - 1) / R * R;
    const long long lo = warp * per, hi = min(m, lo + per);
    const long long nst = (hi > lo) ? (hi - lo + R - 1) / R : 0;
    const int half = lane >> 4, q = lane & 15;  // row within pair, 16-byte chunk
    auto issue = [&](long long k) {
        if (k < nst) {
            const int slot = (int)(k % S);
            const long long e0 = lo + k * R;
            // indices for this stage: lane j < R holds idx[e0 + j]
            const uint32_t myidx = (lane < R && e0 + lane < hi) ? __ldg(idx + e0 + lane) : 0u;
#pragma unroll
            for (int p = 0; p < R / 2; ++p) {
                const int j = 2 * p + half;
                const uint32_t u = __shfl_sync(0xffffffffu, myidx, j);
                if (e0 + j < hi) {
                    const double* src = X + (size_t)u * B + q * 2;
                    const uint32_t d = (uint32_t)__cvta_generic_to_shared(ring + ((size_t)slot * R + j) * B + q * 2);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
                }
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
#pragma unroll
    for (int k = 0; k < S - 1; ++k) issue(k);
    double s = 0.0;
    for (long long k = 0; k < nst; ++k) {
        issue(k + S - 1);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(S - 1) : "memory");
        __syncwarp();
        const int slot = (int)(k % S);
        const int cnt = (int)min((long long)R, hi - (lo + k * R));
        for (int j = 0; j < cnt; ++j) s += ring[((size_t)slot * R + j) * B + lane];
        __syncwarp();
    }
    if (s == 12345.678) out[0] = s;
}

int main(int argc, char** argv) {
    const uint32_t n = argc > 1 ? (uint32_t)atoll(argv[1]) : (1u << 20);
    const long long m = 16586831;
    double* X;
    uint32_t* idx;
    double* out;
    CK(cudaMalloc(&X, (size_t)n * B * 8));
    CK(cudaMalloc(&idx, m * 4));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(X, 0, (size_t)n * B * 8));
    std::vector<uint32_t> h(m);
    std::mt19937_64 rng(1);
    // skewed like R-MAT: mix of hub-heavy and uniform sources
    for (long long i = 0; i < m; ++i) {
        const double r = (rng() >> 11) * 0x1p-53;
        h[i] = r < 0.5 ? (uint32_t)(rng() % (n / 64)) : (uint32_t)(rng() % n);
    }
    CK(cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 5;
        printf("%-34s %8.3f ms  %6.1f G gathers/s  %7.0f GB/s\n", name, ms, m / ms / 1e6, m * 256.0 / ms / 1e6);
    };
    for (int warps : {16, 32, 48, 64}) {
        char nm[64];
        snprintf(nm, 64, "LDG U=16, %d warps/SM", warps);
        timeit(nm, [&] { gather_ldg<16><<<sms * warps / 8, 256>>>(X, idx, m, out); });
    }
    {
        // L2 persistence: the hot rows (the first n/64, half of all gathers) in a
        // persisting access-policy window, the rest streaming
        int maxp = 0;
        CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0));
        const size_t hot = (size_t)(n / 64) * B * 8;
        printf("max persisting L2 %d bytes; hot region %zu bytes\n", maxp, hot);
        for (double frac : {0.5, 1.0}) {
            const size_t win = std::min<size_t>(hot, (size_t)maxp);
            CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)(maxp * frac)));
            cudaStreamAttrValue av{};
            av.accessPolicyWindow.base_ptr = X;
            av.accessPolicyWindow.num_bytes = win;
            av.accessPolicyWindow.hitRatio = 1.0f;
            av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cudaStream_t st;
            CK(cudaStreamCreate(&st));  // blocking: orders with the timing events on the legacy stream
            CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
            for (int warps : {32, 48}) {
                char nm[80];
                snprintf(nm, 80, "LDG U=16 %dw persist %.0f%%", warps, frac * 100);
                timeit(nm, [&] { gather_ldg<16><<<sms * warps / 8, 256, 0, st>>>(X, idx, m, out); });
            }
            av.accessPolicyWindow.num_bytes = 0;
            CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
            CK(cudaStreamDestroy(st));
            CK(cudaCtxResetPersistingL2Cache());
        }
    }
    auto ring = [&](auto kern, int S, int R, int wpb) {
        const size_t smem = (size_t)wpb * S * R * B * 8;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, wpb * 32, smem);
        char nm[80];
        snprintf(nm, 80, "LDGSTS S=%d R=%d %dw x %d CTA/SM", S, R, wpb, occ);
        timeit(nm, [&] { kern<<<sms * occ, wpb * 32, smem>>>(X, idx, m, out); });
    };
    ring(gather_ldgsts<3, 16>, 3, 16, 4);
    ring(gather_ldgsts<4, 16>, 4, 16, 4);
    ring(gather_ldgsts<3, 8>, 3, 8, 4);
    ring(gather_ldgsts<4, 8>, 4, 8, 4);
    ring(gather_ldgsts<6, 8>, 6, 8, 4);
    ring(gather_ldgsts<8, 8>, 8, 8, 2);
    ring(gather_ldgsts<3, 32>, 3, 32, 2);
    printf("X: %u rows (%.0f MB)\n", n, n * 256.0 / 1e6);
    {
        // tensor map over X as [n][32] f64, box 32 x 1 (gather4 takes 4 rows)
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                                 CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                                 CUtensorMapFloatOOBfill)>(fn);
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)B, (cuuint64_t)n};
        cuuint64_t strides[1] = {(cuuint64_t)B * 8};
        cuuint32_t box[2] = {(cuuint32_t)B, 1};
        cuuint32_t es[2] = {1, 1};
        for (auto prom : {CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B}) {
            CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, X, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, prom,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) {
                printf("cuTensorMapEncodeTiled failed %d\n", (int)r);
                break;
            }
            for (int S : {2, 4}) {
                for (int wpb : {4, 8}) {
                    const size_t smem = (size_t)wpb * S * 32 * B * 8 + wpb * S * 8;
                    auto k = S == 2 ? gather_g4<2> : gather_g4<4>;
                    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
                        cudaGetLastError();
                        continue;
                    }
                    int occ = 0;
                    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, wpb * 32, smem);
                    if (occ < 1) continue;
                    char nm[80];
                    snprintf(nm, 80, "gather4 S=%d %dw x %d CTA/SM prom%d", S, wpb, occ, (int)prom);
                    timeit(nm, [&] { k<<<sms * occ, wpb * 32, smem>>>(tm, idx, m, out); });
                }
            }
        }
    }
    for (int S : {2, 4}) {
        for (int wpb : {4, 8}) {
            const size_t smem = (size_t)wpb * S * 32 * B * 8 + wpb * S * 8;
            auto k = S == 2 ? gather_bulk<2> : gather_bulk<4>;
            if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
                cudaGetLastError();
                continue;
            }
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, wpb * 32, smem);
            char nm[80];
            snprintf(nm, 80, "bulk S=%d, %d warps/CTA x %d CTA/SM", S, wpb, occ);
            timeit(nm, [&] { k<<<sms * occ, wpb * 32, smem>>>(X, idx, m, out); });
        }
    }
    return 0;
}
