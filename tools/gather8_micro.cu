// gather8_micro.cu -- microbenchmark: the SpMV's access pattern, random 8-byte
// gathers from an 8 MiB (L2-resident) vector, one per nnz, to find the floor
// of a B = 1 sweep on the B200.
//   A: LDG (lane = nnz) into registers, U in flight per lane, sum in registers
//   B: same with ld.global.cg (no L1 allocation)
//   C: cp.async 8 B into shared memory
//   D: cp.async.bulk (TMA engine, bypasses the LSU/L1 path) of the 16-byte
//      aligned pair holding each gathered double, mbarrier-tracked, U stages
//      of 32 per warp in flight
// argv[1] = vector length in doubles (default 2^20 = 8 MiB, L2-resident;
// 16777216 = C4's 134 MB share vector)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/gather8_micro tools/gather8_micro.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

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

// D: per warp U stages x 32 lanes of 16-byte bulk copies
template <int U>
__global__ void gather_bulk16(const double* __restrict__ X, const uint32_t* __restrict__ idx, long long m, double* out) {
    __shared__ __align__(16) double sm[8][U][64];
    __shared__ uint64_t bar[8][U];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane < U) mbar_init(&bar[w][lane], 1);
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    double s = 0.0;
    uint32_t phase = 0;
    for (long long base = warp * U * 32; base < m; base += nw * U * 32) {
        uint32_t u[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const long long e = base + j * 32 + lane;
            u[j] = e < m ? __ldcs(idx + e) : 0u;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            if (lane == 0) mbar_expect_tx(&bar[w][j], 32 * 16);
            __syncwarp();
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(&sm[w][j][2 * lane]);
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(d),
                         "l"(X + (u[j] & ~1u)), "r"((uint32_t)__cvta_generic_to_shared(&bar[w][j])) : "memory");
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            mbar_wait(&bar[w][j], phase);
            s += sm[w][j][2 * lane + (u[j] & 1)];
        }
        phase ^= 1;
        __syncwarp();
    }
    if (s == 12345.678) out[0] = s;
}

template <int U, int MODE>
__global__ void gather(const double* __restrict__ X, const uint32_t* __restrict__ idx, long long m, double* out) {
    __shared__ double sm[8][U * 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    double s = 0.0;
    for (long long base = warp * U * 32; base < m; base += nw * U * 32) {
        uint32_t u[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const long long e = base + j * 32 + lane;
            u[j] = e < m ? __ldcs(idx + e) : 0u;
        }
        if (MODE == 2) {
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const uint32_t d = (uint32_t)__cvta_generic_to_shared(&sm[w][j * 32 + lane]);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(X + u[j]) : "memory");
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int j = 0; j < U; ++j) s += sm[w][j * 32 + lane];
            __syncwarp();
        } else {
            double v[U];
#pragma unroll
            for (int j = 0; j < U; ++j) v[j] = MODE == 0 ? __ldg(X + u[j]) : __ldcg(X + u[j]);
#pragma unroll
            for (int j = 0; j < U; ++j) s += v[j];
        }
    }
    if (s == 12345.678) out[0] = s;
}

// E: UL LDG gathers + UB 16-byte bulk copies per lane and iteration: does the
// TMA engine's request path add to the LSU's?
template <int UL, int UB>
__global__ void gather_mixed(const double* __restrict__ X, const uint32_t* __restrict__ idx, long long m, double* out) {
    __shared__ __align__(16) double sm[8][UB][64];
    __shared__ uint64_t bar[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) mbar_init(&bar[w], 1);
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    constexpr int U = UL + UB;
    double s = 0.0;
    uint32_t phase = 0;
    for (long long base = warp * U * 32; base < m; base += nw * U * 32) {
        uint32_t u[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const long long e = base + j * 32 + lane;
            u[j] = e < m ? __ldcs(idx + e) : 0u;
        }
        if (lane == 0) mbar_expect_tx(&bar[w], UB * 32 * 16);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < UB; ++j) {
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(&sm[w][j][2 * lane]);
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(d),
                         "l"(X + (u[UL + j] & ~1u)), "r"((uint32_t)__cvta_generic_to_shared(&bar[w])) : "memory");
        }
        double v[UL];
#pragma unroll
        for (int j = 0; j < UL; ++j) v[j] = __ldg(X + u[j]);
#pragma unroll
        for (int j = 0; j < UL; ++j) s += v[j];
        mbar_wait(&bar[w], phase);
#pragma unroll
        for (int j = 0; j < UB; ++j) s += sm[w][j][2 * lane + (u[UL + j] & 1)];
        phase ^= 1;
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
    CK(cudaMalloc(&X, (size_t)n * 8));
    CK(cudaMalloc(&idx, m * 4));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(X, 0, (size_t)n * 8));
    std::vector<uint32_t> h(m);
    std::mt19937_64 rng(1);
    for (long long i = 0; i < m; ++i) {
        const double r = (rng() >> 11) * 0x1p-53;
        h[i] = r < 0.5 ? (uint32_t)(rng() % (n / 64)) : (uint32_t)(rng() % n);
    }
    CK(cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice));
    printf("vector %u doubles (%.0f MB), %lld gathers\n", n, n * 8.0 / 1e6, m);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int r = 0; r < 20; ++r) launch();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 20;
        printf("%-34s %8.4f ms  %6.1f G gathers/s  %5.2f /clk/SM@1.9GHz\n", name, ms, m / ms / 1e6,
               m / ms / 1e6 / sms / 1.9);
    };
    for (int warps : {16, 32, 48, 64}) {
        char nm[64];
        snprintf(nm, 64, "LDG U=16 %d w/SM", warps);
        timeit(nm, [&] { gather<16, 0><<<sms * warps / 8, 256>>>(X, idx, m, out); });
        snprintf(nm, 64, "LDG.cg U=16 %d w/SM", warps);
        timeit(nm, [&] { gather<16, 1><<<sms * warps / 8, 256>>>(X, idx, m, out); });
        snprintf(nm, 64, "LDG U=8 %d w/SM", warps);
        timeit(nm, [&] { gather<8, 0><<<sms * warps / 8, 256>>>(X, idx, m, out); });
        snprintf(nm, 64, "LDGSTS U=16 %d w/SM", warps);
        timeit(nm, [&] { gather<16, 2><<<sms * warps / 8, 256>>>(X, idx, m, out); });
    }
    for (int warps : {16, 32, 48}) {
        char nm[64];
        snprintf(nm, 64, "BULK16 U=8 %d w/SM", warps);
        timeit(nm, [&] { gather_bulk16<8><<<sms * warps / 8, 256>>>(X, idx, m, out); });
        snprintf(nm, 64, "BULK16 U=4 %d w/SM", warps);
        timeit(nm, [&] { gather_bulk16<4><<<sms * warps / 8, 256>>>(X, idx, m, out); });
    }
    for (int warps : {32, 48, 64}) {
        char nm[64];
        snprintf(nm, 64, "MIXED LDG 14 + BULK 2 %d w/SM", warps);
        timeit(nm, [&] { gather_mixed<14, 2><<<sms * warps / 8, 256>>>(X, idx, m, out); });
        snprintf(nm, 64, "MIXED LDG 12 + BULK 4 %d w/SM", warps);
        timeit(nm, [&] { gather_mixed<12, 4><<<sms * warps / 8, 256>>>(X, idx, m, out); });
        snprintf(nm, 64, "MIXED LDG 6 + BULK 2 %d w/SM", warps);
        timeit(nm, [&] { gather_mixed<6, 2><<<sms * warps / 8, 256>>>(X, idx, m, out); });
    }
    return 0;
}
