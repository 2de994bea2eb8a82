// gather8_micro.cu -- microbenchmark: the SpMV's access pattern, random 8-byte
// gathers from an 8 MiB (L2-resident) vector, one per nnz, to find the floor
// of a B = 1 sweep on the B200.
//   A: LDG (lane = nnz) into registers, U in flight per lane, sum in registers
//   B: same with ld.global.cg (no L1 allocation)
//   C: cp.async 8 B into shared memory
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/gather8_micro tools/gather8_micro.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

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

int main() {
    const uint32_t n = 1 << 20;
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
        h[i] = r < 0.5 ? (uint32_t)(rng() % 16384) : (uint32_t)(rng() % n);
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
    // sorted-within-chunk indices: same multiset, better line reuse per instruction
    return 0;
}
