// cpi_sweep1.cuh -- the first family sweep of a seed batch (B = 32 / 64) as a
// push from the seeds.
//
// x⁰ of column b is c on seed_b only, so x¹[v][b] = share⁰[seed_b][b] for
// each out-neighbour v of seed_b and 0 elsewhere: every (row, column) gets at
// most one term, so the pushed value IS the reference's ascending-order sum
// (0 + s), bit for bit, without touching the other ~16 M nonzeros.  Two
// kernels, because rows reached from several seeds are shared:
//   * k_s1_rows: zero the share rows the push will write, make their
//     accumulator rows valid (zeroed if new);
//   * k_s1_push: CTAs (chunk, column b) push column b -- acc += y,
//     share = keep*y/deg, frontier bits, exact fixed-point residual /
//     dangling mass per column; the last CTA advances the ColStates.
// Used for SelfLoop / Drop only: a Uniform spread would reach every row (and
// its dangling mass would feed later spreads through a different reduction
// grouping than the pull's).
#pragma once

#include "cpi_spmm5.cuh"

namespace tpa {

struct Sweep1Args {
    StepArgs s;
    unsigned long long* fx;  // [4B] exact per-column totals, zero between launches
    const uint64_t* __restrict__ out_off;
    const uint32_t* __restrict__ out_tgt;
    SeedList seeds;
    uint32_t* nz_out;
    uint32_t* acc_valid;
    uint32_t* ticket;  // zero between launches
};

template <int B>
__global__ void __launch_bounds__(256) k_s1_rows(Sweep1Args P) {
    const StepArgs& a = P.s;
    const uint32_t b = blockIdx.y;  // column; blockIdx.x strides over the seed's out-edges
    if (!a.state_in[b].active) return;
    const uint32_t seed = P.seeds.s[b];
    const uint64_t lo = __ldg(P.out_off + seed), hi = __ldg(P.out_off + seed + 1);
    // one row per warp: the lanes cover the B columns
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (uint64_t e = lo + blockIdx.x * (blockDim.x / 32) + w; e < hi; e += gridDim.x * (blockDim.x / 32)) {
        const uint32_t v = __ldg(P.out_tgt + e);
#pragma unroll
        for (int c = lane; c < B; c += 32) a.share_out[(size_t)v * B + c] = 0.0;
        const bool valid = (__ldcg(P.acc_valid + (v >> 5)) >> (v & 31)) & 1u;
        if (!valid) {
#pragma unroll
            for (int c = lane; c < B; c += 32) a.acc[(size_t)v * B + c] = 0.0;
            __syncwarp();
            if (lane == 0) atomicOr(P.acc_valid + (v >> 5), 1u << (v & 31));
        }
    }
}

template <int B>
__global__ void __launch_bounds__(256) k_s1_push(Sweep1Args P) {
    const StepArgs& a = P.s;
    const uint32_t b = blockIdx.y;
    const ColState st = a.state_in[b];
    __shared__ unsigned long long s_w[4 * 8];
    unsigned long long f0 = 0, f1 = 0, f2 = 0, f3 = 0;
    const bool want_dm = a.policy == kUniform;
    if (st.active) {
        const uint32_t seed = P.seeds.s[b];
        const uint64_t lo = __ldg(P.out_off + seed), hi = __ldg(P.out_off + seed + 1);
        const double sh0 = a.share_in[(size_t)seed * B + b];  // share⁰[seed][b] as the init wrote it
        for (uint64_t e = lo + blockIdx.x * blockDim.x + threadIdx.x; e < hi; e += (uint64_t)gridDim.x * blockDim.x) {
            const uint32_t v = __ldg(P.out_tgt + e);
            const size_t ix = (size_t)v * B + b;
            const double yy = sh0;                             // the row sum: one term (graph.cpp:249-259)
            a.acc[ix] = dadd(a.acc[ix], yy);                   // cpi.cpp:50
            const uint32_t d = __ldg(a.deg + v);
            a.share_out[ix] = d ? ddiv(dmul(a.keep, yy), (double)d) : 0.0;  // graph.cpp:222
            if (yy != 0.0) atomicOr(P.nz_out + (v >> 5), 1u << (v & 31));
            fx_add(f0, f1, yy);
            if (want_dm && d == 0) fx_add(f2, f3, yy);
        }
    }
    fx_cta_flush(f0, f1, f2, f3, s_w, P.fx + 4 * b);
    // the last CTA advances every column's ColState from the exact totals
    __shared__ uint32_t s_ticket;
    if (threadIdx.x == 0) {
        __threadfence();
        s_ticket = atomicAdd(P.ticket, 1u);
    }
    __syncthreads();
    if (s_ticket != gridDim.x * gridDim.y - 1) return;
    __threadfence();
    for (int bb = threadIdx.x; bb < B; bb += blockDim.x) {
        const ColState st = a.state_in[bb];
        unsigned long long* f = P.fx + 4 * bb;
        ColState sc = st;
        if (sc.active) {
            const double res = fx_decode(atomicAdd(&f[0], 0ull), atomicAdd(&f[1], 0ull));
            const double dm = fx_decode(atomicAdd(&f[2], 0ull), atomicAdd(&f[3], 0ull));
            sc.residual = res;
            sc.iters = a.step;
            sc.converged = res < a.eps;
            sc.active = !sc.converged && (a.terminal < 0 || (int64_t)a.step < a.terminal);
            sc.has_spread = (a.policy == kUniform && dm != 0.0);
            sc.spread = sc.has_spread ? ddiv(dmul(a.keep, dm), (double)a.n) : 0.0;
        }
        a.state_out[bb] = sc;
        f[0] = f[1] = f[2] = f[3] = 0ull;
    }
    if (threadIdx.x == 0) *P.ticket = 0;
}

}  // namespace tpa
