// tpa_relabel.cuh -- the relabelled twin of CSR(Ãᵀ) for B = 1 sweeps
// (PageRank preprocessing, cpi_run over all nodes).
//
// Why: a B = 1 sweep gathers one 8-byte share per nonzero.  Once the share
// vector outgrows the L2 (C4: 134 MB, C5: 2.1 GB) every miss fetches a 64-byte
// DRAM burst for 8 useful bytes, and the hot sources (R-MAT hubs) are spread
// over the whole id range, one per line: at C5 the SpMV moved 188 GB of DRAM
// per sweep against 31 GB of compulsory bytes (profiles/r01_ncu_c5.md).
// Numbering the nodes by out-degree (the number of times a node is gathered
// per sweep) packs the hot shares into few lines, so the L2 keeps them.
//
// How, without changing a single result bit:
//   * new id r = rank of the node in (out-degree desc, id asc) order;
//     perm[r] = old id, twin row r = old row perm[r];
//   * each twin row keeps the old row's nonzeros IN THE OLD ORDER (ascending
//     old source id), only the ids mapped: every row sum is the same sequence
//     of additions as before (the SpMV's per-row order depends on the row's
//     length and positions alone, cpi_spmv2.cuh);
//   * the twin's sweep sums the residual and dangling mass as exact per-row
//     fixed-point values (k_step_spmv2<true>), independent of its tiling;
//   * x⁽⁰⁾ = c/n everywhere is permutation invariant; the window accumulator
//     lives in twin order (the B = 1 workspace's own accumulator when the
//     caller's is elsewhere) and is scattered back (acc[perm[r]] = acc'[r])
//     once at the end of the run.
// Scores are therefore bitwise those of the original CSR under SelfLoop and
// Drop; the residual (and under Uniform the dangling-mass spread) differs
// from the per-tile sums of the original tiling in the last bits only.
// Used only for the dense-start B = 1 runs (no seed ids to map); queries keep
// the original CSR (their 128/256-byte share rows already use whole lines).
// TPA_RELABEL=0 disables it.  Included by tpa_gpu.cu.
#pragma once
// (included inside namespace tpa)

__global__ void k_rl_iota_deg(const uint32_t* __restrict__ deg, uint32_t n, uint32_t* __restrict__ keys,
                              uint32_t* __restrict__ ids) {
    for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < n; u += (uint64_t)gridDim.x * blockDim.x) {
        keys[u] = deg[u];
        ids[u] = (uint32_t)u;
    }
}

// newid[perm[r]] = r; len[r] = nnz of old row perm[r]; deg'[r] = deg[perm[r]]
__global__ void k_rl_map(const uint32_t* __restrict__ perm, const int64_t* __restrict__ rp,
                         const uint32_t* __restrict__ deg, uint32_t n, uint32_t* __restrict__ newid,
                         int64_t* __restrict__ len, uint32_t* __restrict__ deg2) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r <= n; r += (uint64_t)gridDim.x * blockDim.x) {
        if (r == n) {
            len[n] = 0;
            continue;
        }
        const uint32_t v = perm[r];
        newid[v] = (uint32_t)r;
        len[r] = rp[v + 1] - rp[v];
        deg2[r] = deg[v];
    }
}

// twin row r <- old row perm[r], ids mapped, order kept (one warp per row)
__global__ void k_rl_cols(const uint32_t* __restrict__ perm, const int64_t* __restrict__ rp,
                          const uint32_t* __restrict__ col, const uint32_t* __restrict__ newid,
                          const int64_t* __restrict__ rp2, uint32_t n, uint32_t* __restrict__ col2) {
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (uint64_t r = warp; r < n; r += nwarps) {
        const uint32_t v = perm[r];
        const int64_t lo = rp[v], hi = rp[v + 1], d = rp2[r] - lo;
        for (int64_t e = lo + lane; e < hi; e += 32) col2[e + d] = __ldg(newid + __ldg(col + e));
    }
}

__global__ void k_rl_unpermute(const double* __restrict__ acc2, const uint32_t* __restrict__ perm, uint32_t n,
                               double* __restrict__ acc) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x)
        acc[perm[r]] = acc2[r];
}

// Off unless TPA_RELABEL=1.  Measured on the B200 (tools/ab_pre.py, ms per
// PageRank sweep, original -> twin): C2 0.110 -> 0.129, C4 3.24 -> 3.91,
// C5 48.2 -> 53.1.  Packing the hubs does not pay: the twin's rows come in
// out-degree order too (a node's row follows its id), which clusters the
// long rows into the first tiles, and the DRAM-bound C5 sweep is limited by
// its random 64-byte bursts rather than by the hubs' reuse.  Kept as an
// experiment (results are bitwise those of the original CSR; tested).
static bool relabel_enabled(const tpa_graph* g) {
    static const bool on = [] {
        const char* e = std::getenv("TPA_RELABEL");
        return e && e[0] == '1';
    }();
    (void)g;
    return on;
}

// The twin, built on first use (one-time cost: a CUB sort of n degrees, one
// pass over the nonzeros, the SpMV tiling of the twin on the host).
static Relabel* relabel_view(tpa_graph* g) {
    if (!relabel_enabled(g) || g->part) return nullptr;
    if (g->rl) return g->rl.get();
    const cudaStream_t& s = g->stream;  // DevBufs keep a pointer to their stream
    const uint32_t n = g->n;
    const uint64_t m = g->m;
    auto rl = std::make_unique<Relabel>();
    const int blocks = 8 * g->num_sms;
    {
        DevBuf keys, keys2, ids, newid, len;
        keys.ensure((size_t)n * 4, s);
        keys2.ensure((size_t)n * 4, s);
        ids.ensure((size_t)n * 4, s);
        rl->perm.ensure((size_t)n * 4, s);
        k_rl_iota_deg<<<blocks, 256, 0, s>>>(g->deg.as<uint32_t>(), n, keys.as<uint32_t>(), ids.as<uint32_t>());
        CKL("k_rl_iota_deg");
        size_t t1 = 0;
        CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, t1, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                                     ids.as<uint32_t>(), rl->perm.as<uint32_t>(), (int64_t)n, 0, 32,
                                                     s));
        DevBuf temp;
        temp.ensure(t1, s);
        CK(cub::DeviceRadixSort::SortPairsDescending(temp.p, t1, keys.as<uint32_t>(), keys2.as<uint32_t>(),
                                                     ids.as<uint32_t>(), rl->perm.as<uint32_t>(), (int64_t)n, 0, 32,
                                                     s));
        keys.release();
        keys2.release();
        ids.release();
        newid.ensure((size_t)n * 4, s);
        len.ensure((n + 1ull) * 8, s);
        rl->deg.ensure((size_t)n * 4, s);
        rl->row_ptr.ensure((n + 1ull) * 8, s);
        k_rl_map<<<blocks, 256, 0, s>>>(rl->perm.as<uint32_t>(), g->row_ptr.as<int64_t>(), g->deg.as<uint32_t>(), n,
                                        newid.as<uint32_t>(), len.as<int64_t>(), rl->deg.as<uint32_t>());
        CKL("k_rl_map");
        size_t t2 = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, t2, len.as<int64_t>(), rl->row_ptr.as<int64_t>(), (int64_t)n + 1,
                                         s));
        temp.ensure(t2, s);
        CK(cub::DeviceScan::ExclusiveSum(temp.p, t2, len.as<int64_t>(), rl->row_ptr.as<int64_t>(), (int64_t)n + 1,
                                         s));
        rl->col.ensure(std::max<uint64_t>(m, 1) * 4, s);
        k_rl_cols<<<blocks, 256, 0, s>>>(rl->perm.as<uint32_t>(), g->row_ptr.as<int64_t>(), g->col.as<uint32_t>(),
                                         newid.as<uint32_t>(), rl->row_ptr.as<int64_t>(), n, rl->col.as<uint32_t>());
        CKL("k_rl_cols");
        g->launches += 4;
    }
    std::vector<int64_t> rp(n + 1ull);
    CK(cudaMemcpyAsync(rp.data(), rl->row_ptr.p, (n + 1ull) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    auto mv = build_items(rp, n, g->mv_shape.nnz, (uint32_t)g->mv_shape.rows, g->mv_shape.nnz);
    rl->mv.n_items = (uint32_t)mv.size();
    rl->mv.n_groups = (rl->mv.n_items + kGroupItems - 1) / kGroupItems;
    rl->mv.items.ensure(mv.size() * sizeof(uint2), s);
    CK(cudaMemcpyAsync(rl->mv.items.p, mv.data(), mv.size() * sizeof(uint2), cudaMemcpyHostToDevice, s));
    std::vector<longlong2> nr(mv.size());
    for (size_t i = 0; i < mv.size(); ++i) {
        const uint32_t rb = mv[i].x, re = mv[i].y & ~kLongFlag;
        nr[i] = make_longlong2(rp[rb], rp[re]);
    }
    rl->mv.item_nnz.ensure(nr.size() * sizeof(longlong2), s);
    CK(cudaMemcpyAsync(rl->mv.item_nnz.p, nr.data(), nr.size() * sizeof(longlong2), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    g->rl = std::move(rl);
    return g->rl.get();
}

