// tpa_part.cuh -- row-partitioned CPI across GPUs (the north star's multi-GPU
// layout): B = 1 runs (PageRank / preprocess / cpi_run) over a CSR(Ãᵀ) whose
// rows are split into nnz-balanced ranges, one per GPU, with one exchange per
// sweep:
//   * every partition sweeps its own rows with the unchanged K2 kernel
//     (cpi_spmv2.cuh), reading the full share vector (padded global layout,
//     PartInfo) and writing its own slice of the next one;
//   * the residual / dangling totals are exact fixed-point integers, so the
//     sum of every partition's limbs gives the one-GPU totals bit for bit,
//     and k_part_finalize advances the same ColState everywhere;
//   * each partition's limbs ride at the end of its span of the share buffer,
//     so ONE in-place all-gather per sweep moves shares and totals (a sweep
//     without a next iterate -- the terminal one -- all-reduces the limbs).
// Three transports with one driver (run_cpi_part):
//   * one process per GPU over CUDA IPC -- the fused exchange: each rank maps
//     its peers' share buffers and the sweep epilogue stores every share (and
//     the tile limbs) straight into them, so the exchange rides on the
//     sweep's own stores (over NVLink between GPUs) instead of a collective
//     after it; ranks meet per sweep on interprocess events ordered by a
//     host-side stage counter (IpcState);
//   * one process per GPU over NCCL (in-place ncclAllGather of the span) on
//     the partition's stream;
//   * one process driving all partitions (tpa_group): stream-ordered peer
//     copies (cudaMemcpyPeerAsync) and a limb-sum kernel, no host sync.
// Included at the end of tpa_gpu.cu.
#pragma once

#include <dlfcn.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <time.h>
#include <unistd.h>

#include <chrono>

namespace tpa {

// NCCL is resolved at first use, not linked: a process that imports torch
// after this library must still get torch's own libnccl.so.2 (same soname).
// An already-loaded libnccl.so.2 (torch's) is reused; else TPA_NCCL_LIB or
// the system library is opened.
struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId;
    decltype(&ncclCommInitRank) CommInitRank;
    decltype(&ncclAllReduce) AllReduce;
    decltype(&ncclAllGather) AllGather;
    decltype(&ncclCommDestroy) CommDestroy;
    decltype(&ncclGetErrorString) GetErrorString;
};

static const NcclApi& nccl() {
    static std::mutex mu;
    static NcclApi api{};
    static bool loaded = false;
    std::lock_guard<std::mutex> lk(mu);
    if (loaded) return api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) {
        const char* e = std::getenv("TPA_NCCL_LIB");
        h = dlopen(e ? e : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) throw std::runtime_error(std::string("NCCL unavailable: ") + dlerror());
    auto sym = [&](const char* name) {
        void* f = dlsym(h, name);
        if (!f) throw std::runtime_error(std::string("NCCL symbol missing: ") + name);
        return f;
    };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    loaded = true;
    return api;
}

#define NCK(x)                                                                                            \
    do {                                                                                                  \
        const ncclResult_t r_ = (x);                                                                      \
        if (r_ != ncclSuccess) throw cuda_error(std::string(#x) + ": " + nccl().GetErrorString(r_));      \
    } while (0)

static void part_comm_destroy(ncclComm_t c) {
    if (c) nccl().CommDestroy(c);
}

__global__ void k_indeg(const uint32_t* __restrict__ tgt, uint64_t m, uint32_t* __restrict__ indeg) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(indeg + tgt[e], 1u);
}

// Sort keys for partition [lo, hi): local row of in-range edges (others sort
// last), value = the source's index in the padded share layout (stride S).
__global__ void k_part_keys(const uint32_t* __restrict__ tgt, const uint32_t* __restrict__ src, uint64_t m,
                            uint32_t lo, uint32_t hi, const uint32_t* __restrict__ bounds, uint32_t G,
                            uint32_t S, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = tgt[e];
        if (t >= lo && t < hi) {
            const uint32_t u = src[e];
            uint32_t a = 0, b = G;  // largest r with bounds[r] <= u (skips empty partitions)
            while (b - a > 1) {
                const uint32_t mid = (a + b) >> 1;
                if (bounds[mid] <= u) a = mid;
                else b = mid;
            }
            keys[e] = t - lo;
            vals[e] = a * S + (u - bounds[a]);
        } else {
            keys[e] = 0xffffffffu;
            vals[e] = 0u;
        }
    }
}

struct LimbPtrs {
    const unsigned long long* p[64];
};

__global__ void k_sum_limbs(LimbPtrs src, uint32_t G, unsigned long long* __restrict__ total) {
    const int k = threadIdx.x;
    if (k >= 6) return;
    unsigned long long s = 0;
    for (uint32_t r = 0; r < G; ++r) s += src.p[r][k];
    total[k] = s;
}

// Row boundaries balanced by nnz and cut only where the whole graph's SpMV
// tiling (build_items) starts an item: the greedy tiling of a suffix that
// begins at an item start is that suffix of the whole tiling, so every
// partition sweeps exactly the whole graph's tiles and the per-tile residual
// partials -- hence the exact totals -- are the same for any partition count.
// Boundary k is the first cut point whose in-degree prefix reaches
// floor(m*k/G) (partition.py restates this).
static std::vector<uint32_t> partition_rows(const std::vector<uint64_t>& prefix, uint32_t n, uint32_t G) {
    const uint64_t m = prefix[n];
    std::vector<int64_t> rp(prefix.begin(), prefix.end());
    const MvShape sh = mv_shape(n);
    std::vector<uint2> items = build_items(rp, n, sh.nnz, (uint32_t)sh.rows, sh.nnz);
    std::vector<uint32_t> cuts;
    cuts.reserve(items.size() + 1);
    for (const uint2& it : items) cuts.push_back(it.x);
    cuts.push_back(n);
    std::sort(cuts.begin(), cuts.end());
    std::vector<uint64_t> cut_prefix(cuts.size());
    for (size_t i = 0; i < cuts.size(); ++i) cut_prefix[i] = prefix[cuts[i]];
    std::vector<uint32_t> b(G + 1, 0);
    b[G] = n;
    for (uint32_t k = 1; k < G; ++k) {
        const uint64_t target = (uint64_t)((unsigned __int128)m * k / G);
        const size_t i = std::lower_bound(cut_prefix.begin(), cut_prefix.end(), target) - cut_prefix.begin();
        const uint32_t v = i < cuts.size() ? cuts[i] : n;
        b[k] = std::min(n, std::max(b[k - 1], v));
    }
    return b;
}

// Partition `rank` of `nranks` of the graph given by its out-CSR.
static void build_part(tpa_graph* g, uint32_t n, uint64_t m, const uint64_t* out_offsets,
                       const uint32_t* out_targets, uint32_t nranks, uint32_t rank) {
    cudaStream_t s = g->stream;
    const int blocks = 8 * g->num_sms;
    DevBuf d_off, d_tgt, d_src, d_keys, d_vals, d_keys2, d_vals2, d_indeg, d_bounds;
    d_off.ensure((n + 1ull) * 8, s);
    d_tgt.ensure(std::max<uint64_t>(m, 1) * 4, s);
    d_indeg.ensure((size_t)n * 4, s);
    CK(cudaMemcpyAsync(d_off.p, out_offsets, (n + 1ull) * 8, cudaMemcpyHostToDevice, s));
    if (m) CK(cudaMemcpyAsync(d_tgt.p, out_targets, m * 4, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(d_indeg.p, 0, (size_t)n * 4, s));
    k_indeg<<<blocks, 256, 0, s>>>(d_tgt.as<uint32_t>(), m, d_indeg.as<uint32_t>());
    CKL("k_indeg");
    std::vector<uint32_t> indeg(n);
    CK(cudaMemcpyAsync(indeg.data(), d_indeg.p, (size_t)n * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<uint64_t> prefix(n + 1ull, 0);
    for (uint32_t v = 0; v < n; ++v) prefix[v + 1] = prefix[v] + indeg[v];

    auto P = std::make_unique<PartInfo>();
    P->nranks = nranks;
    P->rank = rank;
    P->n_global = n;
    P->m_global = m;
    P->bounds = partition_rows(prefix, n, nranks);
    uint32_t S = 1;
    for (uint32_t r = 0; r < nranks; ++r) S = std::max(S, P->rows(r));
    P->slice = S;
    P->stride = (S + kLimbPad + 31) / 32 * 32;  // word-aligned spans in the B > 1 frontier bitmaps
    const uint32_t lo = P->bounds[rank], hi = P->bounds[rank + 1], nl = hi - lo;
    const uint64_t ml = prefix[hi] - prefix[lo];

    d_src.ensure(std::max<uint64_t>(m, 1) * 4, s);
    d_keys.ensure(std::max<uint64_t>(m, 1) * 4, s);
    d_vals.ensure(std::max<uint64_t>(m, 1) * 4, s);
    d_keys2.ensure(std::max<uint64_t>(m, 1) * 4, s);
    d_vals2.ensure(std::max<uint64_t>(m, 1) * 4, s);
    d_bounds.ensure((nranks + 1ull) * 4, s);
    CK(cudaMemcpyAsync(d_bounds.p, P->bounds.data(), (nranks + 1ull) * 4, cudaMemcpyHostToDevice, s));
    k_expand_src<<<blocks, 256, 0, s>>>(d_off.as<uint64_t>(), n, d_src.as<uint32_t>());
    CKL("k_expand_src");
    k_part_keys<<<blocks, 256, 0, s>>>(d_tgt.as<uint32_t>(), d_src.as<uint32_t>(), m, lo, hi,
                                       d_bounds.as<uint32_t>(), nranks, P->stride, d_keys.as<uint32_t>(),
                                       d_vals.as<uint32_t>());
    CKL("k_part_keys");
    if (m) {
        // stable: the out-CSR order (ascending source) survives within a row
        size_t temp = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, temp, d_keys.as<uint32_t>(), d_keys2.as<uint32_t>(),
                                           d_vals.as<uint32_t>(), d_vals2.as<uint32_t>(), (int64_t)m, 0, 32, s));
        DevBuf d_temp;
        d_temp.ensure(temp, s);
        CK(cub::DeviceRadixSort::SortPairs(d_temp.p, temp, d_keys.as<uint32_t>(), d_keys2.as<uint32_t>(),
                                           d_vals.as<uint32_t>(), d_vals2.as<uint32_t>(), (int64_t)m, 0, 32, s));
    }
    g->col.ensure(std::max<uint64_t>(ml, 1) * 4, g->stream);
    if (ml) CK(cudaMemcpyAsync(g->col.p, d_vals2.p, ml * 4, cudaMemcpyDeviceToDevice, s));
    g->row_ptr.ensure((nl + 1ull) * 8, g->stream);
    k_row_ptr<<<blocks, 256, 0, s>>>(d_keys2.as<uint32_t>(), ml, nl, g->row_ptr.as<int64_t>());
    CKL("k_row_ptr");
    g->deg.ensure(std::max<size_t>((size_t)nl, 1) * 4, g->stream);
    if (nl) k_degrees<<<blocks, 256, 0, s>>>(d_off.as<uint64_t>() + lo, nl, g->deg.as<uint32_t>());
    CKL("k_degrees");
    std::vector<int64_t> rp(nl + 1ull);
    CK(cudaMemcpyAsync(rp.data(), g->row_ptr.p, (nl + 1ull) * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    g->launches += 6;
    g->n = nl;
    g->m = ml;
    g->part = std::move(P);
    build_schedules(g, rp, nl);
}

struct PartRun {
    double c = 0.15, eps = 1e-9;
    uint32_t start = 0;
    int64_t terminal = -1;
    const std::vector<uint32_t>* seeds = nullptr;  // sorted, unique; null: all nodes (PageRank)
    double* out = nullptr;                         // n_global scores (host, or device via UVA)
    ColState state{};
};

static unsigned long long* limbs_slot(Workspace& w, int slot) { return w.limbs.as<unsigned long long>() + slot * 6; }
static unsigned long long* limbs_total(Workspace& w) { return w.limbs.as<unsigned long long>() + 18; }

// The limbs a partition publishes for sweep `slot` (0/1 by parity, 2 = x⁰):
// at the end of its span of share buffer `share` when the sweep writes one,
// else in the workspace.
static unsigned long long* limbs_at(tpa_graph* g, int slot, int share) {
    Workspace& w = g->workspace(1);
    const PartInfo& P = *g->part;
    if (share < 0) return limbs_slot(w, slot);
    return reinterpret_cast<unsigned long long*>(w.share[share].as<double>() + (size_t)P.rank * P.stride + P.slice);
}

// ---- CUDA IPC transport ------------------------------------------------------
struct IpcBlob {
    uint64_t magic;
    uint32_t nranks, rank;
    cudaIpcMemHandle_t share[2], limbs;
    cudaIpcEventHandle_t ev[kIpcRing];
    char shm_name[64];
};
constexpr uint64_t kIpcMagic = 0x3130435049415054ull;  // "TPAIPC01"
static_assert(sizeof(IpcBlob) <= TPA_IPC_BLOB_BYTES, "IPC blob size");

static uint64_t* ipc_counter(IpcState& I, uint32_t r) { return const_cast<uint64_t*>(I.shm + (size_t)r * 8); }

// One exchange point: record this rank's event for the stage, publish the
// stage, wait (host) until every peer has published it -- i.e. enqueued its
// own record -- and make the stream wait on the peers' records.  A rank can
// re-record a ring slot only after every peer has passed the previous stage,
// so each wait refers to the matching record.
static void ipc_exchange(tpa_graph* g) {
    IpcState& I = *g->part->ipc;
    const PartInfo& P = *g->part;
    if (!I.attached) throw std::logic_error("IPC partition used before tpa_part_ipc_attach");
    const uint64_t st = ++I.stage;
    const int slot = (int)(st % kIpcRing);
    CK(cudaEventRecord(I.own_ev[slot], g->stream));
    __atomic_store_n(ipc_counter(I, P.rank), st, __ATOMIC_RELEASE);
    for (uint32_t r = 0; r < P.nranks; ++r) {
        if (r == P.rank) continue;
        uint64_t* c = ipc_counter(I, r);
        uint64_t spins = 0;
        const auto t0 = std::chrono::steady_clock::now();
        while (__atomic_load_n(c, __ATOMIC_ACQUIRE) < st) {
            if (++spins < 4096) continue;
            sched_yield();
            if ((spins & 1023) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(600))
                throw std::runtime_error("IPC partition: rank " + std::to_string(r) + " never reached exchange " +
                                         std::to_string(st));
        }
        CK(cudaStreamWaitEvent(g->stream, I.peers[r].ev[slot], 0));
    }
}

static void ipc_teardown(tpa_graph* g) {
    IpcState& I = *g->part->ipc;
    cudaStreamSynchronize(g->stream);
    for (uint32_t r = 0; r < I.peers.size(); ++r) {
        if (r == g->part->rank) continue;
        IpcState::Peer& q = I.peers[r];
        for (double* p : q.share)
            if (p) cudaIpcCloseMemHandle(p);
        if (q.limbs) cudaIpcCloseMemHandle(q.limbs);
        for (cudaEvent_t e : q.ev)
            if (e) cudaEventDestroy(e);
    }
    for (cudaEvent_t e : I.own_ev)
        if (e) cudaEventDestroy(e);
    if (I.shm) munmap(const_cast<uint64_t*>(I.shm), I.shm_bytes);
    if (I.shm_owner) shm_unlink(I.shm_name);
    g->part->ipc.reset();
    cudaGetLastError();
}

// Every partition's totals for `slot`: with a share buffer, one in-place
// all-gather of the spans (shares + limbs) and a local sum of the G limb
// sets; without, an all-reduce of the limbs.  Stream-ordered, no host sync.
static void part_exchange(std::vector<tpa_graph*>& Pg, int slot, int share, bool stored = false) {
    const uint32_t G = Pg[0]->part->nranks;
    auto sum_local = [&](tpa_graph* g) {  // the G limb sets of g's gathered buffer
        Workspace& w = g->workspace(1);
        const PartInfo& P = *g->part;
        LimbPtrs lp{};
        for (uint32_t r = 0; r < G; ++r)
            lp.p[r] = reinterpret_cast<const unsigned long long*>(w.share[share].as<double>() + (size_t)r * P.stride +
                                                                   P.slice);
        k_sum_limbs<<<1, 32, 0, g->stream>>>(lp, G, limbs_total(w));
        CKL("k_sum_limbs");
        ++g->launches;
    };
    if (Pg.size() == 1 && Pg[0]->part->ipc) {
        tpa_graph* g = Pg[0];
        Workspace& w = g->workspace(1);
        PartInfo& P = *g->part;
        IpcState& I = *P.ipc;
        if (share >= 0) {
            if (!stored)  // x⁰: this rank's span (shares + limbs) into every peer's buffer
                for (uint32_t r = 0; r < G; ++r)
                    if (r != P.rank)
                        CK(cudaMemcpyAsync(I.peers[r].share[share] + (size_t)P.rank * P.stride,
                                           w.share[share].as<double>() + (size_t)P.rank * P.stride,
                                           (size_t)P.stride * 8, cudaMemcpyDeviceToDevice, g->stream));
            ipc_exchange(g);
            sum_local(g);
        } else {
            ipc_exchange(g);
            LimbPtrs lp{};
            for (uint32_t r = 0; r < G; ++r) lp.p[r] = I.peers[r].limbs + slot * 6;
            k_sum_limbs<<<1, 32, 0, g->stream>>>(lp, G, limbs_total(w));
            CKL("k_sum_limbs");
            ++g->launches;
        }
        return;
    }
    if (Pg.size() == 1) {
        tpa_graph* g = Pg[0];
        Workspace& w = g->workspace(1);
        PartInfo& P = *g->part;
        if (share >= 0) {
            if (P.comm) {
                double* buf = w.share[share].as<double>();
                NCK(nccl().AllGather(buf + (size_t)P.rank * P.stride, buf, P.stride, ncclDouble, P.comm, g->stream));
            }
            sum_local(g);
        } else if (P.comm) {
            NCK(nccl().AllReduce(limbs_slot(w, slot), limbs_total(w), 6, ncclUint64, ncclSum, P.comm, g->stream));
        } else {
            CK(cudaMemcpyAsync(limbs_total(w), limbs_slot(w, slot), 48, cudaMemcpyDeviceToDevice, g->stream));
        }
        return;
    }
    // in-process group: every partition waits for every partition's sweep
    std::vector<cudaEvent_t> ev(G);
    for (uint32_t r = 0; r < G; ++r) {
        DeviceGuard dg(Pg[r]->device);
        ev[r] = Pg[r]->take_event();
        CK(cudaEventRecord(ev[r], Pg[r]->stream));
    }
    LimbPtrs lp{};
    for (uint32_t r = 0; r < G; ++r) lp.p[r] = limbs_slot(Pg[r]->workspace(1), slot);
    for (uint32_t q = 0; q < G; ++q) {
        tpa_graph* g = Pg[q];
        DeviceGuard dg(g->device);
        for (uint32_t r = 0; r < G; ++r) CK(cudaStreamWaitEvent(g->stream, ev[r], 0));
        Workspace& w = g->workspace(1);
        if (share >= 0) {
            const PartInfo& P = *g->part;
            for (uint32_t r = 0; r < G && !stored; ++r) {  // stored: the sweep already wrote the peers
                if (r == q) continue;
                double* dst = w.share[share].as<double>() + (size_t)r * P.stride;
                const double* src = Pg[r]->workspace(1).share[share].as<double>() + (size_t)r * P.stride;
                CK(cudaMemcpyPeerAsync(dst, g->device, src, Pg[r]->device, (size_t)P.stride * 8, g->stream));
            }
            sum_local(g);
        } else {
            k_sum_limbs<<<1, 32, 0, g->stream>>>(lp, G, limbs_total(w));
            CKL("k_sum_limbs");
            ++g->launches;
        }
    }
    // the events are reusable once the waits are enqueued
    for (uint32_t r = 0; r < G; ++r) Pg[r]->event_pool.push_back(ev[r]);
}

// cpi_run / pagerank / preprocess over a row partition (B = 1).  All
// partitions run the same sweep sequence: the state they read back is the
// same (exact all-reduced totals).
static void run_cpi_part(std::vector<tpa_graph*>& Pg, PartRun& cfg) {
    const uint32_t G = Pg[0]->part->nranks;
    const uint32_t n = Pg[0]->part->n_global;
    const double keep = 1.0 - cfg.c;
    const int active0 = cfg.terminal != 0;
    std::vector<DevBuf> dx(Pg.size());
    std::vector<StepArgs> A(Pg.size());
    const bool ipc = Pg.size() == 1 && Pg[0]->part->ipc != nullptr;
    if (ipc) {  // every rank is done with the previous run's buffers before any peer store
        DeviceGuard dg(Pg[0]->device);
        ipc_exchange(Pg[0]);
    }
    // x⁰ (cpi.cpp:59-63), accumulated iff the window starts at 0
    for (size_t k = 0; k < Pg.size(); ++k) {
        tpa_graph* g = Pg[k];
        DeviceGuard dg(g->device);
        Workspace& w = g->workspace(1);
        w.limbs.ensure(24 * 8, g->stream);
        const PartInfo& P = *g->part;
        const uint32_t nl = g->n, lo = P.row_begin();
        double* acc0 = cfg.start == 0 ? w.acc.as<double>() : nullptr;
        if (!acc0 && nl) CK(cudaMemsetAsync(w.acc.p, 0, (size_t)nl * 8, g->stream));
        double weight = cfg.c / (double)n;
        if (cfg.seeds) {
            std::vector<double> x0(std::max<uint32_t>(nl, 1), 0.0);
            const double wgt = cfg.c / (double)cfg.seeds->size();
            for (uint32_t sd : *cfg.seeds)
                if (sd >= lo && sd < lo + nl) x0[sd - lo] = wgt;
            dx[k].ensure(x0.size() * 8, g->stream);
            CK(cudaMemcpyAsync(dx[k].p, x0.data(), x0.size() * 8, cudaMemcpyHostToDevice, g->stream));
            CK(cudaStreamSynchronize(g->stream));  // x0 is a local
        }
        if (nl) {
            const int nblk = grid_for(nl, 4 * kThreads, 4 * g->num_sms);
            k_init_dense<<<nblk, kThreads, 0, g->stream>>>(cfg.seeds ? dx[k].as<double>() : nullptr, weight, nl,
                                                           g->deg.as<uint32_t>(), keep,
                                                           w.share[0].as<double>() + (size_t)P.rank * P.stride,
                                                           acc0, w.fx.as<unsigned long long>(), nullptr, nullptr);
            CKL("k_init_dense");
        }
        k_init_finish<<<1, 1, 0, g->stream>>>(w.fx.as<unsigned long long>(), limbs_at(g, 2, 0), g->policy, keep,
                                              n, active0, w.state.as<ColState>(), nullptr, 0);
        CKL("k_init_finish");
        g->launches += 2;
        StepArgs& a = A[k];
        a = StepArgs{};
        a.row_ptr = g->row_ptr.as<int64_t>();
        a.col = g->col.as<uint32_t>();
        a.deg = g->deg.as<uint32_t>();
        a.items = g->mv.items.as<uint2>();
        a.n_items = g->mv.n_items;
        a.n = n;  // the graph's n: Uniform spread (graph.cpp:265-268)
        a.policy = g->policy;
        a.keep = keep;
        a.eps = cfg.eps;
        a.terminal = cfg.terminal;
        a.scale = 1.0;
        a.b_valid = 1;
        a.part = w.part.as<double>();
        a.gpart = w.gpart.as<double>();
        a.group_cnt = w.group_cnt.as<uint32_t>();
        a.done_cnt = w.done_cnt.as<uint32_t>();
    }
    part_exchange(Pg, 2, 0);
    for (size_t k = 0; k < Pg.size(); ++k) {
        tpa_graph* g = Pg[k];
        DeviceGuard dg(g->device);
        Workspace& w = g->workspace(1);
        StepArgs a = A[k];
        a.state_out = w.state.as<ColState>();
        k_part_finalize<<<1, 1, 0, g->stream>>>(limbs_total(w), a, 1, active0);
        CKL("k_part_finalize");
        ++g->launches;
    }

    const int64_t target = cfg.terminal >= 0 ? cfg.terminal : std::numeric_limits<int64_t>::max();
    const uint32_t est = sweeps_estimate(cfg.c, cfg.eps);
    uint64_t done = 0;
    int64_t chunk = std::min<int64_t>(target, (int64_t)est + 1);
    ColState hst{};
    while (chunk > 0) {
        for (int64_t j = 0; j < chunk; ++j) {
            const uint32_t i = (uint32_t)(done + 1 + j);
            const bool last = (int64_t)i == target;
            const bool inw = i >= cfg.start && (cfg.terminal < 0 || (int64_t)i <= cfg.terminal);
            // in-process groups: each sweep stores its shares into the peers' buffers
            const bool fused = (ipc ? G <= (uint32_t)kMaxPeerOut + 1
                                    : Pg.size() > 1 && Pg.size() <= (size_t)kMaxPeerOut + 1) && !last;
            for (size_t k = 0; k < Pg.size(); ++k) {
                tpa_graph* g = Pg[k];
                DeviceGuard dg(g->device);
                Workspace& w = g->workspace(1);
                const PartInfo& P = *g->part;
                StepArgs& a = A[k];
                g->peer_out = PeerOut{};
                if (fused && ipc)
                    for (uint32_t q = 0; q < G; ++q)
                        if (q != P.rank)
                            g->peer_out.p[g->peer_out.n++] = P.ipc->peers[q].share[i & 1] + (size_t)P.rank * P.stride;
                if (fused && !ipc)
                    for (size_t q = 0; q < Pg.size(); ++q)
                        if (q != k)
                            g->peer_out.p[g->peer_out.n++] =
                                Pg[q]->workspace(1).share[i & 1].as<double>() + (size_t)P.rank * P.stride;
                ColState* st = w.state.as<ColState>();
                a.step = i;
                a.share_in = w.share[(i - 1) & 1].as<double>();
                a.share_out = last ? nullptr : w.share[i & 1].as<double>() + (size_t)P.rank * P.stride;
                a.acc = inw ? w.acc.as<double>() : nullptr;
                a.state_in = st + ((i - 1) & 1);
                a.state_out = st + (i & 1);
                if (g->n) {
                    launch_step(g, w, a, nullptr, 1);
                } else {  // an empty partition publishes zero totals (to the peers too)
                    CK(cudaMemsetAsync(limbs_at(g, (int)(i & 1), last ? -1 : (int)(i & 1)), 0, 48, g->stream));
                    for (uint32_t q = 0; q < g->peer_out.n; ++q)
                        CK(cudaMemsetAsync(g->peer_out.p[q] + P.slice, 0, 48, g->stream));
                }
                g->peer_out = PeerOut{};
            }
            part_exchange(Pg, (int)(i & 1), last ? -1 : (int)(i & 1), fused);
            for (size_t k = 0; k < Pg.size(); ++k) {
                tpa_graph* g = Pg[k];
                DeviceGuard dg(g->device);
                Workspace& w = g->workspace(1);
                k_part_finalize<<<1, 1, 0, g->stream>>>(limbs_total(w), A[k], 0, 0);
                CKL("k_part_finalize");
                ++g->launches;
            }
        }
        done += chunk;
        if ((int64_t)done >= target) break;
        tpa_graph* g0 = Pg[0];
        {
            DeviceGuard dg(g0->device);
            CK(cudaMemcpyAsync(&hst, g0->workspace(1).state.as<ColState>() + (done & 1), sizeof(ColState),
                               cudaMemcpyDeviceToHost, g0->stream));
            CK(cudaStreamSynchronize(g0->stream));
        }
        if (!hst.active) break;
        chunk = std::min<int64_t>(target - (int64_t)done, 16);
    }
    // the accumulators, assembled into the caller's n-vector
    for (size_t k = 0; k < Pg.size(); ++k) {
        tpa_graph* g = Pg[k];
        DeviceGuard dg(g->device);
        Workspace& w = g->workspace(1);
        const PartInfo& P = *g->part;
        if (ipc) {
            // the accumulators through the share buffers: each rank stores its
            // rows into every rank's buffer, then reads all spans
            IpcState& I = *P.ipc;
            ipc_exchange(g);  // every rank past its last sweep
            for (uint32_t r = 0; r < G; ++r)
                if (g->n)
                    CK(cudaMemcpyAsync(I.peers[r].share[0] + (size_t)P.rank * P.stride, w.acc.p, (size_t)g->n * 8,
                                       cudaMemcpyDeviceToDevice, g->stream));
            ipc_exchange(g);
            for (uint32_t r = 0; r < G; ++r)
                if (P.rows(r))
                    CK(cudaMemcpyAsync(cfg.out + P.bounds[r], w.share[0].as<double>() + (size_t)r * P.stride,
                                       (size_t)P.rows(r) * 8, cudaMemcpyDefault, g->stream));
        } else if (Pg.size() == 1 && P.comm) {
            DevBuf pad;
            pad.ensure((size_t)G * P.slice * 8, g->stream);
            if (g->n)
                CK(cudaMemcpyAsync(pad.as<double>() + (size_t)P.rank * P.slice, w.acc.p, (size_t)g->n * 8,
                                   cudaMemcpyDeviceToDevice, g->stream));
            NCK(nccl().AllGather(pad.as<double>() + (size_t)P.rank * P.slice, pad.as<double>(), P.slice, ncclDouble,
                              P.comm, g->stream));
            for (uint32_t r = 0; r < G; ++r)
                if (P.rows(r))
                    CK(cudaMemcpyAsync(cfg.out + P.bounds[r], pad.as<double>() + (size_t)r * P.slice,
                                       (size_t)P.rows(r) * 8, cudaMemcpyDefault, g->stream));
        } else if (g->n) {
            CK(cudaMemcpyAsync(cfg.out + P.row_begin(), w.acc.p, (size_t)g->n * 8, cudaMemcpyDefault, g->stream));
        }
        CK(cudaMemcpyAsync(&cfg.state, w.state.as<ColState>() + (done & 1), sizeof(ColState),
                           cudaMemcpyDeviceToHost, g->stream));
    }
    for (tpa_graph* g : Pg) {
        DeviceGuard dg(g->device);
        CK(cudaStreamSynchronize(g->stream));
    }
}

}  // namespace tpa

struct tpa_group {
    std::vector<tpa_graph*> parts;
    std::vector<uint32_t> gdeg;  // global out-degrees (seed shares of query batches)
    std::mutex mu;
};

namespace tpa {

static void require_whole(const tpa_graph* g, const char* what) {
    if (g->part)
        throw std::invalid_argument(std::string(what) +
                                    " is not available on a row-partitioned graph (use a whole-graph replica)");
}

static void part_cpi_run(std::vector<tpa_graph*>& Pg, const uint32_t* seeds, uint64_t n_seeds, double c,
                         double eps, uint32_t start_iter, int64_t terminal_iter, double* out_scores,
                         uint32_t* iterations_run, int* converged, double* residual_l1) {
    const uint32_t n = Pg[0]->part->n_global;
    std::vector<uint32_t> hs;
    if (seeds) {
        if (n_seeds == 0) throw std::invalid_argument("seed set must not be empty");
        hs.assign(seeds, seeds + n_seeds);
        std::sort(hs.begin(), hs.end());
        if (std::adjacent_find(hs.begin(), hs.end()) != hs.end())
            throw std::invalid_argument("seed set contains duplicate ids");
    }
    validate_cpi(c, eps, start_iter, terminal_iter);
    if (seeds) validate_seed(hs.back(), n);
    if (!out_scores) throw std::invalid_argument("null output");
    PartRun cfg;
    cfg.c = c;
    cfg.eps = eps;
    cfg.start = start_iter;
    cfg.terminal = terminal_iter;
    cfg.seeds = seeds ? &hs : nullptr;
    cfg.out = out_scores;
    run_cpi_part(Pg, cfg);
    if (iterations_run) *iterations_run = cfg.state.iters;
    if (converged) *converged = cfg.state.converged;
    if (residual_l1) *residual_l1 = cfg.state.residual;
}

static void part_preprocess(std::vector<tpa_graph*>& Pg, double c, double eps, uint32_t T, double* out) {
    if (T < 1) throw std::invalid_argument("stranger_start (T) must be at least 1");  // tpa.cpp:21-22
    validate_cpi(c, eps, T, -1);
    if (!out) throw std::invalid_argument("null output");
    PartRun cfg;
    cfg.c = c;
    cfg.eps = eps;
    cfg.start = T;
    cfg.terminal = -1;
    cfg.out = out;
    run_cpi_part(Pg, cfg);
}

// ---- row-partitioned query batches (B = 16 / 32 / 64) ------------------------
// The B-seed sweep K3 over the partitions: each partition pulls its rows from
// the padded global share layout [G*stride rows + a zero row][B], stores its
// rows' next shares (and frontier bits) into its own span, and publishes its
// exact residual totals as limbs; the spans and limbs are exchanged per sweep
// and k_part_finalize_b advances the same column states everywhere.  The rows'
// arithmetic is K3's, so the scores equal the whole-graph query_batch bit for
// bit (SelfLoop / Drop; a Uniform spread comes from per-block dangling sums,
// which a partition groups differently: equal within rounding).  tpa.cpp:61-86.
struct SeedShares {
    double v[64];
};

// node id -> row of the padded global share layout (owner r: the last
// partition starting at or before v, skipping empty ones; as k_part_keys)
struct PartMap {
    uint32_t bounds[kMaxPeerOut + 2];
    uint32_t G, stride;
    static PartMap of(const PartInfo& P) {
        PartMap m{};
        m.G = P.nranks;
        m.stride = P.stride;
        for (uint32_t r = 0; r <= P.nranks; ++r) m.bounds[r] = P.bounds[r];
        return m;
    }
    __device__ uint32_t padded(uint32_t v) const {
        uint32_t a = 0, b = G;
        while (b - a > 1) {
            const uint32_t mid = (a + b) >> 1;
            if (bounds[mid] <= v) a = mid;
            else b = mid;
        }
        return a * stride + (v - bounds[a]);
    }
};

// x⁰ of the batch: every partition writes every seed's share row at its owner's
// padded position (the whole x⁰ is known on the host: no exchange needed), the
// frontier bit, and -- for the seeds it owns -- the accumulator row.
__global__ void k_init_seeds_part(const SeedList seeds, SeedShares sh, uint32_t b_valid, int B, double c,
                                  PartMap pm, uint32_t lo, uint32_t hi, double* __restrict__ share0,
                                  double* __restrict__ acc0, uint32_t* __restrict__ nz0,
                                  uint32_t* __restrict__ acc_valid) {
    const int b = threadIdx.x;
    if (b >= (int)b_valid) return;
    const uint32_t seed = seeds.s[b];
    const uint32_t pr = pm.padded(seed);
    for (int k = 0; k < B; ++k) {
        const bool mine = k < (int)b_valid && seeds.s[k] == seed;
        share0[(size_t)pr * B + k] = mine ? sh.v[k] : 0.0;
        if (seed >= lo && seed < hi) acc0[(size_t)(seed - lo) * B + k] = mine ? c : 0.0;
    }
    atomicOr(nz0 + (pr >> 5), 1u << (pr & 31));
    if (seed >= lo && seed < hi) atomicOr(acc_valid + ((seed - lo) >> 5), 1u << ((seed - lo) & 31));
}

struct LimbSets {
    const unsigned long long* p[kMaxPeerOut + 1];
};

// The per-column states after a partitioned sweep: the exact sum of every
// partition's limbs, then K3's update (cpi.cpp:73-80).
__global__ void k_part_finalize_b(LimbSets L, uint32_t G, int B, StepArgs a) {
    const int b = threadIdx.x;
    if (b >= B) return;
    unsigned long long t[6] = {0, 0, 0, 0, 0, 0};
    for (uint32_t r = 0; r < G; ++r)
        for (int k = 0; k < 6; ++k) t[k] += L.p[r][6 * b + k];
    unsigned long long h0, l0, h1, l1;
    limbs_to_fx(t, h0, l0);
    limbs_to_fx(t + 3, h1, l1);
    ColState sc = a.state_in[b];
    if (sc.active) {
        const double res = fx_decode(h0, l0), dm = fx_decode(h1, l1);
        sc.residual = res;
        sc.iters = a.step;
        sc.converged = res < a.eps;
        sc.active = !sc.converged && (a.terminal < 0 || (int64_t)a.step < a.terminal);
        sc.has_spread = (a.policy == kUniform && dm != 0.0);
        sc.spread = sc.has_spread ? ddiv(dmul(a.keep, dm), (double)a.n) : 0.0;
    }
    a.state_out[b] = sc;
}

// One query batch over the in-process partitions Pg (all of one graph).
// stranger: n doubles (host or device, UVA), null for query_na; out: [Btot][n]
// seed-major on the device of Pg[0] (dev) or the host.
static void run_batch_part(std::vector<tpa_graph*>& Pg, const std::vector<uint32_t>& gdeg, const uint32_t* seeds,
                           uint32_t Btot, double c, double eps, uint32_t S, const double* stranger, double scale,
                           double* out, bool dev) {
    const uint32_t G = Pg[0]->part->nranks;
    if (Pg.size() != G) throw std::invalid_argument("a partitioned query batch needs every partition");
    if (G > (uint32_t)kMaxPeerOut + 1) throw std::invalid_argument("a partitioned query batch takes <= 16 partitions");
    const uint32_t n = Pg[0]->part->n_global;
    const double keep = 1.0 - c;
    for (uint32_t b = 0; b < Btot; ++b) validate_seed(seeds[b], n);
    // per partition: the stranger slice and (host output) a device staging buffer
    std::vector<DevBuf> str(G), limbs(G);
    DevBuf stage;
    double* out_dev = out;
    {
        DeviceGuard dg(Pg[0]->device);
        if (!dev) {
            stage.ensure((size_t)std::min<uint32_t>(Btot, 64) * n * 8, Pg[0]->stream);
            out_dev = stage.as<double>();
        }
    }
    for (uint32_t k = 0; k < G; ++k) {
        tpa_graph* g = Pg[k];
        DeviceGuard dg(g->device);
        limbs[k].ensure(64 * 6 * 8, g->stream);
        if (stranger && g->n) {
            str[k].ensure((size_t)g->n * 8, g->stream);
            CK(cudaMemcpyAsync(str[k].p, stranger + g->part->row_begin(), (size_t)g->n * 8, cudaMemcpyDefault,
                               g->stream));
        }
    }
    const int64_t terminal = (int64_t)S - 1;
    for (uint32_t b0 = 0; b0 < Btot; b0 += 64) {
        const uint32_t bv = std::min<uint32_t>(64, Btot - b0);
        const int B = std::max(16, batch_width(bv));
        SeedList sl{};
        SeedShares sh{};
        std::vector<ColState> st0(B);
        for (uint32_t b = 0; b < bv; ++b) {
            const uint32_t sd = seeds[b0 + b];
            sl.s[b] = sd;
            const uint32_t d = gdeg[sd];
            sh.v[b] = d ? (keep * c) / (double)d : 0.0;  // graph.cpp:222 (host IEEE double, no FMA)
            ColState& s = st0[b];
            s.iters = 0;
            s.converged = 0;
            s.residual = c;
            s.active = terminal != 0;
            s.has_spread = Pg[0]->policy == kUniform && d == 0;
            s.spread = s.has_spread ? (keep * c) / (double)n : 0.0;
        }
        for (int b = (int)bv; b < B; ++b) st0[b] = ColState{};
        double* out_b = dev ? out + (size_t)b0 * n : out_dev;
        std::vector<StepArgs> A(G);
        std::vector<MmArgs> M(G);
        for (uint32_t k = 0; k < G; ++k) {
            tpa_graph* g = Pg[k];
            DeviceGuard dg(g->device);
            Workspace& w = g->workspace(B);
            const PartInfo& P = *g->part;
            const size_t rows_sh = (size_t)G * P.stride;
            const size_t bm = (rows_sh + 31) / 32 * 4 + 4;
            CK(cudaMemsetAsync(w.nz[0].p, 0, bm, g->stream));
            CK(cudaMemsetAsync(w.acc_valid.p, 0, ((size_t)g->n + 31) / 32 * 4 + 4, g->stream));
            CK(cudaMemcpyAsync(w.state.p, st0.data(), B * sizeof(ColState), cudaMemcpyHostToDevice, g->stream));
            k_init_seeds_part<<<1, 64, 0, g->stream>>>(sl, sh, bv, B, c, PartMap::of(P), P.row_begin(),
                                                       P.row_begin() + g->n, w.share[0].as<double>(),
                                                       w.acc.as<double>(), w.nz[0].as<uint32_t>(),
                                                       w.acc_valid.as<uint32_t>());
            CKL("k_init_seeds_part");
            ++g->launches;
            StepArgs& a = A[k];
            a = StepArgs{};
            a.row_ptr = g->row_ptr.as<int64_t>();
            a.col = g->col.as<uint32_t>();
            a.deg = g->deg.as<uint32_t>();
            a.n = n;  // the graph's n: Uniform spread, and the seed-major output's row length
            a.policy = g->policy;
            a.keep = keep;
            a.eps = eps;
            a.terminal = terminal;
            a.scale = scale;
            a.b_valid = bv;
            a.stranger = stranger ? str[k].as<double>() : nullptr;
            a.acc = w.acc.as<double>();
            a.done_cnt = w.done_cnt.as<uint32_t>();
            MmArgs& ma = M[k];
            ma = MmArgs{};
            ma.seg_row = g->longs.seg_row.as<uint32_t>();
            ma.seg_lo = g->longs.seg_lo.as<int64_t>();
            ma.seg_long = g->longs.seg_long.as<uint32_t>();
            ma.long_first = g->longs.long_first.as<uint32_t>();
            ma.long_nseg = g->longs.long_nseg.as<uint32_t>();
            ma.long_cnt = w.long_cnt.as<uint32_t>();
            ma.seg_part = w.seg_part.as<double>();
            ma.n_segs = g->longs.n_segs;
            ma.n_blocks = g->n_blocks;
            ma.blocks = g->longs.blocks.as<uint2>();
            ma.zero_row = (uint32_t)rows_sh;
            ma.work_cnt = w.work_cnt.as<uint32_t>();
            ma.fx = w.fx.as<unsigned long long>();
            ma.acc_valid = w.acc_valid.as<uint32_t>();
            ma.limbs_out = limbs[k].as<unsigned long long>();
        }
        for (int64_t i = 1; i <= terminal; ++i) {
            const bool last = i == terminal;
            for (uint32_t k = 0; k < G; ++k) {
                tpa_graph* g = Pg[k];
                DeviceGuard dg(g->device);
                Workspace& w = g->workspace(B);
                const PartInfo& P = *g->part;
                const size_t bm = ((size_t)G * P.stride + 31) / 32 * 4 + 4;
                StepArgs& a = A[k];
                ColState* st = w.state.as<ColState>();
                a.step = (uint32_t)i;
                a.share_in = w.share[(i - 1) & 1].as<double>();
                a.share_out = last ? nullptr : w.share[i & 1].as<double>() + (size_t)P.rank * P.stride * B;
                a.out = last ? out_b + P.row_begin() : nullptr;
                a.state_in = st + ((i - 1) & 1) * B;
                a.state_out = st + (i & 1) * B;
                MmArgs& ma = M[k];
                ma.s = a;
                ma.nz_in = w.nz[(i - 1) & 1].as<uint32_t>();
                ma.nz_out = last ? nullptr : w.nz[i & 1].as<uint32_t>() + P.rank * P.stride / 32;
                if (!last) CK(cudaMemsetAsync(w.nz[i & 1].p, 0, bm, g->stream));
                if (g->n) {
                    launch_step(g, w, a, &ma, B);
                } else {  // an empty partition contributes nothing
                    CK(cudaMemsetAsync(limbs[k].p, 0, (size_t)B * 6 * 8, g->stream));
                }
            }
            // exchange: every partition's span (shares + frontier words) and limbs
            std::vector<cudaEvent_t> ev(G);
            for (uint32_t r = 0; r < G; ++r) {
                DeviceGuard dg(Pg[r]->device);
                ev[r] = Pg[r]->take_event();
                CK(cudaEventRecord(ev[r], Pg[r]->stream));
            }
            LimbSets ls{};
            for (uint32_t r = 0; r < G; ++r) ls.p[r] = limbs[r].as<unsigned long long>();
            for (uint32_t q = 0; q < G; ++q) {
                tpa_graph* g = Pg[q];
                DeviceGuard dg(g->device);
                for (uint32_t r = 0; r < G; ++r) CK(cudaStreamWaitEvent(g->stream, ev[r], 0));
                Workspace& w = g->workspace(B);
                if (!last) {
                    for (uint32_t r = 0; r < G; ++r) {
                        if (r == q) continue;
                        const PartInfo& Pr = *Pg[r]->part;
                        const uint32_t rows = Pr.rows(r);
                        if (!rows) continue;
                        Workspace& wr = Pg[r]->workspace(B);
                        const size_t row0 = (size_t)r * Pr.stride;
                        CK(cudaMemcpyPeerAsync(w.share[i & 1].as<double>() + row0 * B, g->device,
                                               wr.share[i & 1].as<double>() + row0 * B, Pg[r]->device,
                                               (size_t)rows * B * 8, g->stream));
                        CK(cudaMemcpyPeerAsync(w.nz[i & 1].as<uint32_t>() + row0 / 32, g->device,
                                               wr.nz[i & 1].as<uint32_t>() + row0 / 32, Pg[r]->device,
                                               ((size_t)rows + 31) / 32 * 4, g->stream));
                    }
                }
                StepArgs& a = A[q];
                k_part_finalize_b<<<1, 64, 0, g->stream>>>(ls, G, B, a);
                CKL("k_part_finalize_b");
                ++g->launches;
            }
            for (uint32_t r = 0; r < G; ++r) Pg[r]->event_pool.push_back(ev[r]);
        }
        if (!dev) {
            for (uint32_t k = 0; k < G; ++k) {
                DeviceGuard dg(Pg[k]->device);
                CK(cudaStreamSynchronize(Pg[k]->stream));
            }
            DeviceGuard dg(Pg[0]->device);
            CK(cudaMemcpy(out + (size_t)b0 * n, out_dev, (size_t)bv * n * 8, cudaMemcpyDeviceToHost));
        }
    }
    for (tpa_graph* g : Pg) {
        DeviceGuard dg(g->device);
        CK(cudaStreamSynchronize(g->stream));
    }
}

}  // namespace tpa

namespace tpa {

static tpa_graph* make_part_graph(uint32_t n, uint64_t m, const uint64_t* out_offsets, const uint32_t* out_targets,
                                  int policy, uint64_t fingerprint, int device, uint32_t nranks, uint32_t rank) {
    if (n == 0) throw std::invalid_argument("graph must have at least one node");
    if (policy < 0 || policy > 2) throw std::invalid_argument("unknown dangling policy");
    if (!out_offsets || (m && !out_targets)) throw std::invalid_argument("null graph arrays");
    if (out_offsets[n] != m) throw std::invalid_argument("out_offsets[n] != m");
    if (nranks == 0 || rank >= nranks) throw std::invalid_argument("rank must be in [0, nranks)");
    DeviceGuard dg(device);
    auto g = std::make_unique<tpa_graph>();
    g->device = device;
    g->policy = policy;
    g->fingerprint = fingerprint;
    CK(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    g->own_stream = true;
    build_part(g.get(), n, m, out_offsets, out_targets, nranks, rank);
    return g.release();
}

}  // namespace tpa

extern "C" {

int tpa_comm_unique_id(void* id_out) {
    return guard([&] {
        if (!id_out) throw std::invalid_argument("null output");
        ncclUniqueId id;
        NCK(nccl().GetUniqueId(&id));
        static_assert(sizeof(ncclUniqueId) == TPA_COMM_ID_BYTES, "NCCL unique id size");
        std::memcpy(id_out, &id, sizeof(id));
    });
}

int tpa_graph_create_part(uint32_t n, uint64_t m, const uint64_t* out_offsets, const uint32_t* out_targets,
                          int policy, uint64_t fingerprint, int device, uint32_t nranks, uint32_t rank,
                          const void* comm_id, tpa_graph** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output handle");
        if (nranks > 1 && !comm_id)
            throw std::invalid_argument("nranks > 1 needs a communicator id (tpa_comm_unique_id) or tpa_group_create");
        std::unique_ptr<tpa_graph, int (*)(tpa_graph*)> g(
            make_part_graph(n, m, out_offsets, out_targets, policy, fingerprint, device, nranks, rank),
            tpa_graph_destroy);
        if (comm_id) {
            DeviceGuard dg(device);
            ncclUniqueId id;
            std::memcpy(&id, comm_id, sizeof(id));
            NCK(nccl().CommInitRank(&g->part->comm, (int)nranks, id, (int)rank));
        }
        *out = g.release();
    });
}

int tpa_graph_create_part_ipc(uint32_t n, uint64_t m, const uint64_t* out_offsets, const uint32_t* out_targets,
                              int policy, uint64_t fingerprint, int device, uint32_t nranks, uint32_t rank,
                              void* blob_out, tpa_graph** out) {
    return guard([&] {
        if (!out || !blob_out) throw std::invalid_argument("null output");
        if (nranks - 1 > (uint32_t)kMaxPeerOut) throw std::invalid_argument("an IPC partition has 1..16 ranks");
        std::unique_ptr<tpa_graph, int (*)(tpa_graph*)> g(
            make_part_graph(n, m, out_offsets, out_targets, policy, fingerprint, device, nranks, rank),
            tpa_graph_destroy);
        DeviceGuard dg(device);
        PartInfo& P = *g->part;
        P.ipc = std::make_unique<IpcState>();
        IpcState& I = *P.ipc;
        I.peers.resize(nranks);
        // the exported buffers (cudaMalloc): the share ping-pong in the padded
        // global layout and the limb slots; workspace(1) keeps them
        auto w = std::make_unique<Workspace>();
        w->B = 1;
        const size_t nbs = (size_t)nranks * P.stride * sizeof(double);
        w->share[0].ensure_plain(nbs, g->stream);
        w->share[1].ensure_plain(nbs, g->stream);
        w->limbs.ensure_plain(24 * 8, g->stream);
        g->ws[1] = std::move(w);
        Workspace& ws = g->workspace(1);
        IpcBlob b{};
        b.magic = kIpcMagic;
        b.nranks = nranks;
        b.rank = rank;
        for (int k = 0; k < 2; ++k) CK(cudaIpcGetMemHandle(&b.share[k], ws.share[k].p));
        CK(cudaIpcGetMemHandle(&b.limbs, ws.limbs.p));
        for (int k = 0; k < kIpcRing; ++k) {
            CK(cudaEventCreateWithFlags(&I.own_ev[k], cudaEventDisableTiming | cudaEventInterprocess));
            CK(cudaIpcGetEventHandle(&b.ev[k], I.own_ev[k]));
        }
        IpcState::Peer& me = I.peers[rank];
        me.share[0] = ws.share[0].as<double>();
        me.share[1] = ws.share[1].as<double>();
        me.limbs = ws.limbs.as<unsigned long long>();
        for (int k = 0; k < kIpcRing; ++k) me.ev[k] = I.own_ev[k];
        I.shm_bytes = (size_t)nranks * 64;
        if (rank == 0) {  // the stage counters: created by rank 0, opened by the others at attach
            static std::atomic<uint64_t> seq{0};
            struct timespec ts;
            clock_gettime(CLOCK_REALTIME, &ts);
            snprintf(I.shm_name, sizeof(I.shm_name), "/tpa_ipc_%d_%llu_%llx", (int)getpid(),
                     (unsigned long long)seq++, (unsigned long long)ts.tv_nsec);
            const int fd = shm_open(I.shm_name, O_CREAT | O_EXCL | O_RDWR, 0600);
            if (fd < 0) throw std::runtime_error(std::string("shm_open failed: ") + I.shm_name);
            I.shm_owner = true;
            const int rc = ftruncate(fd, (off_t)I.shm_bytes);
            void* p = rc == 0 ? mmap(nullptr, I.shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0) : MAP_FAILED;
            close(fd);
            if (p == MAP_FAILED) throw std::runtime_error("mapping the IPC stage counters failed");
            I.shm = static_cast<volatile uint64_t*>(p);
        }
        std::memcpy(b.shm_name, I.shm_name, sizeof(b.shm_name));
        std::memset(blob_out, 0, TPA_IPC_BLOB_BYTES);
        std::memcpy(blob_out, &b, sizeof(b));
        CK(cudaStreamSynchronize(g->stream));
        *out = g.release();
    });
}

int tpa_part_ipc_attach(tpa_graph* g, const void* blobs) {
    return guard([&] {
        if (!g || !blobs) throw std::invalid_argument("null argument");
        if (!g->part || !g->part->ipc) throw std::invalid_argument("not an IPC partition");
        PartInfo& P = *g->part;
        IpcState& I = *P.ipc;
        if (I.attached) throw std::invalid_argument("IPC partition already attached");
        DeviceGuard dg(g->device);
        const auto* all = static_cast<const unsigned char*>(blobs);
        IpcBlob b0;
        std::memcpy(&b0, all, sizeof(b0));
        for (uint32_t r = 0; r < P.nranks; ++r) {
            IpcBlob b;
            std::memcpy(&b, all + (size_t)r * TPA_IPC_BLOB_BYTES, sizeof(b));
            // (only rank 0's blob names the stage counters: it created them)
            if (b.magic != kIpcMagic || b.nranks != P.nranks || b.rank != r || b0.shm_name[0] != '/')
                throw std::invalid_argument("IPC blobs are not one partitioning's, in rank order");
            if (r == P.rank) continue;
            IpcState::Peer& q = I.peers[r];
            for (int k = 0; k < 2; ++k) {
                void* p = nullptr;
                CK(cudaIpcOpenMemHandle(&p, b.share[k], cudaIpcMemLazyEnablePeerAccess));
                q.share[k] = static_cast<double*>(p);
            }
            void* pl = nullptr;
            CK(cudaIpcOpenMemHandle(&pl, b.limbs, cudaIpcMemLazyEnablePeerAccess));
            q.limbs = static_cast<unsigned long long*>(pl);
            for (int k = 0; k < kIpcRing; ++k) CK(cudaIpcOpenEventHandle(&q.ev[k], b.ev[k]));
        }
        if (!I.shm_owner) {
            std::memcpy(I.shm_name, b0.shm_name, sizeof(I.shm_name));
            const int fd = shm_open(I.shm_name, O_RDWR, 0600);
            if (fd < 0) throw std::runtime_error(std::string("shm_open failed: ") + I.shm_name);
            void* p = mmap(nullptr, I.shm_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
            close(fd);
            if (p == MAP_FAILED) throw std::runtime_error("mapping the IPC stage counters failed");
            I.shm = static_cast<volatile uint64_t*>(p);
        }
        I.attached = true;
    });
}

int tpa_graph_part_info(const tpa_graph* g, uint32_t* nranks, uint32_t* rank, uint32_t* row_begin,
                        uint32_t* row_end, uint32_t* slice) {
    return guard([&] {
        if (!g) throw std::invalid_argument("null graph");
        const PartInfo* P = g->part.get();
        if (nranks) *nranks = P ? P->nranks : 1;
        if (rank) *rank = P ? P->rank : 0;
        if (row_begin) *row_begin = P ? P->row_begin() : 0;
        if (row_end) *row_end = P ? P->bounds[P->rank + 1] : g->n;
        if (slice) *slice = P ? P->slice : g->n;
    });
}

int tpa_group_create(uint32_t n, uint64_t m, const uint64_t* out_offsets, const uint32_t* out_targets, int policy,
                     uint64_t fingerprint, const int* devices, uint32_t nparts, tpa_group** out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output handle");
        if (nparts == 0 || nparts > 64) throw std::invalid_argument("a group has 1..64 partitions");
        if (!devices) throw std::invalid_argument("null device list");
        auto grp = std::make_unique<tpa_group>();
        grp->gdeg.resize(n);
        for (uint32_t u = 0; u < n; ++u) grp->gdeg[u] = (uint32_t)(out_offsets[u + 1] - out_offsets[u]);
        try {
            for (uint32_t r = 0; r < nparts; ++r)
                grp->parts.push_back(
                    make_part_graph(n, m, out_offsets, out_targets, policy, fingerprint, devices[r], nparts, r));
            // peer access between distinct devices (copies and the limb sum read peers)
            for (uint32_t a = 0; a < nparts; ++a)
                for (uint32_t b = 0; b < nparts; ++b) {
                    if (devices[a] == devices[b]) continue;
                    DeviceGuard dg(devices[a]);
                    int ok = 0;
                    CK(cudaDeviceCanAccessPeer(&ok, devices[a], devices[b]));
                    if (!ok) throw std::invalid_argument("group devices lack peer access");
                    const cudaError_t e = cudaDeviceEnablePeerAccess(devices[b], 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
                    cudaGetLastError();
                }
        } catch (...) {
            for (tpa_graph* g : grp->parts) tpa_graph_destroy(g);
            throw;
        }
        *out = grp.release();
    });
}

int tpa_group_destroy(tpa_group* grp) {
    return guard([&] {
        if (!grp) return;
        for (tpa_graph* g : grp->parts) tpa_graph_destroy(g);
        delete grp;
    });
}

int tpa_group_part(tpa_group* grp, uint32_t r, tpa_graph** out) {
    return guard([&] {
        if (!grp || !out) throw std::invalid_argument("null handle");
        if (r >= grp->parts.size()) throw std::out_of_range("partition index out of range");
        *out = grp->parts[r];
    });
}

int tpa_group_cpi_run(tpa_group* grp, const uint32_t* seeds, uint64_t n_seeds, double c, double eps,
                      uint32_t start_iter, int64_t terminal_iter, double* out_scores, uint32_t* iterations_run,
                      int* converged, double* residual_l1) {
    return guard([&] {
        if (!grp) throw std::invalid_argument("null group");
        std::lock_guard<std::mutex> lk(grp->mu);
        part_cpi_run(grp->parts, seeds, n_seeds, c, eps, start_iter, terminal_iter, out_scores, iterations_run,
                     converged, residual_l1);
    });
}

int tpa_group_query_batch(tpa_group* grp, const double* stranger, uint64_t fingerprint, double c, double eps,
                          uint32_t T, const uint32_t* seeds, uint32_t B, uint32_t S, double* out, int flags) {
    return guard([&] {
        if (!grp) throw std::invalid_argument("null group");
        std::lock_guard<std::mutex> lk(grp->mu);
        tpa_graph* g0 = grp->parts[0];
        const bool na = flags & TPA_QUERY_NA;
        // tpa.cpp:63-66 (query) / tpa.cpp:8-17 (query_na's TpaParams::validate)
        if (!na && fingerprint != g0->fingerprint)
            throw std::runtime_error("stale artifact: graph fingerprint mismatch");
        if (!na && (S < 1 || S >= T)) throw std::invalid_argument("family_end (S) must satisfy 1 <= S < T");
        if (na && S < 1) throw std::invalid_argument("family_end (S) must be at least 1");
        if (na && T <= S) throw std::invalid_argument("stranger_start (T) must exceed family_end (S)");
        validate_cpi(c, eps, 0, (int64_t)S - 1);
        if (!na && !stranger) throw std::invalid_argument("null stranger vector");
        if (flags & TPA_NODE_MAJOR) throw std::invalid_argument("a partitioned batch writes seed-major output");
        if (B == 0) return;
        if (!seeds || !out) throw std::invalid_argument("null seeds or output");
        const double scale = 1.0 + tpa_neighbor_scale_factor(c, S, T);
        run_batch_part(grp->parts, grp->gdeg, seeds, B, c, eps, S, na ? nullptr : stranger, scale, out,
                       (flags & TPA_DEVICE_PTRS) != 0);
    });
}

int tpa_group_preprocess(tpa_group* grp, double c, double eps, uint32_t T, double* out_stranger) {
    return guard([&] {
        if (!grp) throw std::invalid_argument("null group");
        std::lock_guard<std::mutex> lk(grp->mu);
        part_preprocess(grp->parts, c, eps, T, out_stranger);
    });
}

}  // extern "C"
