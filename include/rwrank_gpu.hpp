// rwrank_gpu.hpp -- header-only C++ adapter over the C-ABI (tpa_gpu.h) with
// the reference's C++ calling conventions: exceptions of the reference's
// types, std::vector score vectors, std::optional terminal iteration.
//
// Mirrors proj/include/rwrank/{graph,cpi,tpa}.hpp.  Works with any graph
// type that exposes the reference Graph's accessors (node_count(),
// edge_count(), out_offsets(), out_targets(), dangling_policy(),
// fingerprint()) -- in particular rwrank::Graph itself -- so a caller keeps
// building its graphs with the reference code and hands them to the GPU.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "tpa_gpu.h"

namespace rwrank_gpu {

// Status -> the reference's exception type (tpa_gpu.h status table).
inline void check(int rc) {
    if (rc == TPA_OK) return;
    const std::string msg = tpa_last_error();
    switch (rc) {
        case TPA_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case TPA_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        case TPA_ERR_RUNTIME: throw std::runtime_error(msg);
        case TPA_ERR_ALLOC: throw std::bad_alloc();
        default: throw std::runtime_error("CUDA: " + msg);
    }
}

// Device-resident CSR(A^T) of one graph (tpa_graph_create; graph.hpp:26-66).
class DeviceGraph {
public:
    template <class G>
    explicit DeviceGraph(const G& g, int device = 0) {
        tpa_graph* h = nullptr;
        check(tpa_graph_create(g.node_count(), g.edge_count(), g.out_offsets().data(),
                               g.edge_count() ? g.out_targets().data() : nullptr,
                               static_cast<int>(g.dangling_policy()), g.fingerprint(), device, &h));
        h_.reset(h);
        n_ = g.node_count();
        fingerprint_ = g.fingerprint();
    }
    tpa_graph* get() const { return h_.get(); }
    uint32_t node_count() const { return n_; }
    uint64_t fingerprint() const { return fingerprint_; }

private:
    struct Del {
        void operator()(tpa_graph* h) const { tpa_graph_destroy(h); }
    };
    std::unique_ptr<tpa_graph, Del> h_;
    uint32_t n_ = 0;
    uint64_t fingerprint_ = 0;
};

// graph.hpp:96-103
inline void propagation_sweep(DeviceGraph& g, std::span<const double> x, std::span<double> y, double c) {
    if (x.size() != g.node_count() || y.size() != g.node_count())
        throw std::invalid_argument("score vector length does not match node count");
    check(tpa_propagation_sweep(g.get(), x.data(), y.data(), c, 0));
}

struct CpiOut {
    std::vector<double> scores;
    uint32_t iterations_run = 0;
    bool converged = false;
    double residual_l1 = 0.0;
};

// cpi.hpp:44-49 (seeds empty -> all nodes, i.e. pagerank, cpi.hpp:56-57)
inline CpiOut cpi_run(DeviceGraph& g, std::span<const uint32_t> seeds, bool all_nodes, double c, double eps,
                      uint32_t start_iter, std::optional<uint32_t> terminal_iter) {
    CpiOut r;
    r.scores.resize(g.node_count());
    int conv = 0;
    check(tpa_cpi_run(g.get(), all_nodes ? nullptr : seeds.data(), all_nodes ? 0 : seeds.size(), c, eps,
                      start_iter, terminal_iter ? static_cast<int64_t>(*terminal_iter) : -1, r.scores.data(),
                      &r.iterations_run, &conv, &r.residual_l1, 0));
    r.converged = conv != 0;
    return r;
}

// cpi.hpp:59-62
inline std::vector<std::vector<double>> cpi_partition(DeviceGraph& g, std::span<const uint32_t> seeds, double c,
                                                      double eps, std::span<const uint32_t> boundaries) {
    const size_t n = g.node_count(), k = boundaries.size() + 1;
    std::vector<double> flat(n * k);
    check(tpa_cpi_partition(g.get(), seeds.data(), seeds.size(), c, eps, boundaries.data(), boundaries.size(),
                            flat.data(), 0));
    std::vector<std::vector<double>> out(k);
    for (size_t s = 0; s < k; ++s) out[s].assign(flat.begin() + s * n, flat.begin() + (s + 1) * n);
    return out;
}

// tpa.hpp:30-32
inline double neighbor_scale_factor(double c, uint32_t S, uint32_t T) { return tpa_neighbor_scale_factor(c, S, T); }

// Device copy of a StrangerArtifact (tpa.hpp:17-23).
class DeviceArtifact {
public:
    DeviceArtifact(DeviceGraph& g, std::span<const double> stranger, uint64_t fingerprint, double c, double eps,
                   uint32_t T) {
        tpa_artifact* a = nullptr;
        check(tpa_artifact_create(g.get(), stranger.data(), fingerprint, c, eps, T, 0, &a));
        a_.reset(a);
    }
    explicit DeviceArtifact(tpa_artifact* a) { a_.reset(a); }
    const tpa_artifact* get() const { return a_.get(); }

private:
    struct Del {
        void operator()(tpa_artifact* a) const { tpa_artifact_destroy(a); }
    };
    std::unique_ptr<tpa_artifact, Del> a_;
};

// tpa.hpp:25-28: returns the stranger scores; `keep` receives the device copy.
inline std::vector<double> preprocess(DeviceGraph& g, double c, double eps, uint32_t T,
                                      std::unique_ptr<DeviceArtifact>* keep = nullptr) {
    std::vector<double> s(g.node_count());
    tpa_artifact* a = nullptr;
    check(tpa_preprocess(g.get(), c, eps, T, s.data(), keep ? &a : nullptr, 0));
    if (keep) *keep = std::make_unique<DeviceArtifact>(a);
    return s;
}

// tpa.hpp:34-38
inline std::vector<double> query(DeviceGraph& g, const DeviceArtifact& a, uint32_t seed, uint32_t S) {
    std::vector<double> out(g.node_count());
    check(tpa_query(g.get(), a.get(), seed, S, out.data(), 0));
    return out;
}

// Batched query: seeds.size() independent query() results, [B][n].
inline std::vector<double> query_batch(DeviceGraph& g, const DeviceArtifact& a, std::span<const uint32_t> seeds,
                                       uint32_t S) {
    std::vector<double> out((size_t)g.node_count() * seeds.size());
    check(tpa_query_batch(g.get(), a.get(), seeds.data(), (uint32_t)seeds.size(), S, out.data(), 0));
    return out;
}

// tpa.hpp:40-41 (TpaParams fields passed explicitly)
inline std::vector<double> query_na(DeviceGraph& g, uint32_t seed, uint32_t S, uint32_t T, double c, double eps) {
    std::vector<double> out(g.node_count());
    check(tpa_query_na_batch(g.get(), &seed, 1, S, T, c, eps, out.data(), 0));
    return out;
}

}  // namespace rwrank_gpu
