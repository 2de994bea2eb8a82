// rwrank_dropin.cpp -- the GPU drop-in for the reference's hot path.
//
// Defines the rwrank:: entry points declared by the reference's own headers
// proj/include/rwrank/cpi.hpp and tpa.hpp (and propagation_sweep from
// graph.hpp) on top of libtpa_gpu.so.  A maintainer links this TU *instead
// of* proj/src/cpi.cpp and proj/src/tpa.cpp (and with graph.cpp's two
// propagation_sweep symbols weakened, see integration/Makefile); everything
// else -- Graph, I/O, metrics, analysis, persistence, the CLI -- stays the
// reference's code and now runs on the B200 path.  INTEGRATION.md has the
// recipe.  The reference's `threads` arguments select host threads there and
// are accepted and ignored here.
#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "rwrank/cpi.hpp"
#include "rwrank/graph.hpp"
#include "rwrank/tpa.hpp"
#include "rwrank_gpu.hpp"

namespace {

// Device-resident CSR(A^T) per host Graph, rebuilt if the Graph at that
// address changed (its fingerprint covers n, m, offsets, targets, policy).
// At most kGraphCache graphs stay resident (least recently used evicted; a
// caller still holding the shared_ptr keeps its handle alive).
constexpr size_t kGraphCache = 4;
struct GraphSlot {
    const rwrank::Graph* key;
    std::shared_ptr<rwrank_gpu::DeviceGraph> dg;
};
std::mutex g_mu;
// Deliberately never destroyed: device handles must not be released from
// static destructors, which may run after the CUDA runtime has shut down.
auto* g_graphs = new std::vector<GraphSlot>();  // most recent last

std::shared_ptr<rwrank_gpu::DeviceGraph> device_graph(const rwrank::Graph& g) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& v = *g_graphs;
    for (size_t i = 0; i < v.size(); ++i) {
        if (v[i].key != &g) continue;
        GraphSlot s = std::move(v[i]);
        v.erase(v.begin() + i);
        if (s.dg->fingerprint() != g.fingerprint() || s.dg->node_count() != g.node_count()) break;
        v.push_back(std::move(s));
        return v.back().dg;
    }
    if (v.size() >= kGraphCache) v.erase(v.begin());
    v.push_back({&g, std::make_shared<rwrank_gpu::DeviceGraph>(g)});
    return v.back().dg;
}

// Device copies of stranger vectors, so query() does not upload n doubles per
// call (and concurrent queries on one artifact share one copy).  Keyed by the
// device graph, the vector's buffer and size and the artifact's scalars, and
// checked against 64 strided entries of the vector captured at upload: an
// in-place rewrite of the scores is caught unless it leaves every sampled
// entry bit-identical.  At most kArtifactCache entries (LRU).
constexpr size_t kArtifactCache = 8, kSample = 64;
struct ArtSlot {
    const rwrank_gpu::DeviceGraph* g;
    const double* data;
    size_t n;
    uint64_t fp;
    double c, eps;
    uint32_t T;
    std::vector<double> sample;
    std::shared_ptr<rwrank_gpu::DeviceGraph> keep_g;
    std::shared_ptr<rwrank_gpu::DeviceArtifact> a;
};
auto* g_arts = new std::vector<ArtSlot>();

std::vector<double> sample_of(const std::vector<double>& v) {
    std::vector<double> s;
    if (v.empty()) return s;
    s.reserve(kSample);
    for (size_t j = 0; j < kSample; ++j) s.push_back(v[j * (v.size() - 1) / (kSample - 1)]);
    return s;
}

bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * 8) == 0);
}

std::shared_ptr<rwrank_gpu::DeviceArtifact> device_artifact(const std::shared_ptr<rwrank_gpu::DeviceGraph>& dg,
                                                            const rwrank::StrangerArtifact& art,
                                                            std::unique_ptr<rwrank_gpu::DeviceArtifact> fresh = nullptr) {
    const auto& v = art.stranger_scores;
    std::vector<double> smp = sample_of(v);
    std::lock_guard<std::mutex> lk(g_mu);
    auto& c = *g_arts;
    for (size_t i = 0; i < c.size(); ++i) {
        ArtSlot& e = c[i];
        if (e.g == dg.get() && e.data == v.data() && e.n == v.size() && e.fp == art.graph_fingerprint &&
            e.c == art.restart_prob && e.eps == art.tolerance && e.T == art.stranger_start) {
            ArtSlot s = std::move(e);
            c.erase(c.begin() + i);
            if (!fresh && same_bits(s.sample, smp)) {
                c.push_back(std::move(s));
                return c.back().a;
            }
            break;  // stale (rewritten in place) or replaced: upload anew
        }
    }
    if (c.size() >= kArtifactCache) c.erase(c.begin());
    std::shared_ptr<rwrank_gpu::DeviceArtifact> a =
        fresh ? std::shared_ptr<rwrank_gpu::DeviceArtifact>(std::move(fresh))
              : std::make_shared<rwrank_gpu::DeviceArtifact>(*dg, v, art.graph_fingerprint, art.restart_prob,
                                                             art.tolerance, art.stranger_start);
    c.push_back({dg.get(), v.data(), v.size(), art.graph_fingerprint, art.restart_prob, art.tolerance,
                 art.stranger_start, std::move(smp), dg, a});
    return a;
}

bool is_all_nodes(const rwrank::SeedSet& s, rwrank::NodeId n) {
    // sorted + duplicate-free: all nodes iff size == n and the last id is n-1
    return s.size() == n && n > 0 && s.ids().back() == n - 1;
}

}  // namespace

namespace rwrank {

// ---- parameter types (cpi.cpp:11-39, tpa.cpp:8-17 semantics) ---------------
void CpiParams::validate() const {
    if (!(restart_prob > 0.0 && restart_prob < 1.0))
        throw std::invalid_argument("restart probability must be in (0, 1)");
    if (!(tolerance > 0.0)) throw std::invalid_argument("tolerance must be positive");
    if (terminal_iter && *terminal_iter < start_iter)
        throw std::invalid_argument("terminal iteration precedes start iteration");
}

SeedSet::SeedSet(std::vector<NodeId> ids) : ids_(std::move(ids)) {
    if (ids_.empty()) throw std::invalid_argument("seed set must not be empty");
    std::sort(ids_.begin(), ids_.end());
    if (std::adjacent_find(ids_.begin(), ids_.end()) != ids_.end())
        throw std::invalid_argument("seed set contains duplicate ids");
}

SeedSet SeedSet::single(NodeId id) { return SeedSet(std::vector<NodeId>{id}); }

SeedSet SeedSet::all_nodes(NodeId node_count) {
    std::vector<NodeId> ids(node_count);
    std::iota(ids.begin(), ids.end(), NodeId{0});
    return SeedSet(std::move(ids));
}

void SeedSet::validate_against(NodeId node_count) const {
    if (!ids_.empty() && ids_.back() >= node_count)
        throw std::out_of_range("seed id " + std::to_string(ids_.back()) + " out of range for graph with " +
                                std::to_string(node_count) + " nodes");
}

void TpaParams::validate() const {
    if (family_end < 1) throw std::invalid_argument("family_end (S) must be at least 1");
    if (stranger_start <= family_end) throw std::invalid_argument("stranger_start (T) must exceed family_end (S)");
    CpiParams base;
    base.restart_prob = restart_prob;
    base.tolerance = tolerance;
    base.validate();
}

// ---- L0: one sweep (graph.hpp:96-103) ----------------------------------------
void propagation_sweep(const Graph& g, std::span<const double> x, std::span<double> y, double c, int) {
    if (x.size() != g.node_count() || y.size() != g.node_count())
        throw std::invalid_argument("score vector length does not match node count");
    auto dg = device_graph(g);
    rwrank_gpu::propagation_sweep(*dg, x, y, c);
}

ScoreVector propagation_sweep(const Graph& g, const ScoreVector& x, double c, int threads) {
    ScoreVector y(x.size());
    propagation_sweep(g, std::span<const double>(x), std::span<double>(y), c, threads);
    return y;
}

// ---- L1: CPI (cpi.hpp) --------------------------------------------------------
CpiResult cpi_run(const Graph& g, const SeedSet& seeds, const CpiParams& params) {
    params.validate();
    auto dg = device_graph(g);
    const bool all = is_all_nodes(seeds, g.node_count());
    rwrank_gpu::CpiOut o = rwrank_gpu::cpi_run(*dg, seeds.ids(), all, params.restart_prob, params.tolerance,
                                               params.start_iter, params.terminal_iter);
    CpiResult r;
    r.scores = std::move(o.scores);
    r.iterations_run = o.iterations_run;
    r.converged = o.converged;
    r.residual_l1 = o.residual_l1;
    return r;
}

ScoreVector exact_rwr(const Graph& g, NodeId seed, double c, double eps, int threads) {
    CpiParams p;
    p.restart_prob = c;
    p.tolerance = eps;
    p.threads = threads;
    return cpi_run(g, SeedSet::single(seed), p).scores;
}

CpiResult pagerank(const Graph& g, const CpiParams& params) {
    return cpi_run(g, SeedSet::all_nodes(g.node_count()), params);
}

std::vector<ScoreVector> cpi_partition(const Graph& g, const SeedSet& seeds, double c, double eps,
                                       std::span<const std::uint32_t> boundaries, int) {
    auto dg = device_graph(g);
    return rwrank_gpu::cpi_partition(*dg, seeds.ids(), c, eps, boundaries);
}

// ---- L2: TPA (tpa.hpp) ---------------------------------------------------------
StrangerArtifact preprocess(const Graph& g, double c, double eps, std::uint32_t stranger_start, int) {
    auto dg = device_graph(g);
    StrangerArtifact a;
    std::unique_ptr<rwrank_gpu::DeviceArtifact> keep;
    a.stranger_scores = rwrank_gpu::preprocess(*dg, c, eps, stranger_start, &keep);
    a.graph_fingerprint = g.fingerprint();
    a.restart_prob = c;
    a.tolerance = eps;
    a.stranger_start = stranger_start;
    // the vector's buffer survives the moves into the caller's artifact: its
    // queries find this device copy instead of uploading the scores again
    device_artifact(dg, a, std::move(keep));
    return a;
}

double neighbor_scale_factor(double c, std::uint32_t family_end, std::uint32_t stranger_start) {
    return rwrank_gpu::neighbor_scale_factor(c, family_end, stranger_start);
}

ScoreVector query(const Graph& g, const StrangerArtifact& artifact, NodeId seed, std::uint32_t family_end, int) {
    // tpa.cpp:63-66 order: staleness, then the window, before touching the data
    if (artifact.graph_fingerprint != g.fingerprint())
        throw std::runtime_error("stale artifact: graph fingerprint mismatch");
    if (family_end < 1 || family_end >= artifact.stranger_start)
        throw std::invalid_argument("family_end (S) must satisfy 1 <= S < T");
    auto dg = device_graph(g);
    auto da = device_artifact(dg, artifact);
    return rwrank_gpu::query(*dg, *da, seed, family_end);
}

ScoreVector query_na(const Graph& g, NodeId seed, const TpaParams& params, int) {
    params.validate();
    auto dg = device_graph(g);
    return rwrank_gpu::query_na(*dg, seed, params.family_end, params.stranger_start, params.restart_prob,
                                params.tolerance);
}

}  // namespace rwrank
