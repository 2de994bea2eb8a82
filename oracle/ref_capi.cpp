// ref_capi.cpp -- extern "C" wrapper over the UNMODIFIED reference library
// (compiled by oracle/Makefile straight from /root/reference/proj/src into
// oracle/_ref/librwrank_ref.so).  TEST / BASELINE INFRASTRUCTURE ONLY: used by
// tests/ to pin the oracle and the GPU path, by oracle/make_golden.py to emit
// golden fixtures, and by bench.py's reference arm to time the reference CPU
// path on the box's host cores.  Never linked into the product.
//
// Every entry point calls the reference's own public API
// (proj/include/rwrank/{graph,cpi,tpa}.hpp) and converts C++ exceptions into
// status codes with the message kept per thread:
//   0 ok, 1 std::invalid_argument, 2 std::out_of_range, 3 std::runtime_error,
//   5 anything else.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "rwrank/cpi.hpp"
#include "rwrank/graph.hpp"
#include "rwrank/tpa.hpp"

using rwrank::DanglingPolicy;
using rwrank::Graph;
using rwrank::NodeId;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 5;
    }
}

DanglingPolicy pol(int p) { return static_cast<DanglingPolicy>(p); }

rwrank::StrangerArtifact make_artifact(const Graph& g, const double* stranger, uint64_t fp,
                                       double c, double eps, uint32_t T) {
    rwrank::StrangerArtifact a;
    a.stranger_scores.assign(stranger, stranger + g.node_count());
    a.graph_fingerprint = fp;
    a.restart_prob = c;
    a.tolerance = eps;
    a.stranger_start = T;
    return a;
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_graph_from_edges(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t m,
                         int policy, void** out) {
    return guard([&] {
        std::vector<std::pair<NodeId, NodeId>> edges(m);
        for (uint64_t i = 0; i < m; ++i) edges[i] = {src[i], dst[i]};
        *out = new Graph(n, std::move(edges), pol(policy));
    });
}

int ref_graph_random(uint32_t n, uint64_t m, uint64_t seed, int policy, void** out) {
    return guard([&] { *out = new Graph(rwrank::generate_random_graph(n, m, seed, pol(policy))); });
}

// The benchmark's R-MAT generator (BASELINE.json configs C1/C2/C4/C5), restated
// here so the reference arm and the fixture scripts build their graph without
// the product library: edge e is drawn from the mt19937_64 stream of its
// 2^20-edge chunk, seeded (seed * 0x9E3779B97F4A7C15 + chunk * 0xD1B54A32D192ED03 + 1);
// per level one 53-bit uniform picks quadrant (0,0) a, (0,1) b, (1,0) c, (1,1)
// rest, MSB first; self-loops are dropped.  The edges are pre-sorted and
// de-duplicated per source on all host threads, then handed to the
// reference's own Graph constructor (graph.cpp:53-91), which sorts, dedupes,
// repairs and fingerprints them itself -- the pre-sort only spares its
// single-threaded std::sort the random input.
int ref_graph_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                   uint64_t seed, int policy, int threads, void** out) {
    return guard([&] {
        if (scale == 0 || scale > 31) throw std::invalid_argument("rmat scale must be in [1, 31]");
        const uint64_t n = uint64_t(1) << scale, m = n * edge_factor;
        constexpr uint64_t kChunk = 1u << 20;
        const uint64_t nchunks = (m + kChunk - 1) / kChunk;
        const unsigned T = threads > 0 ? unsigned(threads) : std::max(1u, std::thread::hardware_concurrency());
        std::vector<uint32_t> u(m), v(m);
        const double ab = a + b, abc = a + b + c;
        {
            std::atomic<uint64_t> next{0};
            std::vector<std::thread> pool;
            for (unsigned k = 0; k < T; ++k)
                pool.emplace_back([&] {
                    for (uint64_t ch = next++; ch < nchunks; ch = next++) {
                        std::mt19937_64 rng(seed * 0x9E3779B97F4A7C15ULL + ch * 0xD1B54A32D192ED03ULL + 1);
                        const uint64_t e1 = std::min(m, (ch + 1) * kChunk);
                        for (uint64_t e = ch * kChunk; e < e1; ++e) {
                            uint32_t x = 0, y = 0;
                            for (uint32_t lvl = 0; lvl < scale; ++lvl) {
                                const double r = double(rng() >> 11) * 0x1.0p-53;
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
                            u[e] = x;
                            v[e] = y;
                        }
                    }
                });
            for (auto& t : pool) t.join();
        }
        // counting sort by source (serial counts, parallel per-source sorts)
        std::vector<uint64_t> off(n + 1, 0);
        for (uint64_t e = 0; e < m; ++e)
            if (u[e] != v[e]) ++off[u[e] + 1];
        for (uint64_t i = 0; i < n; ++i) off[i + 1] += off[i];
        std::vector<uint32_t> bucket(off[n]);
        {
            std::vector<uint64_t> cur(off.begin(), off.end() - 1);
            for (uint64_t e = 0; e < m; ++e)
                if (u[e] != v[e]) bucket[cur[u[e]]++] = v[e];
        }
        u.clear();
        u.shrink_to_fit();
        v.clear();
        v.shrink_to_fit();
        std::vector<uint64_t> deg(n, 0);
        {
            std::vector<std::thread> pool;
            for (unsigned k = 0; k < T; ++k)
                pool.emplace_back([&, k] {
                    for (uint64_t x = n * k / T; x < n * (k + 1) / T; ++x) {
                        uint32_t* lo = bucket.data() + off[x];
                        uint32_t* hi = bucket.data() + off[x + 1];
                        std::sort(lo, hi);
                        deg[x] = uint64_t(std::unique(lo, hi) - lo);
                    }
                });
            for (auto& t : pool) t.join();
        }
        uint64_t kept = 0;
        for (uint64_t x = 0; x < n; ++x) kept += deg[x];
        std::vector<std::pair<NodeId, NodeId>> edges;
        edges.reserve(kept + n / 2);  // room for the SelfLoop repair edges
        for (uint64_t x = 0; x < n; ++x)
            for (uint64_t i = 0; i < deg[x]; ++i) edges.emplace_back(NodeId(x), bucket[off[x] + i]);
        std::vector<uint32_t>().swap(bucket);
        *out = new Graph(NodeId(n), std::move(edges), pol(policy));
    });
}

// sample_seeds (tools/rwrank_main.cpp:65-83, the CLI's seed sampler; not part
// of the library): uniform without replacement over non-dangling nodes.
int ref_sample_seeds(void* gp, uint64_t count, uint64_t rng_seed, uint32_t* out) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        std::vector<bool> dangling(g.node_count(), false);
        for (NodeId x : g.dangling_nodes()) dangling[x] = true;
        std::vector<NodeId> pool;
        pool.reserve(g.node_count());
        for (NodeId x = 0; x < g.node_count(); ++x)
            if (!dangling[x]) pool.push_back(x);
        if (pool.size() < count)
            throw std::runtime_error("graph has only " + std::to_string(pool.size()) +
                                     " non-dangling nodes; cannot draw " + std::to_string(count) +
                                     " seeds");
        std::mt19937_64 rng(rng_seed);
        for (std::size_t i = 0; i < count; ++i) {
            std::uniform_int_distribution<std::size_t> pick(i, pool.size() - 1);
            std::swap(pool[i], pool[pick(rng)]);
        }
        std::memcpy(out, pool.data(), count * 4);
    });
}

// max in-degree node of the graph and its in-degree (test helper)
void ref_graph_max_indeg(void* gp, uint32_t* node, uint64_t* indeg) {
    const Graph& g = *static_cast<Graph*>(gp);
    std::vector<uint64_t> d(g.node_count(), 0);
    for (NodeId t : g.out_targets()) ++d[t];
    const auto it = std::max_element(d.begin(), d.end());
    *node = NodeId(it - d.begin());
    *indeg = *it;
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }
uint32_t ref_graph_n(void* g) { return static_cast<Graph*>(g)->node_count(); }
uint64_t ref_graph_m(void* g) { return static_cast<Graph*>(g)->edge_count(); }
uint64_t ref_graph_fingerprint(void* g) { return static_cast<Graph*>(g)->fingerprint(); }
uint64_t ref_graph_n_dangling(void* g) { return static_cast<Graph*>(g)->dangling_nodes().size(); }

void ref_graph_csr(void* gp, uint64_t* off, uint32_t* tgt, uint32_t* dangling) {
    const Graph& g = *static_cast<Graph*>(gp);
    if (off) std::memcpy(off, g.out_offsets().data(), g.out_offsets().size() * 8);
    if (tgt) std::memcpy(tgt, g.out_targets().data(), g.out_targets().size() * 4);
    if (dangling)
        std::memcpy(dangling, g.dangling_nodes().data(), g.dangling_nodes().size() * 4);
}

int ref_sweep(void* gp, const double* x, double* y, double c, int threads) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        rwrank::propagation_sweep(g, std::span<const double>(x, g.node_count()),
                                  std::span<double>(y, g.node_count()), c, threads);
    });
}

// seeds == nullptr -> pagerank() (all nodes).  terminal < 0 -> nullopt.
int ref_cpi_run(void* gp, const uint32_t* seeds, uint64_t n_seeds, double c, double eps,
                uint32_t start, int64_t terminal, int threads, double* out, uint32_t* iters,
                int* converged, double* residual) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        rwrank::CpiParams p;
        p.restart_prob = c;
        p.tolerance = eps;
        p.start_iter = start;
        if (terminal >= 0) p.terminal_iter = static_cast<uint32_t>(terminal);
        p.threads = threads;
        rwrank::CpiResult r =
            seeds ? rwrank::cpi_run(g, rwrank::SeedSet(std::vector<NodeId>(seeds, seeds + n_seeds)), p)
                  : rwrank::pagerank(g, p);
        std::memcpy(out, r.scores.data(), r.scores.size() * 8);
        *iters = r.iterations_run;
        *converged = r.converged ? 1 : 0;
        *residual = r.residual_l1;
    });
}

int ref_exact_rwr(void* gp, uint32_t seed, double c, double eps, int threads, double* out) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        rwrank::ScoreVector r = rwrank::exact_rwr(g, seed, c, eps, threads);
        std::memcpy(out, r.data(), r.size() * 8);
    });
}

int ref_cpi_partition(void* gp, const uint32_t* seeds, uint64_t n_seeds, double c, double eps,
                      const uint32_t* bounds, uint64_t nb, int threads, double* out) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        auto parts = rwrank::cpi_partition(
            g, rwrank::SeedSet(std::vector<NodeId>(seeds, seeds + n_seeds)), c, eps,
            std::span<const uint32_t>(bounds, nb), threads);
        for (size_t k = 0; k < parts.size(); ++k)
            std::memcpy(out + k * g.node_count(), parts[k].data(), g.node_count() * 8);
    });
}

double ref_neighbor_scale_factor(double c, uint32_t S, uint32_t T) {
    return rwrank::neighbor_scale_factor(c, S, T);
}

int ref_preprocess(void* gp, double c, double eps, uint32_t T, int threads, double* out,
                   uint64_t* fp_out) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        rwrank::StrangerArtifact a = rwrank::preprocess(g, c, eps, T, threads);
        std::memcpy(out, a.stranger_scores.data(), a.stranger_scores.size() * 8);
        if (fp_out) *fp_out = a.graph_fingerprint;
    });
}

int ref_query(void* gp, const double* stranger, uint64_t fp, double c, double eps, uint32_t T,
              uint32_t seed, uint32_t S, int threads, double* out) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        auto a = make_artifact(g, stranger, fp, c, eps, T);
        rwrank::ScoreVector r = rwrank::query(g, a, seed, S, threads);
        std::memcpy(out, r.data(), r.size() * 8);
    });
}

int ref_query_na(void* gp, uint32_t seed, uint32_t S, uint32_t T, double c, double eps,
                 int threads, double* out) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        rwrank::TpaParams p;
        p.family_end = S;
        p.stranger_start = T;
        p.restart_prob = c;
        p.tolerance = eps;
        rwrank::ScoreVector r = rwrank::query_na(g, seed, p, threads);
        std::memcpy(out, r.data(), r.size() * 8);
    });
}

// Runs `count` independent reference query() calls spread over `workers`
// std::threads sharing one graph + artifact (the reference's own concurrency
// contract, SPEC.md:239 / tpa_test.cpp:148-161).  out (count x n) may be null.
// Returns the wall time in seconds through *seconds.
int ref_query_many(void* gp, const double* stranger, uint64_t fp, double c, double eps,
                   uint32_t T, const uint32_t* seeds, uint32_t count, uint32_t S, int workers,
                   double* out, double* seconds) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        auto a = make_artifact(g, stranger, fp, c, eps, T);
        std::atomic<uint32_t> next{0};
        std::atomic<int> failed{0};
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        const int w = workers < 1 ? 1 : workers;
        for (int k = 0; k < w; ++k)
            pool.emplace_back([&] {
                for (uint32_t i = next++; i < count; i = next++) {
                    try {
                        rwrank::ScoreVector r = rwrank::query(g, a, seeds[i], S, 1);
                        if (out) std::memcpy(out + size_t(i) * g.node_count(), r.data(), r.size() * 8);
                    } catch (...) {
                        failed = 1;
                    }
                }
            });
        for (auto& t : pool) t.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (failed) throw std::runtime_error("a reference query failed");
    });
}

// Times one reference preprocess() call (the CLI's timed region,
// rwrank_main.cpp:122-124) or, with max_sweeps > 0, that many dense
// propagation_sweep calls (for extrapolating configs too large to run whole).
int ref_time_preprocess(void* gp, double c, double eps, uint32_t T, int threads, double* out,
                        double* seconds) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        auto t0 = std::chrono::steady_clock::now();
        rwrank::StrangerArtifact a = rwrank::preprocess(g, c, eps, T, threads);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (out) std::memcpy(out, a.stranger_scores.data(), a.stranger_scores.size() * 8);
    });
}

int ref_time_sweeps(void* gp, uint32_t sweeps, double c, int threads, double* seconds) {
    return guard([&] {
        const Graph& g = *static_cast<Graph*>(gp);
        std::vector<double> x(g.node_count(), 1.0 / g.node_count()), y(g.node_count());
        auto t0 = std::chrono::steady_clock::now();
        for (uint32_t s = 0; s < sweeps; ++s) {
            rwrank::propagation_sweep(g, std::span<const double>(x), std::span<double>(y), c,
                                      threads);
            x.swap(y);
        }
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

}  // extern "C"
