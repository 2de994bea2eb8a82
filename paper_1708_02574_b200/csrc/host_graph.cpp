// host_graph.cpp -- host-side graph plumbing for libtpa_gpu.so.
//
// Not on the hot path.  This is the input side of the boundary: the
// rwrank::Graph construction semantics (graph.cpp:53-91), the two synthetic
// generators the benchmark configs name, the CLI's seed sampler
// (rwrank_main.cpp:65-83) and the artifact fingerprint (graph.cpp:17-33,
// 84-90), written B200-host-first: bucket-by-source construction with
// per-node sorts across all host threads instead of one global std::sort.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "tpa_gpu.h"
#include "tpa_internal.hpp"

struct tpa_host_graph {
    uint32_t n = 0;
    int policy = TPA_SELFLOOP;
    std::vector<uint64_t> off;
    std::vector<uint32_t> tgt;
    std::vector<uint32_t> dangling;
    uint64_t fingerprint = 0;
};

namespace {

unsigned host_threads(int requested) {
    unsigned t = requested > 0 ? unsigned(requested) : std::thread::hardware_concurrency();
    return t ? t : 1;
}

template <class F>
void parallel_ranges(uint64_t total, unsigned threads, F&& f) {
    if (threads <= 1 || total < (1u << 16)) {
        f(0u, uint64_t(0), total);
        return;
    }
    std::vector<std::thread> pool;
    for (unsigned k = 0; k < threads; ++k) {
        const uint64_t lo = total * k / threads, hi = total * (k + 1) / threads;
        pool.emplace_back([&, k, lo, hi] { f(k, lo, hi); });
    }
    for (auto& t : pool) t.join();
}

// FNV-1a over little-endian bytes (graph.cpp:17-33).  Word-at-a-time but
// byte-serial, as the hash definition requires.
struct Fnv {
    uint64_t h = 0xcbf29ce484222325ULL;
    inline void bytes(uint64_t v, int nbytes) {
        for (int i = 0; i < nbytes; ++i) {
            h ^= (v >> (8 * i)) & 0xffu;
            h *= 0x100000001b3ULL;
        }
    }
};

uint64_t fingerprint_of(uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* tgt,
                        int policy) {
    Fnv f;
    f.bytes(n, 4);
    f.bytes(m, 8);
    for (uint64_t i = 0; i <= n; ++i) f.bytes(off[i], 8);
    for (uint64_t i = 0; i < m; ++i) f.bytes(tgt[i], 4);
    f.bytes(uint32_t(policy), 4);
    return f.h;
}

}  // namespace

tpa_host_graph* tpa::make_host_graph(uint32_t n, int policy, std::vector<uint64_t>&& off,
                                     std::vector<uint32_t>&& tgt, std::vector<uint32_t>&& dangling) {
    auto* g = new tpa_host_graph;
    g->n = n;
    g->policy = policy;
    g->off = std::move(off);
    g->tgt = std::move(tgt);
    g->dangling = std::move(dangling);
    g->fingerprint = fingerprint_of(n, g->tgt.size(), g->off.data(), g->tgt.data(), policy);
    return g;
}

namespace {

// graph.cpp:53-91 semantics: validate, sort + dedupe per source, dangling
// list before the policy, SelfLoop repair edge, out-CSR, fingerprint.
tpa_host_graph* build(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t m,
                      int policy, unsigned threads) {
    if (n == 0) throw std::invalid_argument("graph must have at least one node");
    if (policy < 0 || policy > 2) throw std::invalid_argument("unknown dangling policy");
    for (uint64_t i = 0; i < m; ++i)
        if (src[i] >= n || dst[i] >= n)
            throw std::out_of_range("edge endpoint out of range: " + std::to_string(src[i]) +
                                    " -> " + std::to_string(dst[i]));
    // Two-pass counting scatter by source with per-thread cursors (deterministic).
    const unsigned T = host_threads(int(threads));
    std::vector<std::vector<uint64_t>> cnt(T, std::vector<uint64_t>(size_t(n) + 1, 0));
    parallel_ranges(m, T, [&](unsigned k, uint64_t lo, uint64_t hi) {
        auto& c = cnt[k];
        for (uint64_t i = lo; i < hi; ++i) ++c[src[i]];
    });
    const bool serial = !(T > 1 && m >= (1u << 16));
    const unsigned used = serial ? 1 : T;
    std::vector<uint64_t> boff(size_t(n) + 1, 0);
    for (uint32_t u = 0; u < n; ++u) {
        uint64_t s = 0;
        for (unsigned k = 0; k < used; ++k) s += cnt[k][u];
        boff[u + 1] = boff[u] + s;
    }
    // per-thread write cursors: thread k writes after threads < k within bucket u
    std::vector<uint32_t> bucket(m);
    parallel_ranges(n, used, [&](unsigned, uint64_t lo, uint64_t hi) {
        for (uint64_t u = lo; u < hi; ++u) {
            uint64_t pos = boff[u];
            for (unsigned k = 0; k < used; ++k) {
                const uint64_t c = cnt[k][u];
                cnt[k][u] = pos;
                pos += c;
            }
        }
    });
    parallel_ranges(m, used, [&](unsigned k, uint64_t lo, uint64_t hi) {
        auto& c = cnt[k];
        for (uint64_t i = lo; i < hi; ++i) bucket[c[src[i]]++] = dst[i];
    });
    cnt.clear();
    cnt.shrink_to_fit();
    // sort + unique each bucket in place; new degree per node
    std::vector<uint64_t> deg(n, 0);
    parallel_ranges(n, T, [&](unsigned, uint64_t lo, uint64_t hi) {
        for (uint64_t u = lo; u < hi; ++u) {
            uint32_t* b = bucket.data() + boff[u];
            uint32_t* e = bucket.data() + boff[u + 1];
            std::sort(b, e);
            deg[u] = uint64_t(std::unique(b, e) - b);
        }
    });
    auto* g = new tpa_host_graph;
    g->n = n;
    g->policy = policy;
    for (uint32_t u = 0; u < n; ++u)
        if (deg[u] == 0) g->dangling.push_back(u);
    const bool repair = policy == TPA_SELFLOOP;
    g->off.assign(size_t(n) + 1, 0);
    for (uint32_t u = 0; u < n; ++u) g->off[u + 1] = g->off[u] + (deg[u] ? deg[u] : (repair ? 1 : 0));
    g->tgt.resize(g->off[n]);
    parallel_ranges(n, T, [&](unsigned, uint64_t lo, uint64_t hi) {
        for (uint64_t u = lo; u < hi; ++u) {
            if (deg[u])
                std::memcpy(g->tgt.data() + g->off[u], bucket.data() + boff[u], deg[u] * 4);
            else if (repair)
                g->tgt[g->off[u]] = uint32_t(u);
        }
    });
    g->fingerprint = fingerprint_of(n, g->tgt.size(), g->off.data(), g->tgt.data(), policy);
    return g;
}

// generate_random_graph (graph.cpp:166-205) semantics.  The sparse branch
// accepts the first `m` distinct draws in draw order; it is evaluated in
// batches (draw, then keep first occurrences) instead of an unordered_set,
// which yields the identical edge set for the same mt19937_64 stream.
void random_edges(uint32_t node_count, uint64_t m, uint64_t seed, std::vector<uint32_t>& su,
                  std::vector<uint32_t>& sv) {
    if (node_count == 0) throw std::invalid_argument("graph must have at least one node");
    const uint64_t n = node_count;
    const uint64_t max_edges = n * (n - 1);
    if (m > max_edges)
        throw std::invalid_argument("edge_count " + std::to_string(m) + " exceeds n*(n-1) = " +
                                    std::to_string(max_edges));
    std::mt19937_64 rng(seed);
    su.clear();
    sv.clear();
    su.reserve(m);
    sv.reserve(m);
    if (m > max_edges / 4) {
        std::vector<uint64_t> pairs;
        pairs.reserve(max_edges);
        for (uint64_t u = 0; u < n; ++u)
            for (uint64_t v = 0; v < n; ++v)
                if (u != v) pairs.push_back(u * n + v);
        for (uint64_t i = 0; i < m; ++i) {
            std::uniform_int_distribution<uint64_t> pick(i, pairs.size() - 1);
            std::swap(pairs[i], pairs[pick(rng)]);
            su.push_back(uint32_t(pairs[i] / n));
            sv.push_back(uint32_t(pairs[i] % n));
        }
        return;
    }
    std::uniform_int_distribution<uint64_t> pick_u(0, n - 1);
    std::uniform_int_distribution<uint64_t> pick_v(0, n - 2);
    std::vector<uint64_t> accepted;  // keys in acceptance order
    accepted.reserve(m);
    std::vector<uint64_t> sorted_acc;  // sorted copy for membership
    while (accepted.size() < m) {
        const uint64_t want = m - accepted.size();
        std::vector<std::pair<uint64_t, uint64_t>> draws(want);  // (key, draw order)
        for (uint64_t i = 0; i < want; ++i) {
            const uint64_t u = pick_u(rng);
            uint64_t v = pick_v(rng);
            if (v >= u) ++v;
            draws[i] = {u * n + v, i};
        }
        std::vector<std::pair<uint64_t, uint64_t>> byk(draws);
        std::sort(byk.begin(), byk.end());
        std::vector<char> keep(want, 0);
        for (uint64_t i = 0; i < want; ++i) {
            const bool first = i == 0 || byk[i].first != byk[i - 1].first;
            if (first && !std::binary_search(sorted_acc.begin(), sorted_acc.end(), byk[i].first))
                keep[byk[i].second] = 1;
        }
        for (uint64_t i = 0; i < want; ++i)
            if (keep[i]) accepted.push_back(draws[i].first);
        sorted_acc = accepted;
        std::sort(sorted_acc.begin(), sorted_acc.end());
    }
    for (uint64_t k : accepted) {
        su.push_back(uint32_t(k / n));
        sv.push_back(uint32_t(k % n));
    }
}

// R-MAT quadrant recursion.  Edge i is generated from its own mt19937_64
// stream seeded by (seed, i / kChunk) so the edge list is independent of the
// thread count.  MSB first; quadrant (0,0) p=a, (0,1) b, (1,0) c, (1,1) rest.
void rmat_edges(uint32_t scale, uint64_t m, double a, double b, double c, uint64_t seed,
                unsigned threads, std::vector<uint32_t>& su, std::vector<uint32_t>& sv,
                uint64_t& kept) {
    if (scale == 0 || scale > 31) throw std::invalid_argument("rmat scale must be in [1, 31]");
    if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0))
        throw std::invalid_argument("rmat probabilities must be non-negative and sum <= 1");
    constexpr uint64_t kChunk = 1u << 20;
    const uint64_t nchunks = (m + kChunk - 1) / kChunk;
    std::vector<uint32_t> u(m), v(m);
    std::vector<uint8_t> loop(m);
    const double ab = a + b, abc = a + b + c;
    parallel_ranges(nchunks, threads, [&](unsigned, uint64_t lo, uint64_t hi) {
        for (uint64_t ch = lo; ch < hi; ++ch) {
            std::mt19937_64 rng(seed * 0x9E3779B97F4A7C15ULL + ch * 0xD1B54A32D192ED03ULL + 1);
            const uint64_t e0 = ch * kChunk, e1 = std::min(m, e0 + kChunk);
            for (uint64_t e = e0; e < e1; ++e) {
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
                loop[e] = x == y;
            }
        }
    });
    kept = 0;
    for (uint64_t e = 0; e < m; ++e) kept += !loop[e];
    su.resize(kept);
    sv.resize(kept);
    uint64_t k = 0;
    for (uint64_t e = 0; e < m; ++e)
        if (!loop[e]) {
            su[k] = u[e];
            sv[k] = v[e];
            ++k;
        }
}

}  // namespace

extern "C" {

int tpa_host_graph_from_edges(uint32_t n, const uint32_t* src, const uint32_t* dst, uint64_t m,
                              int policy, tpa_host_graph** out) {
    return tpa::guard([&] { *out = build(n, src, dst, m, policy, 0); });
}

int tpa_host_graph_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                        uint64_t seed, int policy, int threads, tpa_host_graph** out) {
    return tpa::guard([&] {
        const uint64_t n = uint64_t(1) << scale;
        if (n > 0xffffffffULL) throw std::invalid_argument("rmat scale too large for uint32 ids");
        std::vector<uint32_t> su, sv;
        uint64_t kept = 0;
        rmat_edges(scale, n * edge_factor, a, b, c, seed, host_threads(threads), su, sv, kept);
        *out = build(uint32_t(n), su.data(), sv.data(), kept, policy, host_threads(threads));
    });
}

int tpa_host_graph_random(uint32_t n, uint64_t m, uint64_t seed, int policy,
                          tpa_host_graph** out) {
    return tpa::guard([&] {
        std::vector<uint32_t> su, sv;
        random_edges(n, m, seed, su, sv);
        *out = build(n, su.data(), sv.data(), su.size(), policy, 0);
    });
}

void tpa_host_graph_destroy(tpa_host_graph* h) { delete h; }

void tpa_host_graph_info(const tpa_host_graph* h, uint32_t* n, uint64_t* m,
                         uint64_t* n_dangling, uint64_t* fingerprint, int* policy) {
    if (n) *n = h->n;
    if (m) *m = h->tgt.size();
    if (n_dangling) *n_dangling = h->dangling.size();
    if (fingerprint) *fingerprint = h->fingerprint;
    if (policy) *policy = h->policy;
}

const uint64_t* tpa_host_graph_offsets(const tpa_host_graph* h) { return h->off.data(); }
const uint32_t* tpa_host_graph_targets(const tpa_host_graph* h) { return h->tgt.data(); }
const uint32_t* tpa_host_graph_dangling(const tpa_host_graph* h) { return h->dangling.data(); }

int tpa_sample_seeds(const tpa_host_graph* h, uint64_t count, uint64_t rng_seed, uint32_t* out) {
    return tpa::guard([&] {
        std::vector<char> dang(h->n, 0);
        for (uint32_t u : h->dangling) dang[u] = 1;
        std::vector<uint32_t> pool;
        pool.reserve(h->n);
        for (uint32_t u = 0; u < h->n; ++u)
            if (!dang[u]) pool.push_back(u);
        if (pool.size() < count)
            throw std::runtime_error("graph has only " + std::to_string(pool.size()) +
                                     " non-dangling nodes; cannot draw " + std::to_string(count) +
                                     " seeds");
        std::mt19937_64 rng(rng_seed);
        for (size_t i = 0; i < count; ++i) {
            std::uniform_int_distribution<size_t> pick(i, pool.size() - 1);
            std::swap(pool[i], pool[pick(rng)]);
        }
        std::memcpy(out, pool.data(), count * 4);
    });
}

uint64_t tpa_fingerprint(uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* tgt,
                         int policy) {
    return fingerprint_of(n, m, off, tgt, policy);
}

}  // extern "C"
