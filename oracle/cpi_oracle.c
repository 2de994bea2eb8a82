/*
 * cpi_oracle.c -- CPU restatement of the reference's Cumulative Power
 * Iteration path.  TEST INFRASTRUCTURE ONLY: the parity checker for the
 * sm_100a kernels.  Nothing in the product (paper_1708_02574_b200/) links,
 * loads or calls this file; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may.
 *
 * Parity pinned: tests/test_oracle.py checks every function here against the
 * reference itself (oracle/_ref/librwrank_ref.so, compiled from
 * /root/reference/proj/src by oracle/Makefile) and against the committed
 * golden vectors in tests/golden/ (made by oracle/make_golden.py from the
 * reference build).  The arithmetic is written in exactly the reference's
 * operation order, so agreement is expected to be bitwise.
 *
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction; the reference is
 * compiled for baseline x86-64 where none happens either).
 *
 * Graph input is the reference's out-edge CSR (graph.hpp:61-62):
 *   off[n+1] (uint64), tgt[m] (uint32), sorted + deduped, SelfLoop repair
 *   edges already present.  policy: 0 SelfLoop, 1 Uniform, 2 Drop
 *   (graph.hpp:19, declaration order).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "cpi_oracle.h"

/* graph.cpp:211-226 (sweep_range) + graph.cpp:230-270 (propagation_sweep,
 * threads == 1 branch).  Push over out-edges in ascending source order,
 * zero-skip at :216, dangling mass at :218-221, Uniform spread at :265-268. */
void oracle_sweep(uint32_t n, const uint64_t *off, const uint32_t *tgt, int policy,
                  const double *x, double *y, double c) {
    const double keep = 1.0 - c;
    double dangling_mass = 0.0;
    for (uint32_t v = 0; v < n; ++v) y[v] = 0.0;
    for (uint32_t u = 0; u < n; ++u) {
        const double xu = x[u];
        if (xu == 0.0) continue;
        const uint32_t deg = (uint32_t)(off[u + 1] - off[u]);
        if (deg == 0) {
            dangling_mass += xu;
            continue;
        }
        const double share = keep * xu / (double)deg;
        for (uint64_t e = off[u]; e < off[u + 1]; ++e) y[tgt[e]] += share;
    }
    if (dangling_mass != 0.0 && policy == ORACLE_UNIFORM) {
        const double spread = keep * dangling_mass / (double)n;
        for (uint32_t v = 0; v < n; ++v) y[v] += spread;
    }
}

/* cpi.cpp:43-47 */
static double l1_sum(const double *v, uint32_t n) {
    double s = 0.0;
    for (uint32_t i = 0; i < n; ++i) s += fabs(v[i]);
    return s;
}

/* cpi.cpp:49-51 */
static void add_into(double *acc, const double *x, uint32_t n) {
    for (uint32_t i = 0; i < n; ++i) acc[i] += x[i];
}

/* upper_bound over the partition boundaries (cpi.cpp:128-129). */
static size_t segment_of(const uint32_t *bounds, size_t nb, uint32_t i) {
    size_t lo = 0, hi = nb;
    while (lo < hi) {
        size_t mid = (lo + hi) / 2;
        if (bounds[mid] <= i) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

/*
 * cpi.cpp:55-83 run_series, with the two sinks the reference uses:
 *  - bounds == NULL: cpi_run's windowed sink (cpi.cpp:92-98):
 *      accumulate iff i >= start && (terminal < 0 || i <= terminal);
 *      continue iff terminal < 0 || i < terminal.
 *  - bounds != NULL: cpi_partition's sink (cpi.cpp:127-132): x^(i) goes to
 *      segment upper_bound(bounds, i); always continue.  out holds
 *      (nb + 1) * n doubles, segment-major.
 * seeds == NULL means all nodes (SeedSet::all_nodes, cpi.cpp:28-32); else the
 * caller passes a sorted duplicate-free list (cpi.cpp:19-24).
 * Returns 0; inputs are assumed validated (validation is host API behaviour,
 * pinned separately in the tests).
 */
int oracle_run_series(uint32_t n, const uint64_t *off, const uint32_t *tgt, int policy,
                      const uint32_t *seeds, uint64_t n_seeds, double c, double eps,
                      uint32_t start, int64_t terminal, const uint32_t *bounds, size_t nb,
                      double *out, uint32_t *iterations_run, int *converged,
                      double *residual_l1) {
    double *x = (double *)calloc(n ? n : 1, sizeof(double));
    double *next = (double *)malloc((n ? n : 1) * sizeof(double));
    const int partition = bounds != NULL;
    const size_t n_out = partition ? (nb + 1) * (size_t)n : (size_t)n;
    uint32_t it = 0;
    int conv = 0;
    double res;

    for (size_t i = 0; i < n_out; ++i) out[i] = 0.0;

    if (seeds == NULL) {
        const double weight = c / (double)n;
        for (uint32_t u = 0; u < n; ++u) x[u] = weight;
    } else {
        const double weight = c / (double)n_seeds;
        for (uint64_t k = 0; k < n_seeds; ++k) x[seeds[k]] = weight;
    }

    res = l1_sum(x, n);
    /* sink(0) */
    {
        int keep_going;
        if (partition) {
            add_into(out + segment_of(bounds, nb, 0) * (size_t)n, x, n);
            keep_going = 1;
        } else {
            if (0 >= start && (terminal < 0 || 0 <= terminal)) add_into(out, x, n);
            keep_going = terminal < 0 || 0 < terminal;
        }
        if (!keep_going) goto done;
    }
    for (uint32_t i = 1;; ++i) {
        double *tmp;
        int keep_going;
        oracle_sweep(n, off, tgt, policy, x, next, c);
        tmp = x; x = next; next = tmp;
        it = i;
        res = l1_sum(x, n);
        if (partition) {
            add_into(out + segment_of(bounds, nb, i) * (size_t)n, x, n);
            keep_going = 1;
        } else {
            if (i >= start && (terminal < 0 || (int64_t)i <= terminal)) add_into(out, x, n);
            keep_going = terminal < 0 || (int64_t)i < terminal;
        }
        if (res < eps) {
            conv = 1;
            break;
        }
        if (!keep_going) break;
    }
done:
    if (iterations_run) *iterations_run = it;
    if (converged) *converged = conv;
    if (residual_l1) *residual_l1 = res;
    free(x);
    free(next);
    return 0;
}

/* tpa.cpp:39-44 */
double oracle_neighbor_scale_factor(double c, uint32_t S, uint32_t T) {
    const double keep = 1.0 - c;
    const double family_mass = 1.0 - pow(keep, (double)S);
    const double neighbor_mass = pow(keep, (double)S) - pow(keep, (double)T);
    return neighbor_mass / family_mass;
}

/* tpa.cpp:19-37: PageRank window [T, inf). */
int oracle_preprocess(uint32_t n, const uint64_t *off, const uint32_t *tgt, int policy,
                      double c, double eps, uint32_t T, double *stranger) {
    return oracle_run_series(n, off, tgt, policy, NULL, 0, c, eps, T, -1, NULL, 0, stranger,
                             NULL, NULL, NULL);
}

/* tpa.cpp:48-57 family_part + tpa.cpp:61-76 query (na == 0) or
 * tpa.cpp:78-86 query_na (na != 0, stranger ignored). */
int oracle_query(uint32_t n, const uint64_t *off, const uint32_t *tgt, int policy,
                 const double *stranger, double c, double eps, uint32_t T, uint32_t seed,
                 uint32_t S, int na, double *out) {
    const double scale = 1.0 + oracle_neighbor_scale_factor(c, S, T);
    oracle_run_series(n, off, tgt, policy, &seed, 1, c, eps, 0, (int64_t)S - 1, NULL, 0, out,
                      NULL, NULL, NULL);
    if (na) {
        for (uint32_t v = 0; v < n; ++v) out[v] *= scale;
    } else {
        for (uint32_t v = 0; v < n; ++v) out[v] = scale * out[v] + stranger[v];
    }
    return 0;
}
