/* cpi_oracle.h -- CPU restatement of the reference CPI path (TEST
 * INFRASTRUCTURE ONLY; see cpi_oracle.c).  Plain C, no reference headers. */
#ifndef CPI_ORACLE_H
#define CPI_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_SELFLOOP = 0, ORACLE_UNIFORM = 1, ORACLE_DROP = 2 };

void oracle_sweep(uint32_t n, const uint64_t *off, const uint32_t *tgt, int policy,
                  const double *x, double *y, double c);

int oracle_run_series(uint32_t n, const uint64_t *off, const uint32_t *tgt, int policy,
                      const uint32_t *seeds, uint64_t n_seeds, double c, double eps,
                      uint32_t start, int64_t terminal, const uint32_t *bounds, size_t nb,
                      double *out, uint32_t *iterations_run, int *converged,
                      double *residual_l1);

double oracle_neighbor_scale_factor(double c, uint32_t S, uint32_t T);

int oracle_preprocess(uint32_t n, const uint64_t *off, const uint32_t *tgt, int policy,
                      double c, double eps, uint32_t T, double *stranger);

int oracle_query(uint32_t n, const uint64_t *off, const uint32_t *tgt, int policy,
                 const double *stranger, double c, double eps, uint32_t T, uint32_t seed,
                 uint32_t S, int na, double *out);

#ifdef __cplusplus
}
#endif
#endif
