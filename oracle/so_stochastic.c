/*
 * so_stochastic.c — oracle restatement of proj/src/stochastic.cpp:109-172
 * (estimate_innovation_covariance) and :217-277 (emulate) (TEST
 * INFRASTRUCTURE, see sphemu_oracle.h). The trend model is outside the hot
 * path: callers pass the mean table of trend.cpp:252-287 and sigma directly.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "sphemu_oracle.h"

enum { kCovBlockRows = 256, kBurnInPerOrder = 10 }; /* stochastic.cpp:16-17 */

int so_estimate_innovation_covariance(const double* resid, int64_t n_rows, int d,
                                      const so_chol_config* c, int threads, double* u_hat,
                                      double* v, double* nugget_out, so_chol_stats* st) {
  (void)threads; /* block order is fixed, so the sum is thread independent */
  if (n_rows < 2 || d < 1) return -1;
  double* u = calloc((size_t)d * d, sizeof(double));
  double* part = malloc(sizeof(double) * (size_t)d * d);
  const int64_t n_blocks = (n_rows + kCovBlockRows - 1) / kCovBlockRows;
  for (int64_t b = 0; b < n_blocks; ++b) {
    int64_t row0 = b * kCovBlockRows;
    int64_t rows = n_rows - row0 < kCovBlockRows ? n_rows - row0 : kCovBlockRows;
    memset(part, 0, sizeof(double) * (size_t)d * d);
    for (int64_t r = 0; r < rows; ++r) {
      const double* x = resid + (size_t)(row0 + r) * d;
      for (int i = 0; i < d; ++i) {
        const double xi = x[i];
        double* pr = part + (size_t)i * d;
        for (int j = 0; j < d; ++j) pr[j] += xi * x[j];
      }
    }
    for (size_t e = 0; e < (size_t)d * d; ++e) u[e] += part[e];
  }
  for (size_t e = 0; e < (size_t)d * d; ++e) u[e] /= (double)n_rows;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) u_hat[(size_t)i * d + j] = (u[(size_t)i * d + j] + u[(size_t)j * d + i]) * 0.5;
  free(part);
  free(u);

  double mean_diag = 0.0;
  for (int i = 0; i < d; ++i) mean_diag += u_hat[(size_t)i * d + i];
  mean_diag /= d;
  if (!(mean_diag > 0.0)) return -2;

  double nugget = (n_rows < d) ? 1e-8 * mean_diag : 0.0;
  const double cap = 1e-2 * mean_diag;
  double* dense = malloc(sizeof(double) * (size_t)d * d);
  int rc;
  for (;;) {
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) dense[(size_t)i * d + j] = u_hat[(size_t)i * d + j] + (i == j ? nugget : 0.0);
    int failed = -1;
    rc = so_tiled_cholesky_dense(dense, d, c, v, st, &failed);
    if (rc == 0) break;
    if (rc != 1) break;
    double next = (nugget == 0.0) ? 1e-8 * mean_diag : 10.0 * nugget;
    if (next > cap) {
      rc = 2;
      break;
    }
    nugget = next;
  }
  free(dense);
  if (nugget_out) *nugget_out = nugget;
  return rc;
}

int so_emulate(const so_plan* p, const double* v, int d, const double* phi, int order,
               const double* means, const double* sigma, const double* v2, int t_out,
               uint64_t seed, int r_len, int threads, double* out) {
  if (t_out < 1 || r_len < 1) return -1;
  const int burn = kBurnInPerOrder * order;
  const size_t points = (size_t)so_plan_points(p);
  double* root_v2 = malloc(sizeof(double) * points);
  for (size_t loc = 0; loc < points; ++loc) root_v2[loc] = sqrt(v2[loc]);
  so_rng rng;
  so_rng_seed(&rng, seed);
  double* eta = malloc(sizeof(double) * (size_t)d);
  double* f = malloc(sizeof(double) * (size_t)d);
  double* state = calloc((size_t)(order > 0 ? order : 1) * d, sizeof(double));
  double* draws = malloc(sizeof(double) * (size_t)t_out * d);
  double* synth = malloc(sizeof(double) * points * (size_t)t_out);
  for (int r = 0; r < r_len; ++r) {
    memset(state, 0, sizeof(double) * (size_t)(order > 0 ? order : 1) * d);
    for (int step = 0; step < burn + t_out; ++step) {
      for (int i = 0; i < d; ++i) eta[i] = so_rng_normal(&rng);
      /* xi = V * eta (dense GEMV, stochastic.cpp:246) */
      for (int i = 0; i < d; ++i) {
        const double* vr = v + (size_t)i * d;
        double acc = 0.0;
        for (int j = 0; j < d; ++j) acc += vr[j] * eta[j];
        f[i] = acc;
      }
      for (int q = 0; q < order; ++q)
        for (int i = 0; i < d; ++i) f[i] += phi[(size_t)q * d + i] * state[(size_t)q * d + i];
      for (int q = order - 1; q > 0; --q)
        memcpy(state + (size_t)q * d, state + (size_t)(q - 1) * d, sizeof(double) * (size_t)d);
      if (order > 0) memcpy(state, f, sizeof(double) * (size_t)d);
      if (step >= burn) memcpy(draws + (size_t)(step - burn) * d, f, sizeof(double) * (size_t)d);
    }
    double* outr = out + (size_t)r * t_out * points;
    for (int t = 0; t < t_out; ++t)
      for (size_t loc = 0; loc < points; ++loc) outr[(size_t)t * points + loc] = so_rng_normal(&rng);
    so_inverse_sht_batch(p, draws, t_out, synth, threads);
    for (int t = 0; t < t_out; ++t) {
      double* slice = outr + (size_t)t * points;
      const double* m = means + (size_t)t * points;
      const double* sy = synth + (size_t)t * points;
      for (size_t loc = 0; loc < points; ++loc) {
        double eps = root_v2[loc] * slice[loc];
        slice[loc] = m[loc] + sigma[loc] * (sy[loc] + eps);
      }
    }
  }
  free(synth);
  free(draws);
  free(state);
  free(f);
  free(eta);
  free(root_v2);
  return 0;
}
