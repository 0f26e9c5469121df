/* so_trend.c — CPU restatement of the reference's trend mean structure
 * (TEST INFRASTRUCTURE, see sphemu_oracle.h). Follows proj/src/trend.cpp:
 * year_of / require_lag_history (18-25), ForcingTrajectory::has_year /
 * at_year / lagged_mean (35-57), eval_mean_trend (65-83), mean_table
 * (252-287), detrend (289-305), retrend (307-324). Built with
 * -ffp-contract=off like the reference's default Release build. */
#include <math.h>
#include <stdlib.h>

#include "sphemu_oracle.h"

static const double kTwoPi = 2.0 * 3.14159265358979323846; /* trend.cpp:14 */
static const double kLagWeightCutoff = 1e-12;              /* trend.cpp:15 */

static int64_t year_of(int64_t t, int period) { return (t + period - 1) / period; }

static int has_year(const double* fx, int64_t nx, const double* fh, int64_t nh, int64_t year) {
  (void)fx;
  (void)fh;
  if (year >= 1) return year <= nx;
  return -year < nh;
}

static double at_year(const double* fx, int64_t nx, const double* fh, int64_t nh, int64_t year) {
  if (!has_year(fx, nx, fh, nh, year)) return 0.0;
  if (year >= 1) return fx[year - 1];
  return fh[-year];
}

static double lagged_mean(const double* fx, int64_t nx, const double* fh, int64_t nh, int64_t year, double rho) {
  double acc = 0.0, w = 1.0;
  for (int64_t s = 1;; ++s) {
    if (!has_year(fx, nx, fh, nh, year - s)) break;
    acc += w * at_year(fx, nx, fh, nh, year - s);
    w *= rho;
    if (w < kLagWeightCutoff) break;
  }
  return (1.0 - rho) * acc;
}

double so_eval_mean_trend(const double* records, int harmonics, int period, int64_t loc, int64_t t,
                          const double* fx, int64_t n_x, const double* fh, int64_t n_h, int* err) {
  const double* rec = records + loc * (5 + 2 * (int64_t)harmonics);
  double m = rec[0];
  *err = 0;
  if (n_x != 0 || n_h != 0) {
    int64_t year = year_of(t, period);
    if (rec[2] != 0.0 && !has_year(fx, n_x, fh, n_h, year - 1)) {
      *err = -2;
      return 0.0;
    }
    m += rec[1] * at_year(fx, n_x, fh, n_h, year) + rec[2] * lagged_mean(fx, n_x, fh, n_h, year, rec[3]);
  }
  double base = kTwoPi * (double)(t % period) / period;
  for (int k = 1; k <= harmonics; ++k)
    m += rec[4 + (k - 1)] * cos(base * k) + rec[4 + harmonics + (k - 1)] * sin(base * k);
  return m;
}

int so_mean_table(const double* records, int64_t points, int harmonics, int period,
                  const double* fx, int64_t n_x, const double* fh, int64_t n_h,
                  int t_len, int64_t t_start, double* table) {
  if (t_start < 1) return -1;
  const int64_t stride = 5 + 2 * (int64_t)harmonics;
  const int big_k = harmonics;
  double* cs = (double*)malloc(sizeof(double) * 2 * (big_k > 1 ? big_k : 1));
  const int with_forcing = n_x != 0 || n_h != 0;
  for (int row = 0; row < t_len; ++row) {
    int64_t t = t_start + row;
    double base = kTwoPi * (double)(t % period) / period;
    for (int k = 1; k <= big_k; ++k) {
      cs[2 * (k - 1)] = cos(base * k);
      cs[2 * (k - 1) + 1] = sin(base * k);
    }
    double xv = 0.0, lv = 0.0;
    int64_t year = year_of(t, period);
    if (with_forcing) xv = at_year(fx, n_x, fh, n_h, year);
    double* out = table + (int64_t)row * points;
    for (int64_t loc = 0; loc < points; ++loc) {
      const double* rec = records + loc * stride;
      double m = rec[0];
      if (with_forcing) {
        if (rec[2] != 0.0 && !has_year(fx, n_x, fh, n_h, year - 1)) {
          free(cs);
          return -2;
        }
        if (loc == 0) lv = lagged_mean(fx, n_x, fh, n_h, year, rec[3]);
        m += rec[1] * xv + rec[2] * lv;
      }
      for (int k = 1; k <= big_k; ++k)
        m += rec[4 + (k - 1)] * cs[2 * (k - 1)] + rec[4 + big_k + (k - 1)] * cs[2 * (k - 1) + 1];
      out[loc] = m;
    }
  }
  free(cs);
  return 0;
}

int so_trend_apply(int mode, const double* in, int r_len, int t_len, const double* records, int64_t points,
                   int harmonics, int period, const double* fx, int64_t n_x, const double* fh, int64_t n_h,
                   int64_t t_start, double* out) {
  const int64_t stride = 5 + 2 * (int64_t)harmonics;
  double* table = (double*)malloc(sizeof(double) * ((size_t)t_len * points + 1));
  int rc = so_mean_table(records, points, harmonics, period, fx, n_x, fh, n_h, t_len, t_start, table);
  if (rc) {
    free(table);
    return rc;
  }
  for (int r = 0; r < r_len; ++r)
    for (int t = 0; t < t_len; ++t) {
      const double* src = in + ((int64_t)r * t_len + t) * points;
      double* dst = out + ((int64_t)r * t_len + t) * points;
      const double* m = table + (int64_t)t * points;
      for (int64_t loc = 0; loc < points; ++loc) {
        const double sigma = records[loc * stride + stride - 1];
        dst[loc] = mode == 0 ? (src[loc] - m[loc]) / sigma : m[loc] + sigma * src[loc];
      }
    }
  free(table);
  return 0;
}
