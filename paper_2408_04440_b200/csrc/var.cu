// var.cu — fit_var (proj/src/stochastic.cpp:30-107) on the device: the
// per-coefficient AR(P) least squares that produces the innovation sample Xi
// feeding estimate_innovation_covariance.
//
// One thread per packed coefficient index; a CTA covers 128 consecutive
// indices, so every (replicate, step) row of the coefficient series is read
// fully coalesced, and the residual rows are written coalesced in the layout
// estimate_innovation_covariance consumes (rows replicate-major, columns the
// coefficient). Pass 1 accumulates the P x P normal matrix and right-hand
// side in the reference's (r, t) order with explicit round-to-nearest ops (no
// FMA contraction), so A and b are bitwise the reference's; the solve is a
// full-pivoting LU with Eigen's rank rule (|pivot| > 1e-13 |max pivot|,
// stochastic.cpp:72-74) and the standard errors come from the same factors.
// Pass 2 re-reads the series (L2-resident for typical sizes) for the
// residuals, their sum of squares and their column mean. Stability
// (companion spectral radius >= 1 - 1e-8, stochastic.cpp:19-27,101-102) is
// decided by the Schur-Cohn step-down test on the lag polynomial scaled to
// radius 1 - 1e-8 (all reflection coefficients inside the unit disc <=>
// every root strictly inside), no eigenvalue solver needed. HBM-bound:
// algorithmic bytes = 8 * r_len * t_len * d (series, read twice) + 8 * n_rows * d (residuals).
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

#include "common.cuh"
#include "sphemu_gpu.h"

namespace sphemu_gpu {
namespace {

constexpr int kVarThreads = 64;  // d is only L^2: small CTAs spread the indices over all SMs
constexpr int kMaxOrder = 16;
constexpr int kVarUnroll = 8;    // time rows in flight per thread (fast path)

__device__ __forceinline__ double ser(const double* c, int64_t d, int t_len, int r, int t, int64_t idx) {
  return __ldg(c + ((int64_t)r * t_len + t) * d + idx);
}

__device__ void lu_factor_solve(double* a, const double* rhs, int P, double* ph, bool& degenerate_out, int* rp, int* cp) {
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < i; ++j) a[i * P + j] = a[j * P + i];
  // Full-pivoting LU in place (Eigen FullPivLU): row perm rp, column perm cp.
  for (int i = 0; i < P; ++i) rp[i] = cp[i] = i;
  double maxpivot = 0.0;
  int rank = 0;
  for (int k = 0; k < P; ++k) {
    double big = -1.0;
    int bi = k, bj = k;
    for (int j = k; j < P; ++j)  // column-major scan: first maximum wins like Eigen's maxCoeff
      for (int i = k; i < P; ++i) {
        const double v = fabs(a[i * P + j]);
        if (v > big) { big = v; bi = i; bj = j; }
      }
    if (big > maxpivot) maxpivot = big;  // Eigen tracks the largest pivot seen
    if (big == 0.0) break;
    if (bi != k) {
      for (int j = 0; j < P; ++j) { const double tmp = a[k * P + j]; a[k * P + j] = a[bi * P + j]; a[bi * P + j] = tmp; }
      const int ti = rp[k]; rp[k] = rp[bi]; rp[bi] = ti;
    }
    if (bj != k) {
      for (int i = 0; i < P; ++i) { const double tmp = a[i * P + k]; a[i * P + k] = a[i * P + bj]; a[i * P + bj] = tmp; }
      const int tj = cp[k]; cp[k] = cp[bj]; cp[bj] = tj;
    }
    const double piv = a[k * P + k];
    for (int i = k + 1; i < P; ++i) a[i * P + k] /= piv;
    for (int i = k + 1; i < P; ++i)
      for (int j = k + 1; j < P; ++j) a[i * P + j] -= a[i * P + k] * a[k * P + j];
  }
  for (int k = 0; k < P; ++k)
    if (fabs(a[k * P + k]) > 1e-13 * maxpivot) ++rank;
  const bool degenerate = rank < P;
  // Solves A z = b through the factors: z = Q U^-1 L^-1 Pr b.
  auto lu_solve = [&](const double* b, double* z) {
    double w[kMaxOrder];
    for (int i = 0; i < P; ++i) w[i] = b[rp[i]];
    for (int i = 0; i < P; ++i)
      for (int j = 0; j < i; ++j) w[i] -= a[i * P + j] * w[j];
    for (int i = P - 1; i >= 0; --i) {
      for (int j = i + 1; j < P; ++j) w[i] -= a[i * P + j] * w[j];
      w[i] /= a[i * P + i];
    }
    for (int i = 0; i < P; ++i) z[cp[i]] = w[i];
  };
  if (degenerate) {
    for (int p = 0; p < P; ++p) ph[p] = 0.0;
  } else {
    lu_solve(rhs, ph);
  }
  degenerate_out = degenerate;
}

__device__ int finish_fit(const double* a, int P, const double* ph, bool degenerate, double rss, int64_t n_rows,
                                double* se_out, int64_t d, int64_t idx, const int* rp, const int* cp) {
  auto lu_solve = [&](const double* b, double* z) {
    double w[kMaxOrder];
    for (int i = 0; i < P; ++i) w[i] = b[rp[i]];
    for (int i = 0; i < P; ++i)
      for (int j = 0; j < i; ++j) w[i] -= a[i * P + j] * w[j];
    for (int i = P - 1; i >= 0; --i) {
      for (int j = i + 1; j < P; ++j) w[i] -= a[i * P + j] * w[j];
      w[i] /= a[i * P + i];
    }
    for (int i = 0; i < P; ++i) z[cp[i]] = w[i];
  };
  // Standard errors (stochastic.cpp:92-98): sqrt(max(0, s2 * (A^-1)_pp)).
  for (int p = 0; p < P; ++p) se_out[(int64_t)p * d + idx] = 0.0;
  if (!degenerate && n_rows > P) {
    const double s2 = rss / (double)(n_rows - P);
    double e_p[kMaxOrder], col[kMaxOrder];
    for (int p = 0; p < P; ++p) {
      for (int i = 0; i < P; ++i) e_p[i] = i == p ? 1.0 : 0.0;
      lu_solve(e_p, col);
      se_out[(int64_t)p * d + idx] = sqrt(fmax(0.0, s2 * col[p]));
    }
  }
  // Stability: roots of z^P - phi_1 z^(P-1) - ... - phi_P strictly inside
  // radius rho = 1 - 1e-8 <=> Schur-Cohn step-down of the polynomial in w = z / rho.
  const double rho = 1.0 - 1e-8;
  double c[kMaxOrder + 1];  // monic: c[0] = 1, c[k] = -phi_k / rho^k
  double rk = 1.0;
  c[0] = 1.0;
  for (int k = 1; k <= P; ++k) {
    rk *= rho;
    c[k] = -ph[k - 1] / rk;
  }
  bool unstable = false;
  for (int k = P; k >= 1 && !unstable; --k) {
    const double kap = c[k];
    if (fabs(kap) >= 1.0) {
      unstable = true;
      break;
    }
    const double den = 1.0 - kap * kap;
    double nc[kMaxOrder + 1];
    for (int i = 0; i < k; ++i) nc[i] = (c[i] - kap * c[k - i]) / den;
    for (int i = 0; i < k; ++i) c[i] = nc[i];
  }
  return (degenerate ? 1 : 0) | (unstable ? 2 : 0);
}

// Order 0 (stochastic.cpp:48-58): pooled demeaned series.
__device__ void fit_order0(const double* __restrict__ coeffs, int r_len, int t_len, int64_t d, int64_t idx,
                           double* __restrict__ resid, double* __restrict__ colmean, int* __restrict__ flags) {
  const int64_t n_rows = (int64_t)r_len * t_len;
  double mean = 0.0;
  for (int r = 0; r < r_len; ++r)
    for (int t = 0; t < t_len; ++t) mean = __dadd_rn(mean, ser(coeffs, d, t_len, r, t, idx));
  mean = __ddiv_rn(mean, (double)n_rows);
  double sum = 0.0;
  for (int r = 0; r < r_len; ++r)
    for (int t = 0; t < t_len; ++t) {
      const double e = __dsub_rn(ser(coeffs, d, t_len, r, t, idx), mean);
      resid[((int64_t)r * t_len + t) * d + idx] = e;
      sum += e;
    }
  colmean[idx] = sum / (double)n_rows;
  flags[idx] = 0;
}

// Fast path for a compile-time order: the lag window, A's upper triangle and
// b live in registers, kVarUnroll time rows are loaded before they are
// consumed (in order), so each warp keeps several coalesced row loads in flight.
template <int P>
__global__ void __launch_bounds__(kVarThreads) k_fit_var_fixed(const double* __restrict__ coeffs, int r_len,
                                                               int t_len, int64_t d, double* __restrict__ phi_out,
                                                               double* __restrict__ se_out,
                                                               double* __restrict__ resid,
                                                               double* __restrict__ colmean,
                                                               int* __restrict__ flags) {
  const int64_t idx = (int64_t)blockIdx.x * kVarThreads + threadIdx.x;
  if (idx >= d) return;
  const int64_t n_rows = (int64_t)r_len * (t_len - P);
  double au[P * (P + 1) / 2], rhs[P];
#pragma unroll
  for (int i = 0; i < P * (P + 1) / 2; ++i) au[i] = 0.0;
#pragma unroll
  for (int i = 0; i < P; ++i) rhs[i] = 0.0;
  // Pass 1 (stochastic.cpp:63-71): A += x x^T, b += x y in (r, t) order.
  for (int r = 0; r < r_len; ++r) {
    double win[P];  // win[p] = y(t - 1 - p)
#pragma unroll
    for (int p = 0; p < P; ++p) win[p] = ser(coeffs, d, t_len, r, P - 1 - p, idx);
    for (int t0 = P; t0 < t_len; t0 += kVarUnroll) {
      double yv[kVarUnroll];
#pragma unroll
      for (int u = 0; u < kVarUnroll; ++u)  // clamped, unpredicated: independent loads in flight
        yv[u] = ser(coeffs, d, t_len, r, min(t0 + u, t_len - 1), idx);
#pragma unroll
      for (int u = 0; u < kVarUnroll; ++u) {
        if (t0 + u < t_len) {
          int q = 0;
#pragma unroll
          for (int i = 0; i < P; ++i) {
#pragma unroll
            for (int j = i; j < P; ++j, ++q) au[q] = __dadd_rn(au[q], __dmul_rn(win[i], win[j]));
            rhs[i] = __dadd_rn(rhs[i], __dmul_rn(win[i], yv[u]));
          }
#pragma unroll
          for (int p = P - 1; p > 0; --p) win[p] = win[p - 1];
          win[0] = yv[u];
        }
      }
    }
  }
  double a[P * P];
  {
    int q = 0;
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int j = i; j < P; ++j, ++q) a[i * P + j] = au[q];
  }
  int rp[P], cp[P];
  double ph[P];
  bool degenerate;
  lu_factor_solve(a, rhs, P, ph, degenerate, rp, cp);
#pragma unroll
  for (int p = 0; p < P; ++p) phi_out[(int64_t)p * d + idx] = ph[p];
  // Pass 2 (stochastic.cpp:82-91): residuals, rss, column mean.
  const int rows_per_rep = t_len - P;
  double rss = 0.0, sum = 0.0;
  for (int r = 0; r < r_len; ++r) {
    double win[P];
#pragma unroll
    for (int p = 0; p < P; ++p) win[p] = ser(coeffs, d, t_len, r, P - 1 - p, idx);
    for (int t0 = P; t0 < t_len; t0 += kVarUnroll) {
      double yv[kVarUnroll];
#pragma unroll
      for (int u = 0; u < kVarUnroll; ++u)  // clamped, unpredicated: independent loads in flight
        yv[u] = ser(coeffs, d, t_len, r, min(t0 + u, t_len - 1), idx);
#pragma unroll
      for (int u = 0; u < kVarUnroll; ++u) {
        if (t0 + u < t_len) {
          double pred = 0.0;
#pragma unroll
          for (int p = 0; p < P; ++p) pred = __dadd_rn(pred, __dmul_rn(ph[p], win[p]));
          const double e = __dsub_rn(yv[u], pred);
          __stcs(resid + ((int64_t)r * rows_per_rep + (t0 + u - P)) * d + idx, e);
          rss = __dadd_rn(rss, __dmul_rn(e, e));
          sum += e;
#pragma unroll
          for (int p = P - 1; p > 0; --p) win[p] = win[p - 1];
          win[0] = yv[u];
        }
      }
    }
  }
  colmean[idx] = sum / (double)n_rows;
  flags[idx] = finish_fit(a, P, ph, degenerate, rss, n_rows, se_out, d, idx, rp, cp);
}

// Generic order (5..16) and order 0.
__global__ void __launch_bounds__(kVarThreads) k_fit_var(const double* __restrict__ coeffs, int r_len, int t_len,
                                                         int64_t d, int order, double* __restrict__ phi_out,
                                                         double* __restrict__ se_out, double* __restrict__ resid,
                                                         double* __restrict__ colmean, int* __restrict__ flags) {
  const int64_t idx = (int64_t)blockIdx.x * kVarThreads + threadIdx.x;
  if (idx >= d) return;
  const int P = order;
  if (P == 0) {
    fit_order0(coeffs, r_len, t_len, d, idx, resid, colmean, flags);
    return;
  }
  const int64_t n_rows = (int64_t)r_len * (t_len - P);
  double a[kMaxOrder * kMaxOrder], rhs[kMaxOrder], x[kMaxOrder];
  for (int i = 0; i < P * P; ++i) a[i] = 0.0;
  for (int i = 0; i < P; ++i) rhs[i] = 0.0;
  for (int r = 0; r < r_len; ++r)
    for (int t = P; t < t_len; ++t) {
      for (int p = 0; p < P; ++p) x[p] = ser(coeffs, d, t_len, r, t - 1 - p, idx);
      const double y = ser(coeffs, d, t_len, r, t, idx);
      for (int i = 0; i < P; ++i) {
        for (int j = i; j < P; ++j) a[i * P + j] = __dadd_rn(a[i * P + j], __dmul_rn(x[i], x[j]));
        rhs[i] = __dadd_rn(rhs[i], __dmul_rn(x[i], y));
      }
    }
  int rp[kMaxOrder], cp[kMaxOrder];
  double ph[kMaxOrder];
  bool degenerate;
  lu_factor_solve(a, rhs, P, ph, degenerate, rp, cp);
  for (int p = 0; p < P; ++p) phi_out[(int64_t)p * d + idx] = ph[p];
  const int rows_per_rep = t_len - P;
  double rss = 0.0, sum = 0.0;
  for (int r = 0; r < r_len; ++r)
    for (int t = P; t < t_len; ++t) {
      double pred = 0.0;
      for (int p = 0; p < P; ++p) pred = __dadd_rn(pred, __dmul_rn(ph[p], ser(coeffs, d, t_len, r, t - 1 - p, idx)));
      const double e = __dsub_rn(ser(coeffs, d, t_len, r, t, idx), pred);
      resid[((int64_t)r * rows_per_rep + (t - P)) * d + idx] = e;
      rss = __dadd_rn(rss, __dmul_rn(e, e));
      sum += e;
    }
  colmean[idx] = sum / (double)n_rows;
  flags[idx] = finish_fit(a, P, ph, degenerate, rss, n_rows, se_out, d, idx, rp, cp);
}

}  // namespace
}  // namespace sphemu_gpu

extern "C" int sphemu_gpu_fit_var(const double* coeffs, int where_in, int r_len, int t_len, int64_t d, int order,
                                  double* phi, double* phi_se, double* residuals, int where_resid,
                                  int64_t* zeroed_count, int64_t* unstable_count, double* residual_mean_norm) {
  using namespace sphemu_gpu;
  return guard([&] {
    if (order < 0) throw std::invalid_argument("lag order must be non-negative");
    if (t_len <= order) throw std::invalid_argument("series too short for the requested lag order");
    if (order > kMaxOrder) throw std::invalid_argument("lag order must lie in [0, 16]");
    if (r_len < 1 || d < 1) throw std::invalid_argument("empty coefficient series");
    const int64_t n_rows = (int64_t)r_len * (t_len - order);
    const size_t n_in = (size_t)r_len * t_len * d, n_res = (size_t)n_rows * d;
    // One device block for the small outputs: phi | se | column means | flags.
    const int64_t op = order > 0 ? order : 0;
    DevBuf<double> dIn, dRes;
    double* const dSmall = scratch<double>(0, (size_t)(2 * op + 2) * d);
    double* dPhi = dSmall;
    double* dSe = dPhi + op * d;
    double* dMean = dSe + op * d;
    int* dFlags = reinterpret_cast<int*>(dMean + d);
    const double* cin = coeffs;
    if (where_in == SPHEMU_HOST) {
      dIn.alloc(n_in);
      SPH_CUDA(cudaMemcpy(dIn.get(), coeffs, sizeof(double) * n_in, cudaMemcpyHostToDevice));
      cin = dIn.get();
    }
    double* res = residuals;
    if (where_resid == SPHEMU_HOST) {
      dRes.alloc(n_res);
      res = dRes.get();
    }
    const unsigned grid = (unsigned)ceil_div(d, kVarThreads);
    switch (order) {
      case 1: k_fit_var_fixed<1><<<grid, kVarThreads>>>(cin, r_len, t_len, d, dPhi, dSe, res, dMean, dFlags); break;
      case 2: k_fit_var_fixed<2><<<grid, kVarThreads>>>(cin, r_len, t_len, d, dPhi, dSe, res, dMean, dFlags); break;
      case 3: k_fit_var_fixed<3><<<grid, kVarThreads>>>(cin, r_len, t_len, d, dPhi, dSe, res, dMean, dFlags); break;
      case 4: k_fit_var_fixed<4><<<grid, kVarThreads>>>(cin, r_len, t_len, d, dPhi, dSe, res, dMean, dFlags); break;
      default: k_fit_var<<<grid, kVarThreads>>>(cin, r_len, t_len, d, order, dPhi, dSe, res, dMean, dFlags);
    }
    SPH_LAUNCH_CHECK();
    if (where_resid == SPHEMU_HOST)
      SPH_CUDA(cudaMemcpy(residuals, res, sizeof(double) * n_res, cudaMemcpyDeviceToHost));
    std::vector<double> small((size_t)(2 * op + 2) * d);
    SPH_CUDA(cudaMemcpy(small.data(), dSmall, sizeof(double) * small.size(), cudaMemcpyDeviceToHost));
    if (op > 0) {
      if (phi) std::copy(small.begin(), small.begin() + op * d, phi);
      if (phi_se) std::copy(small.begin() + op * d, small.begin() + 2 * op * d, phi_se);
    }
    const double* mean = small.data() + 2 * op * d;
    const int* flags = reinterpret_cast<const int*>(mean + d);
    int64_t zeroed = 0, unstable = 0;
    double ss = 0.0;
    for (int64_t i = 0; i < d; ++i) {
      zeroed += flags[i] & 1;
      unstable += (flags[i] >> 1) & 1;
      ss += mean[i] * mean[i];
    }
    if (zeroed_count) *zeroed_count = zeroed;
    if (unstable_count) *unstable_count = unstable;
    if (residual_mean_norm) *residual_mean_norm = std::sqrt(ss);
  });
}
