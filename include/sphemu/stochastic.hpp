// sphemu/stochastic.hpp — the hot-path part of proj/include/sphemu/stochastic.hpp
// (covariance + emulation generator, stochastic.hpp:36-86) without Eigen
// (absent here): matrices are dense row-major std::vector<double>,
// and emulate takes the model pieces it consumes explicitly (the trend is
// evaluated by the caller into per-step means, trend.cpp:252-287).
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "sphemu/detail_status.hpp"
#include "sphemu/grid.hpp"
#include "sphemu/mpchol.hpp"
#include "sphemu/sht.hpp"
#include "sphemu/trend.hpp"
#include "sphemu_gpu.h"

namespace sphemu {

// InnovationModel (stochastic.hpp:36-42): u_hat and v are dim x dim row-major.
struct InnovationModel {
  int dim = 0;
  std::vector<double> u_hat;
  std::vector<double> v;
  double nugget = 0.0;
  PrecisionVariant factored_variant = PrecisionVariant::kDp;
  FactorizationStats factor_stats;
};

// estimate_innovation_covariance (stochastic.cpp:109-172) on the device;
// residuals is rows x d row-major with rows = r_len * (t_len - order).
inline InnovationModel estimate_innovation_covariance(std::span<const double> residuals, std::int64_t rows, int d,
                                                      int r_len, int t_len, int order,
                                                      const MpCholConfig& chol_config, int threads = 1) {
  (void)threads;
  if (d < 1 || residuals.size() != static_cast<std::size_t>(rows) * d)
    throw std::invalid_argument("residual buffer does not match rows x d");
  chol_config.validate();
  const sphemu_chol_config c = chol_config.c_config();
  InnovationModel m;
  m.dim = d;
  m.u_hat.resize(static_cast<std::size_t>(d) * d);
  m.v.resize(static_cast<std::size_t>(d) * d);
  sphemu_chol_stats st{};
  detail::check(sphemu_gpu_estimate_innovation_covariance(residuals.data(), SPHEMU_HOST, rows, d, r_len, t_len,
                                                          order, &c, m.u_hat.data(), SPHEMU_HOST, m.v.data(),
                                                          SPHEMU_HOST, &m.nugget, &st));
  m.factored_variant = chol_config.variant;
  m.factor_stats = detail::from_c(st);
  return m;
}

enum class EmulationRng { kReference = SPHEMU_RNG_REFERENCE, kPhilox = SPHEMU_RNG_PHILOX };

// emulate (stochastic.cpp:217-277): r_len replicates of t_out steps. v is the
// d x d innovation factor, phi the order x d lag coefficients, means
// t_out x points, sigma and v2 per point. kReference reproduces the
// reference's single serial random stream; kPhilox draws on the device.
inline FieldSeries emulate(const ShtPlan& plan, std::span<const double> v, int d, std::span<const double> phi,
                           int order, std::span<const double> means, std::span<const double> sigma,
                           std::span<const double> v2, int t_out, std::uint64_t seed, int r_len = 1,
                           EmulationRng rng = EmulationRng::kReference) {
  const std::size_t pts = plan.spec.points();
  if (d != plan.band_limit * plan.band_limit || v.size() != static_cast<std::size_t>(d) * d ||
      phi.size() != static_cast<std::size_t>(order) * d || means.size() != static_cast<std::size_t>(t_out) * pts ||
      sigma.size() != pts || v2.size() != pts)
    throw std::invalid_argument("emulation inputs do not match the plan");
  FieldSeries out(plan.spec, t_out, r_len);
  std::vector<double> phi_pad(phi.begin(), phi.end());
  if (phi_pad.empty()) phi_pad.assign(static_cast<std::size_t>(d), 0.0);
  detail::check(sphemu_gpu_emulate(plan.device->h, v.data(), d, phi_pad.data(), order, means.data(), sigma.data(),
                                   v2.data(), t_out, seed, r_len, static_cast<int>(rng), out.values.data()));
  return out;
}

// emulate(model, plan, forcing, t_out, seed, r_len, threads, t_start)
// (stochastic.hpp:84-86) with the model's trend and forcing: the mean table
// (stochastic.cpp:229) and sigma are evaluated on the device.
inline FieldSeries emulate(const ShtPlan& plan, std::span<const double> v, int d, std::span<const double> phi,
                           int order, const TrendModel& trend, const ForcingTrajectory& forcing,
                           std::span<const double> v2, int t_out, std::uint64_t seed, int r_len = 1,
                           std::int64_t t_start = 1, EmulationRng rng = EmulationRng::kReference) {
  const std::size_t pts = plan.spec.points();
  if (!(trend.spec == plan.spec) || d != plan.band_limit * plan.band_limit ||
      v.size() != static_cast<std::size_t>(d) * d || phi.size() != static_cast<std::size_t>(order) * d ||
      trend.values.size() != pts * trend.record_stride() || v2.size() != pts)
    throw std::invalid_argument("transform plan does not match the model");
  FieldSeries out(plan.spec, t_out, r_len);
  std::vector<double> phi_pad(phi.begin(), phi.end());
  if (phi_pad.empty()) phi_pad.assign(static_cast<std::size_t>(d), 0.0);
  detail::check(sphemu_gpu_emulate_trend(plan.device->h, v.data(), d, phi_pad.data(), order, trend.values.data(),
                                         trend.config.harmonics, trend.config.period, forcing.x.data(),
                                         static_cast<std::int64_t>(forcing.x.size()), forcing.history.data(),
                                         static_cast<std::int64_t>(forcing.history.size()), t_start, v2.data(), t_out,
                                         seed, r_len, static_cast<int>(rng), out.values.data()));
  return out;
}

// VarModel / VarFit (stochastic.hpp:18-37) with the residuals as a dense
// row-major (rows x d) vector instead of an Eigen matrix.
struct VarModel {
  int band_limit = 0;
  int order = 0;
  std::vector<double> phi;  // order rows of band_limit^2 coefficients
  std::int64_t zeroed_count = 0;
  std::int64_t unstable_count = 0;
  double phi_at(int p, std::size_t idx) const {
    return phi[static_cast<std::size_t>(p - 1) * band_limit * band_limit + idx];
  }
};

struct VarFit {
  VarModel model;
  std::int64_t residual_rows = 0;
  std::vector<double> residuals;
  std::vector<double> phi_se;
  double residual_mean_norm = 0.0;
};

// fit_var (stochastic.cpp:30-107) on the device.
inline VarFit fit_var(const CoeffSeries& coeffs, int order) {
  const std::int64_t d = static_cast<std::int64_t>(coeffs.slice_stride());
  VarFit fit;
  fit.model.band_limit = coeffs.band_limit;
  fit.model.order = order;
  const int rows_per_rep = order > 0 ? coeffs.t_len - order : coeffs.t_len;
  fit.residual_rows = static_cast<std::int64_t>(coeffs.r_len) * (rows_per_rep > 0 ? rows_per_rep : 0);
  fit.residuals.resize(static_cast<std::size_t>(fit.residual_rows * d));
  fit.model.phi.assign(static_cast<std::size_t>(order > 0 ? order : 0) * d, 0.0);
  fit.phi_se.assign(fit.model.phi.size(), 0.0);
  detail::check(sphemu_gpu_fit_var(coeffs.values.data(), SPHEMU_HOST, coeffs.r_len, coeffs.t_len, d, order,
                                   fit.model.phi.data(), fit.phi_se.data(), fit.residuals.data(), SPHEMU_HOST,
                                   &fit.model.zeroed_count, &fit.model.unstable_count, &fit.residual_mean_norm));
  return fit;
}

}  // namespace sphemu
