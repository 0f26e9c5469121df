// sphemu/stochastic.hpp — the hot-path part of proj/include/sphemu/stochastic.hpp
// (covariance + emulation generator, stochastic.hpp:36-86) without Eigen
// (absent here): matrices are dense row-major std::vector<double>,
// and emulate takes the model pieces it consumes explicitly (the trend is
// evaluated by the caller into per-step means, trend.cpp:252-287).
#pragma once

#include <cstdint>
#include <memory>
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

namespace detail {
// Owner of a device-resident tiled factor (sphemu_chol_t).
struct CholHandle {
  sphemu_chol_t h = nullptr;
  CholHandle() = default;
  explicit CholHandle(sphemu_chol_t x) : h(x) {}
  CholHandle(const CholHandle&) = delete;
  CholHandle& operator=(const CholHandle&) = delete;
  ~CholHandle() {
    if (h) sphemu_gpu_chol_destroy(h);
  }
};
}  // namespace detail

// InnovationModel (stochastic.hpp:36-42): u_hat and v are dim x dim row-major.
// `factor` (when set) is the same V kept on the device as tiles at their
// storage precision: emulate(EmulatorModel, ...) draws from it directly.
struct InnovationModel {
  int dim = 0;
  std::vector<double> u_hat;
  std::vector<double> v;
  double nugget = 0.0;
  PrecisionVariant factored_variant = PrecisionVariant::kDp;
  FactorizationStats factor_stats;
  std::shared_ptr<detail::CholHandle> factor;
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

// estimate_innovation_covariance keeping V on the device as the tiled factor
// (the handle train hands to emulate); residuals host or device (where).
inline InnovationModel estimate_innovation_factor(const double* residuals, int where, std::int64_t rows, int d,
                                                  int r_len, int t_len, int order, const MpCholConfig& chol_config,
                                                  bool dense_v = true) {
  chol_config.validate();
  const sphemu_chol_config c = chol_config.c_config();
  InnovationModel m;
  m.dim = d;
  m.u_hat.resize(static_cast<std::size_t>(d) * d);
  sphemu_chol_stats st{};
  sphemu_chol_t h = nullptr;
  detail::check(sphemu_gpu_innovation_factor(residuals, where, rows, d, r_len, t_len, order, &c, m.u_hat.data(),
                                             SPHEMU_HOST, &m.nugget, &st, &h));
  m.factor = std::make_shared<detail::CholHandle>(h);
  if (dense_v) {
    m.v.resize(static_cast<std::size_t>(d) * d);
    detail::check(sphemu_gpu_chol_store_dense(h, m.v.data(), SPHEMU_HOST, d));
  }
  m.factored_variant = chol_config.variant;
  m.factor_stats = detail::from_c(st);
  return m;
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

// NoiseField (stochastic.hpp:60-66) and fit_noise_field (stochastic.cpp:176-196) on the device.
struct NoiseField {
  GridSpec spec;
  std::vector<double> v2;
};

inline NoiseField fit_noise_field(const FieldSeries& detrended, const FieldSeries& reconstructed) {
  detrended.validate();
  reconstructed.validate();
  if (!(detrended.spec == reconstructed.spec) || detrended.t_len != reconstructed.t_len ||
      detrended.r_len != reconstructed.r_len)
    throw std::invalid_argument("detrended and reconstructed series differ in shape");
  NoiseField n;
  n.spec = detrended.spec;
  n.v2.resize(detrended.spec.points());
  detail::check(sphemu_gpu_noise_field(detrended.values.data(), reconstructed.values.data(), SPHEMU_HOST,
                                       static_cast<std::int64_t>(detrended.r_len) * detrended.t_len,
                                       static_cast<std::int64_t>(detrended.spec.points()), n.v2.data(), SPHEMU_HOST));
  return n;
}

// EmulatorModel (stochastic.hpp:68-79).
struct EmulatorModel {
  GridSpec spec;
  int band_limit = 0;
  TrendModel trend;
  VarModel var;
  InnovationModel innovation;
  NoiseField noise;

  void validate() const {  // stochastic.cpp:198-215
    spec.validate();
    if (band_limit < 1 || !spec.admissible(band_limit))
      throw std::invalid_argument("model band limit is not resolved by its grid");
    const std::size_t d = static_cast<std::size_t>(band_limit) * band_limit;
    if (!(trend.spec == spec)) throw std::invalid_argument("trend grid differs from model grid");
    if (trend.values.size() != spec.points() * trend.record_stride())
      throw std::invalid_argument("trend parameter block has the wrong size");
    if (var.band_limit != band_limit || var.phi.size() != static_cast<std::size_t>(var.order) * d)
      throw std::invalid_argument("lag coefficient block has the wrong size");
    if (innovation.dim != static_cast<int>(d) || innovation.u_hat.size() != d * d ||
        (innovation.v.size() != d * d && !innovation.factor))
      throw std::invalid_argument("innovation covariance has the wrong size");
    if (!(noise.spec == spec) || noise.v2.size() != spec.points())
      throw std::invalid_argument("noise field has the wrong size");
  }
};

// TrainConfig (pipeline.hpp): trend, lag order, band limit, factorization.
struct TrainConfig {
  int band_limit = 0;
  TrendConfig trend;
  int var_order = 2;
  MpCholConfig chol;
  int threads = 1;
};

// fit_trend(series, {}, config) (trend.cpp:129-250) without forcing, on the device.
inline TrendModel fit_trend(const FieldSeries& series, const ForcingTrajectory& forcing, TrendConfig config) {
  if (!forcing.x.empty() || !forcing.history.empty())
    throw std::invalid_argument("the device trend fit takes no forcing trajectory");
  series.validate();
  TrendModel m;
  m.spec = series.spec;
  m.config = config;
  m.values.resize(series.spec.points() * m.record_stride());
  detail::check(sphemu_gpu_fit_trend(series.values.data(), SPHEMU_HOST, series.r_len, series.t_len,
                                     static_cast<std::int64_t>(series.spec.points()), config.harmonics, config.period,
                                     m.values.data(), SPHEMU_HOST));
  return m;
}

// train (pipeline.cpp:18-54): trend -> detrend -> forward SHT -> fit_var ->
// innovation covariance + factor (kept on the device) -> noise field.
inline EmulatorModel train(const FieldSeries& series, const ForcingTrajectory& forcing, const TrainConfig& config) {
  series.validate();
  const int band_limit = config.band_limit > 0 ? config.band_limit : series.spec.max_band_limit();
  if (!series.spec.admissible(band_limit))
    throw std::invalid_argument("training grid does not resolve band limit " + std::to_string(band_limit));
  EmulatorModel model;
  model.spec = series.spec;
  model.band_limit = band_limit;
  model.trend = fit_trend(series, forcing, config.trend);
  FieldSeries standardized = detrend(series, model.trend, forcing);
  ShtPlan plan = build_plan(series.spec, band_limit);
  CoeffSeries coeffs = forward_sht_batch(plan, standardized, config.threads);
  VarFit vf = fit_var(coeffs, config.var_order);
  model.var = vf.model;
  model.innovation = estimate_innovation_factor(vf.residuals.data(), SPHEMU_HOST, vf.residual_rows,
                                                band_limit * band_limit, series.r_len, series.t_len, config.var_order,
                                                config.chol);
  FieldSeries reconstructed = inverse_sht_batch(plan, coeffs, config.threads);
  model.noise = fit_noise_field(standardized, reconstructed);
  model.validate();
  return model;
}

// emulate(model, plan, forcing, t_out, seed, r_len, threads, t_start)
// (stochastic.hpp:84-86): from the device-resident factor when the model
// holds one (sphemu_gpu_emulate_chol_trend), else from the dense V.
inline FieldSeries emulate(const EmulatorModel& model, const ShtPlan& plan, const ForcingTrajectory& forcing,
                           int t_out, std::uint64_t seed, int r_len = 1, int threads = 1, std::int64_t t_start = 1,
                           EmulationRng rng = EmulationRng::kReference) {
  (void)threads;
  model.validate();
  if (!(plan.spec == model.spec) || plan.band_limit != model.band_limit)
    throw std::invalid_argument("transform plan does not match the model");
  const int d = model.band_limit * model.band_limit;
  if (!model.innovation.factor)
    return emulate(plan, model.innovation.v, d, model.var.phi, model.var.order, model.trend, forcing, model.noise.v2,
                   t_out, seed, r_len, t_start, rng);
  FieldSeries out(plan.spec, t_out, r_len);
  std::vector<double> phi_pad(model.var.phi.begin(), model.var.phi.end());
  if (phi_pad.empty()) phi_pad.assign(static_cast<std::size_t>(d), 0.0);
  detail::check(sphemu_gpu_emulate_chol_trend(
      model.innovation.factor->h, plan.device->h, phi_pad.data(), model.var.order, model.trend.values.data(),
      model.trend.config.harmonics, model.trend.config.period, forcing.x.data(),
      static_cast<std::int64_t>(forcing.x.size()), forcing.history.data(),
      static_cast<std::int64_t>(forcing.history.size()), t_start, model.noise.v2.data(), t_out, seed, 0, r_len,
      static_cast<int>(rng), out.values.data(), SPHEMU_HOST));
  return out;
}

}  // namespace sphemu
