// sphemu/trend.hpp — the mean-structure part of proj/include/sphemu/trend.hpp
// (TrendConfig, ForcingTrajectory, TrendModel, mean_table, detrend, retrend;
// trend.hpp:14-82) backed by the device kernels of trend.cu. fit_trend
// (Eigen least squares) and the TRND file format stay out of scope.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

#include "sphemu/detail_status.hpp"
#include "sphemu/grid.hpp"
#include "sphemu_gpu.h"

namespace sphemu {

struct TrendConfig {  // trend.hpp:14-20
  int harmonics = 5;
  int period = 8760;

  void validate() const {  // trend.cpp:27-33
    if (period != 12 && period != 365 && period != 8760)
      throw std::invalid_argument("period must be 12, 365 or 8760 steps per year");
    if (harmonics < 0) throw std::invalid_argument("harmonics must be non-negative");
    if (2 * harmonics >= period) throw std::invalid_argument("harmonics must stay below half the period");
  }
};

struct ForcingTrajectory {  // trend.hpp:24-35
  std::vector<double> x;
  std::vector<double> history;
  bool empty() const { return x.empty() && history.empty(); }
};

struct TrendModel {  // trend.hpp:37-59 (records: beta0, beta1, beta2, rho, a_1..a_K, b_1..b_K, sigma)
  GridSpec spec;
  TrendConfig config;
  std::vector<double> values;
  int collinear_warnings = 0;

  std::size_t record_stride() const { return 5 + 2 * static_cast<std::size_t>(config.harmonics); }
  double sigma(std::size_t loc) const { return values[loc * record_stride() + record_stride() - 1]; }
};

// mean_table (trend.hpp:79-82): t_len x points, time-major.
inline std::vector<double> mean_table(const TrendModel& model, const ForcingTrajectory& forcing, int t_len,
                                      std::int64_t t_start = 1) {
  const std::int64_t points = static_cast<std::int64_t>(model.spec.points());
  std::vector<double> table(static_cast<std::size_t>(t_len < 0 ? 0 : t_len) * points);
  detail::check(sphemu_gpu_mean_table(model.values.data(), points, model.config.harmonics, model.config.period,
                                      forcing.x.data(), static_cast<std::int64_t>(forcing.x.size()),
                                      forcing.history.data(), static_cast<std::int64_t>(forcing.history.size()),
                                      t_len, t_start, table.data(), SPHEMU_HOST));
  return table;
}

namespace detail {
template <class F>
FieldSeries trend_apply(F fn, const FieldSeries& series, const TrendModel& model, const ForcingTrajectory& forcing,
                        std::int64_t t_start) {
  if (!(series.spec == model.spec)) throw std::invalid_argument("series grid differs from model");
  FieldSeries out(series.spec, series.t_len, series.r_len);
  check(fn(series.values.data(), SPHEMU_HOST, series.r_len, series.t_len, model.values.data(),
           static_cast<std::int64_t>(model.spec.points()), model.config.harmonics, model.config.period,
           forcing.x.data(), static_cast<std::int64_t>(forcing.x.size()), forcing.history.data(),
           static_cast<std::int64_t>(forcing.history.size()), t_start, out.values.data(), SPHEMU_HOST));
  return out;
}
}  // namespace detail

// Standardized residuals (y - m_t) / sigma (trend.hpp:69-71).
inline FieldSeries detrend(const FieldSeries& series, const TrendModel& model, const ForcingTrajectory& forcing,
                           std::int64_t t_start = 1) {
  return detail::trend_apply(sphemu_gpu_detrend, series, model, forcing, t_start);
}

// Inverse map m_t + sigma * z (trend.hpp:73-75).
inline FieldSeries retrend(const FieldSeries& standardized, const TrendModel& model,
                           const ForcingTrajectory& forcing, std::int64_t t_start = 1) {
  return detail::trend_apply(sphemu_gpu_retrend, standardized, model, forcing, t_start);
}

}  // namespace sphemu
