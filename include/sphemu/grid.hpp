// sphemu/grid.hpp — drop-in for proj/include/sphemu/grid.hpp:12-75 (the
// grid and field containers the SHT API consumes; host-side values only).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <numbers>
#include <span>
#include <stdexcept>
#include <vector>

namespace sphemu {

// Equiangular grid with both poles: theta_i = pi i / (n_theta - 1), phi_j = 2 pi j / n_phi (grid.cpp:18-38).
struct GridSpec {
  int n_theta = 0;
  int n_phi = 0;

  static GridSpec from_band_limit(int band_limit) {
    if (band_limit < 1) throw std::invalid_argument("band limit must be positive");
    return GridSpec{band_limit + 1, 2 * band_limit};
  }
  double theta(int i) const { return std::numbers::pi * i / (n_theta - 1); }
  double phi(int j) const { return 2.0 * std::numbers::pi * j / n_phi; }
  std::size_t points() const { return static_cast<std::size_t>(n_theta) * n_phi; }
  int max_band_limit() const { return std::min(n_theta - 1, (n_phi + 1) / 2); }
  bool admissible(int band_limit) const { return band_limit >= 1 && band_limit <= max_band_limit(); }
  void validate() const {
    if (n_theta < 2) throw std::invalid_argument("grid needs at least two latitude rings");
    if (n_phi < 1) throw std::invalid_argument("grid needs at least one longitude point");
  }
  bool operator==(const GridSpec&) const = default;
};

struct ResolutionSummary {
  int band_limit = 0;
  double degrees_per_cell = 0.0;
  double km_per_cell = 0.0;
  std::int64_t grid_points = 0;
};

inline ResolutionSummary resolution_summary(int band_limit) {
  if (band_limit < 2) throw std::invalid_argument("band limit must be at least 2");
  return ResolutionSummary{band_limit, 180.0 / band_limit, 180.0 * 111.2 / band_limit,
                           static_cast<std::int64_t>(band_limit - 1) * (2 * band_limit)};
}

// One field, row-major with theta the slow index.
struct EquiangularField {
  GridSpec spec;
  std::vector<double> values;

  EquiangularField() = default;
  explicit EquiangularField(GridSpec s) : spec(s), values(s.points(), 0.0) {}
  double& at(int i, int j) { return values[static_cast<std::size_t>(i) * spec.n_phi + j]; }
  double at(int i, int j) const { return values[static_cast<std::size_t>(i) * spec.n_phi + j]; }
};

// (replicate, time, theta, phi) series.
struct FieldSeries {
  GridSpec spec;
  int t_len = 0;
  int r_len = 0;
  std::vector<double> values;

  FieldSeries() = default;
  FieldSeries(GridSpec s, int t, int r)
      : spec(s), t_len(t), r_len(r), values(static_cast<std::size_t>(r) * t * s.points(), 0.0) {}
  std::size_t slice_stride() const { return spec.points(); }
  std::span<double> slice(int r, int t) {
    return {values.data() + (static_cast<std::size_t>(r) * t_len + t) * slice_stride(), slice_stride()};
  }
  std::span<const double> slice(int r, int t) const {
    return {values.data() + (static_cast<std::size_t>(r) * t_len + t) * slice_stride(), slice_stride()};
  }
  void validate() const {
    spec.validate();
    if (t_len < 1 || r_len < 1) throw std::invalid_argument("series needs t_len, r_len >= 1");
    if (values.size() != static_cast<std::size_t>(r_len) * t_len * spec.points())
      throw std::invalid_argument("series buffer does not match its dimensions");
    for (double v : values)
      if (!std::isfinite(v)) throw std::invalid_argument("series contains non-finite samples");
  }
};

}  // namespace sphemu
