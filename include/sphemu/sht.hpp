// sphemu/sht.hpp — drop-in for proj/include/sphemu/sht.hpp:22-129 on the B200
// path. ShtPlan keeps the reference's public fields (spec, band_limit,
// wigner) and gains an opaque device plan (sphemu_gpu_sht_create); the
// transforms run on the GPU through the C-ABI (include/sphemu_gpu.h). The
// host-side operator tables of the CPU plan (e_phi, w1, w2, i_mat, FFTW
// plans) have no counterpart: the device plan holds the composed Legendre
// operators instead.
#pragma once

#include <complex>
#include <cstddef>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "sphemu/detail_status.hpp"
#include "sphemu/grid.hpp"
#include "sphemu/wigner.hpp"
#include "sphemu_gpu.h"

namespace sphemu {

// Packed real coefficients per degree l: m = 0, then (Re, Im) for m = 1..l (sht.hpp:24-45).
struct HarmonicVector {
  int band_limit = 0;
  std::vector<double> values;

  HarmonicVector() = default;
  explicit HarmonicVector(int l_max_plus_1)
      : band_limit(l_max_plus_1), values(static_cast<std::size_t>(l_max_plus_1) * l_max_plus_1, 0.0) {}
  static std::size_t packed_size(int band_limit) { return static_cast<std::size_t>(band_limit) * band_limit; }
  static std::size_t index_mean(int l) { return static_cast<std::size_t>(l) * l; }
  static std::size_t index_re(int l, int m) { return static_cast<std::size_t>(l) * l + 2 * m - 1; }
  static std::size_t index_im(int l, int m) { return static_cast<std::size_t>(l) * l + 2 * m; }

  // Negative m through z_{l,-m} = (-1)^m conj(z_{l,m}).
  std::complex<double> coeff(int l, int m) const {
    if (m == 0) return {values[index_mean(l)], 0.0};
    const int a = m < 0 ? -m : m;
    const std::complex<double> z{values[index_re(l, a)], values[index_im(l, a)]};
    if (m > 0) return z;
    return (a % 2 ? -1.0 : 1.0) * std::conj(z);
  }
  void set_coeff(int l, int m, std::complex<double> z) {
    if (m == 0) {
      values[index_mean(l)] = z.real();
      return;
    }
    values[index_re(l, m)] = z.real();
    values[index_im(l, m)] = z.imag();
  }
  // sum |z_{l,m}|^2 over m = -l..l.
  double parseval_energy() const {
    double e = 0.0;
    for (int l = 0; l < band_limit; ++l) {
      e += values[index_mean(l)] * values[index_mean(l)];
      for (int m = 1; m <= l; ++m) e += 2.0 * (values[index_re(l, m)] * values[index_re(l, m)] +
                                               values[index_im(l, m)] * values[index_im(l, m)]);
    }
    return e;
  }
};

// (replicate, time, packed index) series.
struct CoeffSeries {
  int band_limit = 0;
  int t_len = 0;
  int r_len = 0;
  std::vector<double> values;

  CoeffSeries() = default;
  CoeffSeries(int l_max_plus_1, int t, int r)
      : band_limit(l_max_plus_1), t_len(t), r_len(r),
        values(static_cast<std::size_t>(r) * t * l_max_plus_1 * l_max_plus_1, 0.0) {}
  std::size_t slice_stride() const { return HarmonicVector::packed_size(band_limit); }
  std::span<double> slice(int r, int t) {
    return {values.data() + (static_cast<std::size_t>(r) * t_len + t) * slice_stride(), slice_stride()};
  }
  std::span<const double> slice(int r, int t) const {
    return {values.data() + (static_cast<std::size_t>(r) * t_len + t) * slice_stride(), slice_stride()};
  }
};

namespace detail {
struct DevicePlan {
  sphemu_sht_t h = nullptr;
  ~DevicePlan() {
    if (h) sphemu_gpu_sht_destroy(h);
  }
};
}  // namespace detail

struct ShtPlan {
  GridSpec spec;
  int band_limit = 0;
  std::shared_ptr<const WignerTables> wigner;
  std::shared_ptr<detail::DevicePlan> device;  // the B200 plan (composed operators in HBM)

  int ext_len() const { return 2 * spec.n_theta - 2; }
  std::size_t fourier_cols() const { return static_cast<std::size_t>(2 * band_limit - 1); }
};

// build_plan (sht.cpp:111-171): invalid_argument on an inadmissible grid or a Wigner cap violation.
inline ShtPlan build_plan(GridSpec spec, int band_limit, std::shared_ptr<const WignerTables> tables = nullptr) {
  spec.validate();
  if (!spec.admissible(band_limit))
    throw std::invalid_argument("grid " + std::to_string(spec.n_theta) + "x" + std::to_string(spec.n_phi) +
                                " does not resolve band limit " + std::to_string(band_limit));
  if (tables && tables->band_limit() < band_limit)
    throw std::invalid_argument("Wigner tables cover a smaller band limit than requested");
  ShtPlan p;
  p.spec = spec;
  p.band_limit = band_limit;
  p.wigner = tables ? std::move(tables) : build_wigner_tables(band_limit);
  p.device = std::make_shared<detail::DevicePlan>();
  detail::check(
      sphemu_gpu_sht_create(spec.n_theta, spec.n_phi, band_limit, p.wigner->memory_cap_bytes(), &p.device->h));
  return p;
}

// Scratch of the CPU path; the device plan owns its buffers.
struct ShtWorkspace {};

inline void forward_sht(const ShtPlan& plan, std::span<const double> field, std::span<double> coeffs_out,
                        ShtWorkspace* = nullptr) {
  if (field.size() != plan.spec.points() || coeffs_out.size() != HarmonicVector::packed_size(plan.band_limit))
    throw std::invalid_argument("field or coefficient span has the wrong length");
  detail::check(sphemu_gpu_sht_forward(plan.device->h, field.data(), SPHEMU_HOST, 1, coeffs_out.data(), SPHEMU_HOST));
}

inline void inverse_sht(const ShtPlan& plan, std::span<const double> coeffs, std::span<double> field_out,
                        ShtWorkspace* = nullptr) {
  if (field_out.size() != plan.spec.points() || coeffs.size() != HarmonicVector::packed_size(plan.band_limit))
    throw std::invalid_argument("field or coefficient span has the wrong length");
  detail::check(sphemu_gpu_sht_inverse(plan.device->h, coeffs.data(), SPHEMU_HOST, 1, field_out.data(), SPHEMU_HOST));
}

inline HarmonicVector forward_sht(const ShtPlan& plan, const EquiangularField& field) {
  if (!(field.spec == plan.spec)) throw std::invalid_argument("field grid does not match the plan");
  HarmonicVector out(plan.band_limit);
  forward_sht(plan, field.values, out.values);
  return out;
}

inline EquiangularField inverse_sht(const ShtPlan& plan, const HarmonicVector& coeffs) {
  if (coeffs.band_limit != plan.band_limit) throw std::invalid_argument("band limit does not match the plan");
  EquiangularField out(plan.spec);
  inverse_sht(plan, coeffs.values, out.values);
  return out;
}

// synth_bandlimited (sht.hpp:143, sht.cpp:435-466): direct synthesis on any grid, including under-resolved ones.
inline EquiangularField synth_bandlimited(const HarmonicVector& coeffs, GridSpec target) {
  EquiangularField out(target);
  detail::check(sphemu_gpu_synth_bandlimited(coeffs.values.data(), SPHEMU_HOST, 1, coeffs.band_limit, target.n_theta,
                                             target.n_phi, out.values.data(), SPHEMU_HOST));
  return out;
}

// Batches (sht.cpp:374-404); threads is accepted for API parity (the device batches every slice).
inline CoeffSeries forward_sht_batch(const ShtPlan& plan, const FieldSeries& series, int threads = 1) {
  (void)threads;
  series.validate();
  if (!(series.spec == plan.spec)) throw std::invalid_argument("series grid does not match the plan");
  CoeffSeries out(plan.band_limit, series.t_len, series.r_len);
  detail::check(sphemu_gpu_sht_forward(plan.device->h, series.values.data(), SPHEMU_HOST,
                                       static_cast<int64_t>(series.r_len) * series.t_len, out.values.data(),
                                       SPHEMU_HOST));
  return out;
}

inline FieldSeries inverse_sht_batch(const ShtPlan& plan, const CoeffSeries& series, int threads = 1) {
  (void)threads;
  if (series.band_limit != plan.band_limit) throw std::invalid_argument("band limit does not match the plan");
  FieldSeries out(plan.spec, series.t_len, series.r_len);
  detail::check(sphemu_gpu_sht_inverse(plan.device->h, series.values.data(), SPHEMU_HOST,
                                       static_cast<int64_t>(series.r_len) * series.t_len, out.values.data(),
                                       SPHEMU_HOST));
  return out;
}

}  // namespace sphemu
