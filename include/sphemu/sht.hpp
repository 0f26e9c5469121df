// sphemu/sht.hpp — drop-in for proj/include/sphemu/sht.hpp:22-129 on the B200
// path. ShtPlan keeps the reference's public fields (spec, band_limit,
// wigner) and gains an opaque device plan (sphemu_gpu_sht_create); the
// transforms run on the GPU through the C-ABI (include/sphemu_gpu.h). The
// host-side operator tables of the CPU plan (e_phi, w1, w2, i_mat, FFTW
// plans) have no counterpart: the device plan holds the composed Legendre
// operators instead.
#pragma once

#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <memory>
#include <random>
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
  p.wigner = tables ? std::move(tables) : detail_lazy_wigner_tables(band_limit, std::size_t{2} << 30);
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

// ---- generators and independent checks (sht.hpp:20-23,130-163) ----------
// Host utilities of the reference's header: test-data generators and
// quadrature references, not the transform path (which is the device plan).

// I(q) = int_0^pi e^{iq theta} sin theta d theta (sht.cpp:30-37).
inline std::complex<double> i_integral(long long q) {
  const double pi = 3.14159265358979323846;
  if (q & 1) {
    if (q == 1) return {0.0, pi / 2.0};
    if (q == -1) return {0.0, -pi / 2.0};
    return {0.0, 0.0};
  }
  return {2.0 / (1.0 - static_cast<double>(q) * static_cast<double>(q)), 0.0};
}

// 4pi-normalized P~_{l,m}(cos theta) with Condon-Shortley phase, packed by
// l(l+1)/2 + m (sht.cpp:406-427).
inline std::vector<double> normalized_legendre_all(int band_limit, double theta) {
  const double pi = 3.14159265358979323846;
  const int big_l = band_limit;
  std::vector<double> p(static_cast<std::size_t>(big_l) * (big_l + 1) / 2, 0.0);
  const double ct = std::cos(theta), st = std::sin(theta);
  auto at = [&p](int l, int m) -> double& { return p[static_cast<std::size_t>(l) * (l + 1) / 2 + m]; };
  at(0, 0) = 1.0 / std::sqrt(4.0 * pi);
  for (int m = 1; m < big_l; ++m) at(m, m) = -std::sqrt((2.0 * m + 1.0) / (2.0 * m)) * st * at(m - 1, m - 1);
  for (int m = 0; m + 1 < big_l; ++m) at(m + 1, m) = std::sqrt(2.0 * m + 3.0) * ct * at(m, m);
  for (int m = 0; m < big_l; ++m)
    for (int l = m + 2; l < big_l; ++l) {
      const double a = std::sqrt((4.0 * l * l - 1.0) / (static_cast<double>(l) * l - m * m));
      const double b = std::sqrt((static_cast<double>(l - 1) * (l - 1) - m * m) /
                                 (4.0 * static_cast<double>(l - 1) * (l - 1) - 1.0));
      at(l, m) = a * (ct * at(l - 1, m) - b * at(l - 2, m));
    }
  return p;
}

inline double normalized_legendre(int l, int m, double theta) {
  if (l < 0 || m < 0 || m > l) throw std::out_of_range("Legendre index");
  return normalized_legendre_all(l + 1, theta)[static_cast<std::size_t>(l) * (l + 1) / 2 + m];
}

// Packed slots ~ N(0, (1/(l+1))^2) from the reference's GaussianRng stream
// (sht.cpp:507-518, rng.hpp:12-39: mt19937_64 >> 11 uniforms, Box-Muller with a spare).
inline HarmonicVector draw_random_coefficients(int band_limit, std::uint64_t seed) {
  if (band_limit < 1) throw std::invalid_argument("band limit must be positive");
  HarmonicVector out(band_limit);
  std::mt19937_64 eng(seed);
  double spare = 0.0;
  bool has = false;
  auto normal = [&]() {
    if (has) {
      has = false;
      return spare;
    }
    const double u1 = static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(a);
    has = true;
    return r * std::cos(a);
  };
  for (int l = 0; l < band_limit; ++l) {
    const double scale = 1.0 / (l + 1);
    const std::size_t lo = HarmonicVector::index_mean(l);
    for (std::size_t idx = lo; idx <= lo + 2 * static_cast<std::size_t>(l); ++idx) out.values[idx] = scale * normal();
  }
  return out;
}

// draw_random_coefficients followed by the (device) inverse transform (sht.cpp:520-527).
inline EquiangularField synth_random_field(const ShtPlan& plan, std::uint64_t seed) {
  return inverse_sht(plan, draw_random_coefficients(plan.band_limit, seed));
}
inline EquiangularField synth_random_field(GridSpec spec, int band_limit, std::uint64_t seed) {
  return synth_random_field(build_plan(spec, band_limit), seed);
}

namespace detail {
inline void naive_dft(const std::complex<double>* in, std::complex<double>* out, int n) {  // sign -1
  const double tp = 6.283185307179586476925286766559;
  for (int k = 0; k < n; ++k) {
    std::complex<double> s{0.0, 0.0};
    for (int j = 0; j < n; ++j) s += in[j] * std::polar(1.0, -tp * static_cast<double>((static_cast<long long>(k) * j) % n) / n);
    out[k] = s;
  }
}
}  // namespace detail

// Trapezoid-in-theta quadrature analysis of a function (sht.cpp:468-505): an
// independent reference, O(n_theta_quad L^2).
inline HarmonicVector quadrature_oracle_sht(const std::function<double(double, double)>& f, int band_limit,
                                            int n_theta_quad) {
  if (band_limit < 1 || n_theta_quad < 3) throw std::invalid_argument("oracle needs a band limit and at least 3 rings");
  const double pi = 3.14159265358979323846, two_pi = 2.0 * pi;
  const int big_l = band_limit, n_phi = 2 * big_l;
  const double h = pi / (n_theta_quad - 1);
  HarmonicVector out(big_l);
  std::vector<std::complex<double>> f_m(big_l), acc(static_cast<std::size_t>(big_l) * (big_l + 1) / 2, {0.0, 0.0});
  std::vector<double> ring(n_phi);
  for (int i = 0; i < n_theta_quad; ++i) {
    const double theta = h * i;
    const double w = h * std::sin(theta) * ((i == 0 || i == n_theta_quad - 1) ? 0.5 : 1.0);
    if (w == 0.0) continue;
    for (int j = 0; j < n_phi; ++j) ring[j] = f(theta, two_pi * j / n_phi);
    for (int m = 0; m < big_l; ++m) {
      std::complex<double> s{0.0, 0.0};
      for (int j = 0; j < n_phi; ++j) s += ring[j] * std::polar(1.0, -m * two_pi * j / n_phi);
      f_m[m] = s * (two_pi / n_phi);
    }
    const auto p = normalized_legendre_all(big_l, theta);
    for (int l = 0; l < big_l; ++l)
      for (int m = 0; m <= l; ++m)
        acc[static_cast<std::size_t>(l) * (l + 1) / 2 + m] += w * p[static_cast<std::size_t>(l) * (l + 1) / 2 + m] * f_m[m];
  }
  for (int l = 0; l < big_l; ++l) {
    out.values[HarmonicVector::index_mean(l)] = acc[static_cast<std::size_t>(l) * (l + 1) / 2].real();
    for (int m = 1; m <= l; ++m) {
      const auto z = acc[static_cast<std::size_t>(l) * (l + 1) / 2 + m];
      out.values[HarmonicVector::index_re(l, m)] = z.real();
      out.values[HarmonicVector::index_im(l, m)] = z.imag();
    }
  }
  return out;
}

// Surface integral of field^2 from ring transforms and I(q) only
// (sht.cpp:529-574); DFTs evaluated directly (a diagnostic, O(n^2) per ring).
inline double field_energy_quadrature(const EquiangularField& field) {
  const GridSpec& spec = field.spec;
  spec.validate();
  const int big_l = spec.max_band_limit(), n_theta = spec.n_theta, n_phi = spec.n_phi, n_ext = 2 * n_theta - 2;
  std::vector<std::complex<double>> in(n_phi), out(n_phi);
  std::vector<std::complex<double>> g(static_cast<std::size_t>(2 * big_l - 1) * n_theta);
  const int mid = big_l - 1;
  for (int i = 0; i < n_theta; ++i) {
    for (int j = 0; j < n_phi; ++j) in[j] = {field.values[static_cast<std::size_t>(i) * n_phi + j], 0.0};
    detail::naive_dft(in.data(), out.data(), n_phi);
    for (int c = 0; c < 2 * big_l - 1; ++c) {
      const int m = c - mid;
      g[static_cast<std::size_t>(c) * n_theta + i] = out[(m % n_phi + n_phi) % n_phi] / static_cast<double>(n_phi);
    }
  }
  std::vector<std::complex<double>> ext(n_ext), spec1(n_ext), kappa(2 * big_l - 1);
  double energy = 0.0;
  for (int c = 0; c < 2 * big_l - 1; ++c) {
    const int m = c - mid;
    const double par = (m & 1) ? -1.0 : 1.0;
    const std::complex<double>* gm = g.data() + static_cast<std::size_t>(c) * n_theta;
    for (int i = 0; i < n_theta; ++i) ext[i] = gm[i];
    for (int k = 1; k <= n_theta - 2; ++k) ext[n_theta - 1 + k] = par * gm[n_theta - 1 - k];
    detail::naive_dft(ext.data(), spec1.data(), n_ext);
    for (int cc = 0; cc < 2 * big_l - 1; ++cc) {
      const int mp = cc - mid;
      kappa[cc] = spec1[(mp % n_ext + n_ext) % n_ext] / static_cast<double>(n_ext);
    }
    std::complex<double> contrib{0.0, 0.0};
    for (int a = 0; a < 2 * big_l - 1; ++a)
      for (int b = 0; b < 2 * big_l - 1; ++b) contrib += kappa[a] * std::conj(kappa[b]) * i_integral(a - b);
    energy += contrib.real();
  }
  return 6.283185307179586476925286766559 * energy;
}

}  // namespace sphemu
