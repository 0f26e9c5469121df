// ref_wrap.cpp — extern "C" entry points over the reference's OWN code
// (proj/include/sphemu/{half,rng}.hpp, proj/src/{wigner,grid,sht}.cpp compiled
// from /root/reference by oracle/ref/build_ref.sh). Used only by tests/ to pin
// the oracle restatement and to write tests/golden/ fixtures.
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "sphemu/grid.hpp"
#include "sphemu/half.hpp"
#include "sphemu/rng.hpp"
#include "sphemu/sht.hpp"
#include "sphemu/wigner.hpp"

using namespace sphemu;

extern "C" {

double ref_quantize_half(double v, long long* sat) { return detail::quantize_half(v, sat); }
unsigned short ref_half_from_float(float v, long long* sat) { return detail::half_from_float(v, sat); }
float ref_half_to_float(unsigned short h) { return detail::half_to_float(h); }

void ref_rng_normals(std::uint64_t seed, std::int64_t n, double* out) {
  detail::GaussianRng rng(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = rng.normal();
}
void ref_rng_uniforms(std::uint64_t seed, std::int64_t n, double* out) {
  detail::GaussianRng rng(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = rng.uniform();
}

void ref_i_integral(long long q, double* re, double* im) {
  auto z = i_integral(q);
  *re = z.real();
  *im = z.imag();
}

// Dumps d^l_{m2,m} for 0<=l<L, -l<=m2,m<=l packed (l, m2+l, m+l) into out
// (size sum (2l+1)^2) and q(l,m,m2) for 0<=m<=l, 0<=m2<L into qout.
int ref_wigner_dump(int L, double* out, double* qout, int* renorm) {
  try {
    auto t = build_wigner_tables(L, std::size_t{1} << 62);
    std::size_t o = 0;
    for (int l = 0; l < L; ++l)
      for (int m2 = -l; m2 <= l; ++m2)
        for (int m = -l; m <= l; ++m) out[o++] = t->d_half_pi(l, m2, m);
    o = 0;
    for (int l = 0; l < L; ++l)
      for (int m = 0; m <= l; ++m)
        for (int m2 = 0; m2 < L; ++m2) qout[o++] = t->q(l, m, m2);
    *renorm = t->renormalization_warnings();
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_wigner_check_cap(int L, std::size_t cap) {
  try {
    (void)build_wigner_tables(L, cap);
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

double ref_wigner_brute(int l, int m2, int m) { return wigner_brute_force(l, m2, m); }

static int sht_batch(int n_theta, int n_phi, int L, const double* in, std::int64_t n, double* out,
                     bool forward, int threads) {
  try {
    GridSpec spec{n_theta, n_phi};
    ShtPlan plan = build_plan(spec, L);
    if (forward) {
      FieldSeries s(spec, static_cast<int>(n), 1);
      std::memcpy(s.values.data(), in, s.values.size() * sizeof(double));
      CoeffSeries c = forward_sht_batch(plan, s, threads);
      std::memcpy(out, c.values.data(), c.values.size() * sizeof(double));
    } else {
      CoeffSeries c(L, static_cast<int>(n), 1);
      std::memcpy(c.values.data(), in, c.values.size() * sizeof(double));
      FieldSeries s = inverse_sht_batch(plan, c, threads);
      std::memcpy(out, s.values.data(), s.values.size() * sizeof(double));
    }
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  }
}

int ref_forward_sht_batch(int n_theta, int n_phi, int L, const double* fields, std::int64_t n,
                          double* coeffs, int threads) {
  return sht_batch(n_theta, n_phi, L, fields, n, coeffs, true, threads);
}
int ref_inverse_sht_batch(int n_theta, int n_phi, int L, const double* coeffs, std::int64_t n,
                          double* fields, int threads) {
  return sht_batch(n_theta, n_phi, L, coeffs, n, fields, false, threads);
}

int ref_forward_sht_via_weights(int n_theta, int n_phi, int L, const double* field, double* coeffs) {
  GridSpec spec{n_theta, n_phi};
  ShtPlan plan = build_plan(spec, L);
  forward_sht_via_weights(plan, std::span<const double>(field, spec.points()),
                          std::span<double>(coeffs, static_cast<std::size_t>(L) * L));
  return 0;
}

void ref_draw_random_coefficients(int L, std::uint64_t seed, double* out) {
  HarmonicVector h = draw_random_coefficients(L, seed);
  std::memcpy(out, h.values.data(), h.values.size() * sizeof(double));
}

void ref_synth_bandlimited(const double* coeffs, int L, int n_theta, int n_phi, double* out) {
  HarmonicVector h(L);
  std::memcpy(h.values.data(), coeffs, h.values.size() * sizeof(double));
  EquiangularField f = synth_bandlimited(h, GridSpec{n_theta, n_phi});
  std::memcpy(out, f.values.data(), f.values.size() * sizeof(double));
}

void ref_normalized_legendre_all(int L, double theta, double* out) {
  auto p = normalized_legendre_all(L, theta);
  std::memcpy(out, p.data(), p.size() * sizeof(double));
}

double ref_field_energy_quadrature(const double* field, int n_theta, int n_phi) {
  EquiangularField f(GridSpec{n_theta, n_phi});
  std::memcpy(f.values.data(), field, f.values.size() * sizeof(double));
  return field_energy_quadrature(f);
}

int ref_max_band_limit(int n_theta, int n_phi) { return GridSpec{n_theta, n_phi}.max_band_limit(); }

}  // extern "C"
