// C++ drop-in API checks (include/sphemu/*.hpp over the C-ABI), mirroring the
// reference's own test cases: proj/tests/test_mpchol.cpp, test_sht.cpp,
// test_grid.cpp, test_wigner.cpp, test_stochastic.cpp (file:line in each case).
// Prints "ALL PASSED" and exits 0 when every check holds. Needs a GPU.
#include <cmath>
#include <cstdio>
#include <numbers>
#include <random>
#include <string>
#include <vector>

#include "sphemu/sphemu.hpp"

static int g_fail = 0;
#define CHECK(cond)                                                       \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
      ++g_fail;                                                           \
    }                                                                     \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// Unblocked host Cholesky (the untiled oracle of tests/support/reference.cpp).
static std::vector<double> host_cholesky(std::vector<double> a, int n) {
  for (int j = 0; j < n; ++j) {
    double s = a[j * n + j];
    for (int k = 0; k < j; ++k) s -= a[j * n + k] * a[j * n + k];
    a[j * n + j] = std::sqrt(s);
    for (int i = j + 1; i < n; ++i) {
      double t = a[i * n + j];
      for (int k = 0; k < j; ++k) t -= a[i * n + k] * a[j * n + k];
      a[i * n + j] = t / a[j * n + j];
    }
    for (int c = j + 1; c < n; ++c) a[j * n + c] = 0.0;
  }
  return a;
}

int main() {
  using namespace sphemu;
  CHECK(std::string(kVersion) == "0.1.0");

  // grid.cpp:18-49 (test_grid.cpp)
  GridSpec g = GridSpec::from_band_limit(45);
  CHECK(g.n_theta == 46 && g.n_phi == 90 && g.max_band_limit() == 45 && g.admissible(45) && !g.admissible(46));
  CHECK(std::fabs(g.theta(45) - std::numbers::pi) < 1e-15);
  CHECK(resolution_summary(180).grid_points == 179 * 360);
  CHECK(throws<std::invalid_argument>([] { GridSpec{1, 4}.validate(); }));

  // quantize KATs (test_mpchol.cpp:177-202)
  {
    std::vector<double> t{1.0 / 3.0};
    ConversionCounters cc;
    quantize_tile(t, Precision::kSingle, &cc);
    CHECK(t[0] == static_cast<double>(1.0f / 3.0f) && cc.demotions_sp == 1);
    std::vector<double> h{1.0 / 3.0, 65505.0, -70000.0};
    ConversionCounters ch;
    quantize_tile(h, Precision::kHalf, &ch);
    CHECK(h[0] == 0.333251953125 && h[1] == 65504.0 && h[2] == -65504.0);
    CHECK(ch.half_saturations == 1 && ch.demotions_hp == 3);
  }

  // DAG (test_mpchol.cpp:47-71)
  for (auto [nt, want] : {std::pair{4, 20}, std::pair{8, 120}}) {
    TaskGraph dag = build_task_graph(nt);
    int sources = 0;
    for (auto d : dag.indegree) sources += d == 0;
    CHECK(static_cast<int>(dag.size()) == want && sources == 1);
  }

  // precision map (test_mpchol.cpp:73-108)
  {
    MpCholConfig c;
    c.variant = PrecisionVariant::kDpSpHp;
    PrecisionMap m = assign_precisions(10, c);
    CHECK(m.count(Precision::kDouble) == 10 && m.count(Precision::kSingle) == 3);
    CHECK(m.at(1, 0) == Precision::kSingle && m.at(2, 1) == Precision::kSingle && m.at(3, 2) == Precision::kSingle);
    c.band_width_dp = 2;
    CHECK(assign_precisions(10, c).count(Precision::kDouble) == 19);
  }

  // 2x2 known answer at b = 1 and 2 (test_mpchol.cpp:36-45)
  for (int b : {1, 2}) {
    MpCholConfig c;
    c.tile_size = b;
    c.compute = SPHEMU_COMPUTE_FP64;
    auto r = tiled_cholesky_dense(std::vector<double>{4, 2, 2, 3}, 2, c);
    CHECK(r.factor[0] == 2.0 && r.factor[1] == 0.0 && r.factor[2] == 1.0 && r.factor[3] == std::sqrt(2.0));
  }

  // DP factor vs the untiled oracle, n in {96, 100}, b = 32, seed 3 (test_mpchol.cpp:110-121)
  for (int n : {96, 100}) {
    std::vector<double> a = make_spd_test_matrix(n, 3);
    CHECK(a[1] == a[n]);  // exactly symmetric
    MpCholConfig c;
    c.tile_size = 32;
    auto r = tiled_cholesky_dense(a, n, c);
    auto want = host_cholesky(a, n);
    double md = 0.0;
    for (std::size_t e = 0; e < want.size(); ++e) md = std::fmax(md, std::fabs(r.factor[e] - want[e]));
    CHECK(md < 1e-13);
    CHECK(r.stats.n_tiles == (n + 31) / 32 && r.stats.tasks_potrf == r.stats.n_tiles);
    // in-place TiledMatrix path gives the same factor
    TiledMatrix t = TiledMatrix::from_dense(a, n, 32);
    tiled_cholesky(t, c);
    CHECK(t.to_dense_lower() == r.factor);
  }

  // indefinite input -> NotPositiveDefiniteError on tile 1 (test_mpchol.cpp:142-154)
  {
    std::vector<double> a(16, 0.0);
    a[0] = a[5] = a[15] = 1.0;
    a[10] = -1.0;
    MpCholConfig c;
    c.tile_size = 2;
    int tile = -2;
    try {
      tiled_cholesky_dense(a, 4, c);
    } catch (const NotPositiveDefiniteError& e) {
      tile = e.tile_index();
    }
    CHECK(tile == 1);
  }

  // stats JSON schema (mpchol.cpp:437-457)
  {
    MpCholConfig c;
    c.variant = PrecisionVariant::kDpSp;
    c.tile_size = 32;
    auto r = tiled_cholesky_dense(make_spd_test_matrix(64, 1), 64, c);
    const std::string js = r.stats.to_json();
    CHECK(js.find("\"variant\": \"dpsp\"") != std::string::npos && js.find("\"total\": 4,") != std::string::npos);
  }

  // SHT: constant field (test_sht.cpp:72-83) and round trip (test_sht.cpp:85-102)
  {
    ShtPlan p = build_plan(GridSpec::from_band_limit(16), 16);
    EquiangularField f(p.spec);
    for (auto& v : f.values) v = 2.5;
    HarmonicVector z = forward_sht(p, f);
    CHECK(std::fabs(z.values[0] - 2.5 * std::sqrt(4.0 * std::numbers::pi)) < 1e-13);
    std::mt19937_64 rng(7);
    std::normal_distribution<double> nd;
    HarmonicVector c(16);
    for (int l = 0; l < 16; ++l) {
      c.set_coeff(l, 0, {nd(rng), 0.0});
      for (int m = 1; m <= l; ++m) c.set_coeff(l, m, {nd(rng), nd(rng)});
    }
    HarmonicVector back = forward_sht(p, inverse_sht(p, c));
    double md = 0.0;
    for (std::size_t e = 0; e < c.values.size(); ++e) md = std::fmax(md, std::fabs(back.values[e] - c.values[e]));
    CHECK(md < 1e-10);
    CHECK(std::fabs(c.parseval_energy() - back.parseval_energy()) < 1e-8 * c.parseval_energy());
    // batch == single
    FieldSeries s(p.spec, 3, 2);
    for (std::size_t e = 0; e < s.values.size(); ++e) s.values[e] = std::sin(0.001 * e);
    CoeffSeries cs = forward_sht_batch(p, s, 4);
    std::vector<double> one(HarmonicVector::packed_size(16));
    forward_sht(p, s.slice(1, 2), one);
    double bd = 0.0;
    for (std::size_t e = 0; e < one.size(); ++e) bd = std::fmax(bd, std::fabs(one[e] - cs.slice(1, 2)[e]));
    CHECK(bd < 1e-14);
    // direct synthesis agrees with the plan on a resolved grid (test_sht.cpp:145-152)
    EquiangularField via_plan = inverse_sht(p, c), direct = synth_bandlimited(c, p.spec);
    double sd = 0.0;
    for (std::size_t e = 0; e < direct.values.size(); ++e)
      sd = std::fmax(sd, std::fabs(via_plan.values[e] - direct.values[e]));
    CHECK(sd < 1e-9);
    CHECK(synth_bandlimited(c, GridSpec{9, 16}).values.size() == 9 * 16);  // under-resolved target
  }
  CHECK(throws<std::invalid_argument>([] { build_plan(GridSpec{9, 16}, 9); }));           // test_sht.cpp:196-199
  CHECK(throws<std::invalid_argument>([] { build_wigner_tables(720); }));                 // 2 GiB cap (F5)
  CHECK(!throws<std::invalid_argument>([] { build_wigner_tables(720, std::size_t{4} << 30); }));
  {  // test_wigner.cpp:23-31 closed forms, read from the device-built tables
    auto w = build_wigner_tables(8);
    CHECK(std::fabs(w->d_half_pi(1, 0, 0)) < 1e-15);
    CHECK(std::fabs(w->d_half_pi(1, 1, 1) - 0.5) < 1e-15);
    CHECK(std::fabs(w->d_half_pi(1, 1, 0) + std::sqrt(0.5)) < 1e-15);
    CHECK(std::fabs(w->d_half_pi(2, 0, 0) + 0.5) < 1e-15);
    CHECK(w->d_half_pi(3, 4, 0) == 0.0);
    CHECK(throws<std::out_of_range>([&] { w->d_half_pi(8, 0, 0); }));
  }
  // test_wigner.cpp:23-31 factorial sums
  CHECK(std::fabs(wigner_brute_force(1, 1, -1) - 0.5) < 1e-14);
  CHECK(std::fabs(wigner_brute_force(2, 2, 0) - std::sqrt(3.0 / 8.0)) < 1e-14);
  {  // test_wigner.cpp:33-43 recursion vs factorial sum, l <= 12
    auto t = build_wigner_tables(13);
    double worst = 0.0;
    for (int l = 0; l <= 12; ++l)
      for (int m2 = -l; m2 <= l; ++m2)
        for (int m = -l; m <= l; ++m)
          worst = std::fmax(worst, std::fabs(t->d_half_pi(l, m2, m) - wigner_brute_force(l, m2, m)));
    CHECK(worst < 1e-12);
  }
  {  // test_wigner.cpp:45-59 orthonormal rows, no renormalization
    auto t = build_wigner_tables(32);
    CHECK(t->renormalization_warnings() == 0);
    double worst = 0.0;
    for (int l = 0; l < 32; ++l)
      for (int m = 0; m <= l; ++m)
        for (int mp = m; mp <= l; ++mp) {
          double dot = 0.0;
          for (int m2 = -l; m2 <= l; ++m2) dot += t->d_half_pi(l, m2, m) * t->d_half_pi(l, m2, mp);
          worst = std::fmax(worst, std::fabs(dot - (m == mp ? 1.0 : 0.0)));
        }
    CHECK(worst < 1e-10);
  }
  {  // test_wigner.cpp:61-73 synthesis products, sizes
    auto t = build_wigner_tables(4);
    CHECK(std::fabs(t->q(0, 0, 0) - 0.2820947917738781) < 1e-15);
    CHECK(std::fabs(t->q(1, 0, 1) - std::sqrt(3.0 / (4.0 * std::numbers::pi)) * 0.5) < 1e-15);
    CHECK(t->q(1, 1, 3) == 0.0);
    CHECK(t->q_entry_count() == 4u * 4u * 5u / 2u);
    CHECK(t->memory_bytes() == WignerTables::estimated_bytes(4));
    CHECK(throws<std::out_of_range>([&] { t->q(4, 0, 0); }));
  }
  {  // test_wigner.cpp:75-104 WIGD cache round trip, load_or_build
    auto built = build_wigner_tables(10);
    const std::string path = "/tmp/sphemu_cpp_tables.wigd";
    write_wigd(path, *built);
    auto loaded = read_wigd(path);
    CHECK(loaded->band_limit() == 10 && loaded->renormalization_warnings() == built->renormalization_warnings());
    bool same = true;
    for (int l = 0; l < 10; ++l)
      for (int m2 = -l; m2 <= l; ++m2)
        for (int m = 0; m <= l; ++m) same &= loaded->d_half_pi(l, m2, m) == built->d_half_pi(l, m2, m);
    for (int l = 0; l < 10; ++l)
      for (int m = 0; m <= l; ++m)
        for (int m2 = 0; m2 <= l; ++m2) same &= loaded->q(l, m, m2) == built->q(l, m, m2);
    CHECK(same);
    std::remove("/tmp/sphemu_cpp_cache.wigd");
    auto first = load_or_build_wigner(6, "/tmp/sphemu_cpp_cache.wigd");
    auto second = load_or_build_wigner(6, "/tmp/sphemu_cpp_cache.wigd");
    CHECK(second->band_limit() == 6 && second->d_half_pi(5, 3, 2) == first->d_half_pi(5, 3, 2));
    auto third = load_or_build_wigner(7, "/tmp/sphemu_cpp_cache.wigd");  // mismatched band limit: rebuilt
    CHECK(third->band_limit() == 7);
  }
  // test_sht.cpp:51-59 I(q) known answers
  CHECK(i_integral(0).real() == 2.0 && i_integral(2).real() == 2.0 / (1.0 - 4.0));
  CHECK(i_integral(1).imag() == std::numbers::pi / 2.0 && i_integral(-1).imag() == -std::numbers::pi / 2.0);
  CHECK(i_integral(3) == std::complex<double>(0.0, 0.0));
  {  // generators (sht.cpp:406-527): Legendre vs the plan, random fields, energy quadrature
    CHECK(std::fabs(normalized_legendre(0, 0, 0.3) - 1.0 / std::sqrt(4.0 * std::numbers::pi)) < 1e-15);
    CHECK(throws<std::out_of_range>([] { normalized_legendre(2, 3, 0.1); }));
    HarmonicVector c1 = draw_random_coefficients(8, 5), c2 = draw_random_coefficients(8, 5);
    CHECK(c1.values == c2.values && c1.values != draw_random_coefficients(8, 6).values);
    ShtPlan p8 = build_plan(GridSpec{17, 32}, 8);
    EquiangularField f = synth_random_field(p8, 5);
    EquiangularField direct = synth_bandlimited(c1, p8.spec);
    double md = 0.0;
    for (std::size_t e = 0; e < f.values.size(); ++e) md = std::fmax(md, std::fabs(f.values[e] - direct.values[e]));
    CHECK(md < 1e-10);
    CHECK(synth_random_field(GridSpec{17, 32}, 8, 5).values == f.values);
    // Parseval (test_sht.cpp:135-143): energy quadrature = sum |f_lm|^2 for a band-limited field
    CHECK(std::fabs(field_energy_quadrature(f) - c1.parseval_energy()) < 1e-8 * c1.parseval_energy());
    // quadrature oracle (test_sht.cpp:104-110): a single Y_{2,1} pattern is recovered
    HarmonicVector q = quadrature_oracle_sht(
        [](double th, double ph) { return std::sin(th) * std::cos(th) * std::cos(ph); }, 4, 4001);
    CHECK(std::fabs(q.values[HarmonicVector::index_mean(2)]) < 1e-6);
    CHECK(std::fabs(q.values[HarmonicVector::index_im(2, 1)]) < 1e-6 && std::fabs(q.values[HarmonicVector::index_re(2, 1)]) > 0.1);
  }

  {  // train -> emulate (pipeline.cpp:18-54, stochastic.cpp:217-277) through the C++ API, factor kept on the device
    const int L = 6, t_len = 120, r_len = 2;
    GridSpec spec = GridSpec::from_band_limit(L);
    ShtPlan p = build_plan(spec, L);
    FieldSeries series(spec, t_len, r_len);
    std::mt19937_64 rng(91);
    std::normal_distribution<double> nd;
    for (int r = 0; r < r_len; ++r) {
      std::vector<double> state(L * L, 0.0);
      for (int t = 0; t < t_len; ++t) {
        HarmonicVector c(L);
        for (int i = 0; i < L * L; ++i) c.values[i] = state[i] = 0.55 * state[i] + 0.3 * nd(rng);
        EquiangularField f = inverse_sht(p, c);
        auto sl = series.slice(r, t);
        for (std::size_t loc = 0; loc < sl.size(); ++loc)
          sl[loc] = 1.7 + 1.1 * std::cos(2.0 * std::numbers::pi * (t + 1) / 12.0) + f.values[loc] + 0.05 * nd(rng);
      }
    }
    TrainConfig tc;
    tc.band_limit = L;
    tc.trend.harmonics = 2;
    tc.trend.period = 12;
    tc.var_order = 2;
    tc.chol.tile_size = 16;
    EmulatorModel m = train(series, {}, tc);
    CHECK(m.innovation.factor != nullptr && m.innovation.v.size() == 36u * 36u && m.noise.v2.size() == spec.points());
    CHECK(std::fabs(m.trend.values[0] - 1.7) < 0.2);  // intercept of the seasonal series
    FieldSeries a = emulate(m, p, {}, 8, 42, 2);
    FieldSeries b2 = emulate(p, m.innovation.v, 36, m.var.phi, m.var.order, m.trend, ForcingTrajectory{}, m.noise.v2, 8,
                             42, 2);
    double md = 0.0, mx = 0.0;
    for (std::size_t e = 0; e < a.values.size(); ++e) {
      md = std::fmax(md, std::fabs(a.values[e] - b2.values[e]));
      mx = std::fmax(mx, std::fabs(b2.values[e]));
    }
    CHECK(md <= 1e-10 * mx);  // the tiled (dp) factor path = the dense-V path
    CHECK(throws<std::invalid_argument>([&] { fit_trend(series, ForcingTrajectory{{1.0, 2.0}, {}}, tc.trend); }));
  }

  // covariance + nugget (test_stochastic.cpp:159-210)
  {
    const int d = 36, r_len = 2, t_len = 40, order = 2;
    const std::int64_t rows = r_len * (t_len - order);
    std::vector<double> xi(static_cast<std::size_t>(rows) * d);
    std::mt19937_64 rng(99);
    std::normal_distribution<double> nd;
    for (auto& x : xi) x = nd(rng);
    MpCholConfig c;
    c.tile_size = 16;
    InnovationModel m = estimate_innovation_covariance(xi, rows, d, r_len, t_len, order, c);
    double mu = 0.0, mv = 0.0, mx = 0.0;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) {
        double u = 0.0, vv = 0.0;
        for (std::int64_t r = 0; r < rows; ++r) u += xi[r * d + i] * xi[r * d + j];
        u /= static_cast<double>(rows);
        for (int k = 0; k < d; ++k) vv += m.v[i * d + k] * m.v[j * d + k];
        mu = std::fmax(mu, std::fabs(u - m.u_hat[i * d + j]));
        mv = std::fmax(mv, std::fabs(vv - m.u_hat[i * d + j] - (i == j ? m.nugget : 0.0)));
        mx = std::fmax(mx, std::fabs(u));
      }
    CHECK(mu < 1e-12 * mx && mv < 1e-12 * mx && m.nugget == 0.0);
  }

  // fit_var: silent and explosive series (test_stochastic.cpp:144-157)
  {
    CoeffSeries coeffs(2, 400, 1);
    for (int t = 0; t < 400; ++t) coeffs.slice(0, t)[0] = static_cast<double>(t + 1);
    VarFit fit = fit_var(coeffs, 1);
    CHECK(fit.model.zeroed_count == 3 && fit.model.unstable_count == 1);
    CHECK(fit.model.phi_at(1, 0) > 1.0 && fit.model.phi_at(1, 1) == 0.0);
    CHECK(fit.residual_rows == 399);
    CHECK(throws<std::invalid_argument>([&] { fit_var(coeffs, 400); }));
  }

  // trend mean structure (test_trend.cpp:165-206)
  {
    TrendModel m;
    m.spec = GridSpec{3, 4};
    m.config.harmonics = 1;
    m.config.period = 12;
    m.config.validate();
    const std::size_t pts = m.spec.points();
    for (std::size_t loc = 0; loc < pts; ++loc) {
      const double rec[7] = {1.0 + 0.1 * loc, 0.0, 0.0, 0.6, 0.5, -0.25, 0.5 + 0.05 * loc};
      m.values.insert(m.values.end(), rec, rec + 7);
    }
    auto table = mean_table(m, {}, 24, 12);  // t = 12: base 0 -> beta0 + a_1
    CHECK(table.size() == 24 * pts && table[0] == m.values[0] + 0.5);
    FieldSeries y(m.spec, 24, 2);
    for (std::size_t i = 0; i < y.values.size(); ++i) y.values[i] = std::sin(0.1 * i);
    FieldSeries back = retrend(detrend(y, m, {}), m, {});
    double worst = 0.0;
    for (std::size_t i = 0; i < y.values.size(); ++i) worst = std::fmax(worst, std::fabs(back.values[i] - y.values[i]));
    CHECK(worst < 1e-12);
    CHECK(throws<std::invalid_argument>([&] { mean_table(m, {}, 4, 0); }));
    CHECK(throws<std::invalid_argument>([] { TrendConfig{2, 13}.validate(); }));
  }

  if (g_fail == 0) std::printf("ALL PASSED\n");
  return g_fail ? 1 : 0;
}
