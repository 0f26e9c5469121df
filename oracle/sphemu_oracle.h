/*
 * sphemu_oracle.h — CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load liboracle.so.
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Parity pinning: see oracle/README.md and DESIGN.md §3
 * — the oracle is pinned against (a) the known-answer tests of the reference's
 * own test suite and (b) oracle/_ref, the reference's wigner.cpp / grid.cpp /
 * sht.cpp / half.hpp / rng.hpp compiled from /root/reference with an exact-DFT
 * shim standing in for FFTW.
 */
#ifndef SPHEMU_ORACLE_H
#define SPHEMU_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------- rng.hpp:12-39 (mt19937_64 + explicit Box-Muller) ---------------- */
typedef struct {
  uint64_t mt[312];
  int mti;
  double spare;
  int has_spare;
} so_rng;

void so_rng_seed(so_rng* r, uint64_t seed);
uint64_t so_rng_raw(so_rng* r);
double so_rng_uniform(so_rng* r);
double so_rng_normal(so_rng* r);
/* Fill out[0..n) with successive normal() draws of GaussianRng(seed). */
void so_rng_normals(uint64_t seed, int64_t n, double* out);

/* ---------------- half.hpp:13-85 (binary16 RNE with saturation) ---------------- */
uint16_t so_half_from_float(float v, long long* saturations);
float so_half_to_float(uint16_t h);
double so_quantize_half(double v, long long* saturations);
double so_quantize_single(double v);
/* BF16 storage class (extension; no reference oracle, F2): float RNE to bf16,
 * saturating to +-max finite bf16 like the half path saturates. */
double so_quantize_bf16(double v, long long* saturations);

/* ---------------- mpchol.hpp / mpchol.cpp ---------------- */
enum { SO_DP = 0, SO_SP = 1, SO_HP = 2 };                     /* mpchol.hpp:11 */
enum { SO_V_DP = 0, SO_V_DPSP = 1, SO_V_DPSPHP = 2, SO_V_DPHP = 3 }; /* mpchol.hpp:12 */
enum { SO_HP_FP16 = 0, SO_HP_BF16 = 1 };

typedef struct {
  int variant;         /* mpchol.hpp:19 */
  int tile_size;       /* mpchol.hpp:20 (default 128) */
  int band_width_dp;   /* mpchol.hpp:22 (default 1) */
  double sp_fraction;  /* mpchol.hpp:24 (default 0.05) */
  int workers;         /* mpchol.hpp:25 */
  int hp_format;       /* extension: SO_HP_FP16 (reference) or SO_HP_BF16 */
} so_chol_config;

typedef struct {
  int64_t demotions_sp, demotions_hp, half_saturations; /* mpchol.hpp:95-99 */
} so_counters;

typedef struct {
  int n, tile_size, n_tiles, workers, variant;
  int64_t tasks_potrf, tasks_trsm, tasks_syrk, tasks_gemm;
  int64_t tiles_dp, tiles_sp, tiles_hp;
  int64_t bytes_dp, bytes_sp, bytes_hp;
  so_counters conv;
  double wall_seconds;
} so_chol_stats;

/* Returns 0 ok, -1 invalid config (mpchol.cpp:55-61). */
int so_config_validate(const so_chol_config* c);
/* mpchol.cpp:67-93: out[i*(i+1)/2 + j] = precision of tile (i, j). */
int so_assign_precisions(int n_tiles, const so_chol_config* c, uint8_t* out);

/* mpchol.cpp:156-205. Task arrays of length so_task_count(nt). kinds 0..3 =
 * potrf, trsm, syrk, gemm (mpchol.hpp:73). Successors as CSR (succ_off has
 * count+1 entries, succ has edge_count entries). */
int64_t so_task_count(int n_tiles);
int64_t so_task_graph(int n_tiles, uint8_t* kind, int32_t* ti, int32_t* tj, int32_t* tk,
                      int64_t* succ_off, int32_t* succ, int32_t* indegree, int64_t succ_cap);

/* mpchol.cpp:207-225 (HP through fp16, or bf16 when hp_format == SO_HP_BF16). */
void so_quantize_tile(double* tile, int64_t n, int prec, int hp_format, so_counters* c);

/* Packed tile layout (mpchol.cpp:95-154): tiles (i,j), j<=i, packed by
 * i(i+1)/2+j, each row-major with tile_rows(i) x tile_rows(j) doubles. */
int64_t so_tiled_size(int n, int b);
void so_tiled_from_dense(const double* a, int n, int b, double* tiles);
void so_tiled_to_dense_lower(const double* tiles, int n, int b, double* a);

/* mpchol.cpp:351-410: in-place tiled factorization with the DAG scheduler.
 * Returns 0 ok, 1 not positive definite (failed_tile set), -1 bad config. */
int so_tiled_cholesky(double* tiles, int n, const so_chol_config* c, so_chol_stats* st,
                      int* failed_tile);
/* mpchol.cpp:412-417 */
int so_tiled_cholesky_dense_map(const double* a, int n, const so_chol_config* c, const uint8_t* map,
                                double* factor, so_chol_stats* st, int* failed_tile);
int so_tiled_cholesky_dense(const double* a, int n, const so_chol_config* c, double* factor,
                            so_chol_stats* st, int* failed_tile);
/* mpchol.cpp:419-435 */
void so_make_spd(int n, uint64_t seed, double* a);
/* The per-row scale d_i of make_spd_test_matrix and pw[k] = pow(0.9, k). */
void so_make_spd_factors(int n, uint64_t seed, double* d, double* pw);

/* tests/support/reference.cpp:10-44 */
int so_dense_cholesky(const double* a, int n, double* l);
double so_relative_residual(const double* a, const double* l, int n, int threads);

/* Optional OpenBLAS stand-in for Eigen's tile kernels (cpu-baseline timing
 * only). Returns 0 when loaded. */
int so_use_blas(const char* path);

/* ---------------- sht.hpp / sht.cpp / wigner.cpp / fft.cpp ---------------- */
/* Complex DFT, sign -1 analysis, +1 unnormalized synthesis (fft.hpp:12-29). */
void so_dft(int n, int sign, const double* in_ri, double* out_ri);

/* sht.cpp:30-37 */
void so_i_integral(long long q, double* re, double* im);

typedef struct so_wigner so_wigner;
/* wigner.cpp:49-134 (cap as wigner.hpp:48-49; returns NULL over cap). */
so_wigner* so_wigner_build(int band_limit, size_t cap_bytes);
void so_wigner_free(so_wigner* w);
double so_wigner_d(const so_wigner* w, int l, int m2, int m);   /* wigner.cpp:136-150 */
double so_wigner_q(const so_wigner* w, int l, int m, int m2);   /* wigner.cpp:165-170 */
int so_wigner_renorm_warnings(const so_wigner* w);
size_t so_wigner_bytes(int band_limit);                          /* wigner.cpp:54-60 */
double so_wigner_brute(int l, int m2, int m);                    /* wigner.cpp:31-47 */
const double* so_wigner_q_table(const so_wigner* w);            /* rows (l,m), L cols */

typedef struct so_plan so_plan;
/* sht.cpp:111-171 minus the w1/w2 tables (only the via-weights test path uses them). */
so_plan* so_plan_build(int n_theta, int n_phi, int band_limit, const so_wigner* tables);
void so_plan_free(so_plan* p);
int so_plan_points(const so_plan* p);
int so_grid_max_band_limit(int n_theta, int n_phi);             /* grid.cpp:27-29 */
/* sht.cpp:226-263 / 304-357 (single slice) */
void so_forward_sht(const so_plan* p, const double* field, double* coeffs);
void so_inverse_sht(const so_plan* p, const double* coeffs, double* field);
/* sht.cpp:374-404 with the parallel_for partition of thread_pool.hpp:17-43 */
void so_forward_sht_batch(const so_plan* p, const double* fields, int64_t n, double* coeffs,
                          int threads);
void so_inverse_sht_batch(const so_plan* p, const double* coeffs, int64_t n, double* fields,
                          int threads);
/* sht.cpp:406-427 */
void so_normalized_legendre_all(int band_limit, double theta, double* p);
/* sht.cpp:435-466 */
void so_synth_bandlimited(const double* coeffs, int band_limit, int n_theta, int n_phi,
                          double* field);
/* sht.cpp:507-518 */
void so_draw_random_coefficients(int band_limit, uint64_t seed, double* out);
/* sht.cpp:529-574 */
double so_field_energy_quadrature(const double* field, int n_theta, int n_phi);
/* sht.cpp:58-69 */
double so_parseval_energy(const double* coeffs, int band_limit);

/* ---------------- stochastic.cpp ---------------- */
/* stochastic.cpp:109-172: u_hat (d x d row-major) and factor v (dense lower).
 * Returns 0 ok, 2 gave up (nugget over cap), -2 non-positive mean diagonal. */
int so_estimate_innovation_covariance(const double* resid, int64_t n_rows, int d,
                                      const so_chol_config* c, int threads, double* u_hat,
                                      double* v, double* nugget, so_chol_stats* st);
/* stochastic.cpp:217-277, trend evaluated by the caller into means
 * (t_out x points, trend.cpp:252-287) and sigma (points). v is dense d x d
 * (lower factor, zeros included, as the reference multiplies it). phi is
 * order x d. out is (r_len, t_out, points). */
int so_emulate(const so_plan* p, const double* v, int d, const double* phi, int order,
               const double* means, const double* sigma, const double* v2, int t_out,
               uint64_t seed, int r_len, int threads, double* out);

/* ---------------- trend.cpp:18-57,59-83,252-324 (mean structure) ----------------
 * records: points x (5 + 2K) TrendModel::values; forcing {x[n_x], history[n_h]}
 * (n_x = n_h = 0: empty trajectory). Return 0, or -1 for t_start < 1,
 * -2 for a missing lag history (require_lag_history, trend.cpp:21-25). */
double so_eval_mean_trend(const double* records, int harmonics, int period, int64_t loc, int64_t t,
                          const double* fx, int64_t n_x, const double* fh, int64_t n_h, int* err);
int so_mean_table(const double* records, int64_t points, int harmonics, int period,
                  const double* fx, int64_t n_x, const double* fh, int64_t n_h,
                  int t_len, int64_t t_start, double* table);
/* mode 0: detrend (y - m) / sigma (trend.cpp:289-305); 1: retrend m + sigma z
 * (trend.cpp:307-324). in/out are (r_len, t_len, points). */
int so_trend_apply(int mode, const double* in, int r_len, int t_len, const double* records, int64_t points,
                   int harmonics, int period, const double* fx, int64_t n_x, const double* fh, int64_t n_h,
                   int64_t t_start, double* out);

#ifdef __cplusplus
}
#endif
#endif
