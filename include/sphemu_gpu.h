/*
 * sphemu_gpu.h — C-ABI of the B200-native sphemu hot path.
 *
 * The reference (proj/, CPU-only C++20) has no C-ABI; its drop-in boundary is
 * the C++ API of mpchol.hpp / sht.hpp / wigner.hpp / stochastic.hpp and the
 * pybind11 module of bindings/module.cpp. Every entry point below names the
 * reference interface it replaces. Plain pointers and sizes only; no C++
 * exceptions or torch types cross this boundary. Status codes are returned;
 * sphemu_gpu_last_error() describes the last failure on the calling thread.
 *
 * Pointer kinds: functions taking a `where` argument accept host memory
 * (SPHEMU_HOST) or device memory on the current device (SPHEMU_DEVICE).
 */
#ifndef SPHEMU_GPU_H
#define SPHEMU_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---- */
#define SPHEMU_OK 0
#define SPHEMU_ERR_INVALID_ARG 1  /* std::invalid_argument in the reference */
#define SPHEMU_ERR_NOT_SPD 2      /* NotPositiveDefiniteError (mpchol.hpp:122-130) */
#define SPHEMU_ERR_CUDA 3
#define SPHEMU_ERR_NCCL 4
#define SPHEMU_ERR_OOM 5
#define SPHEMU_ERR_RUNTIME 6      /* std::runtime_error in the reference */

#define SPHEMU_HOST 0
#define SPHEMU_DEVICE 1

const char* sphemu_gpu_last_error(void);
const char* sphemu_gpu_version(void); /* "0.1.0" like proj/include/sphemu/version.hpp:4 */
int sphemu_gpu_device_count(void);
int sphemu_gpu_set_device(int device);
/* Number of kernel launches this process issued from the library (evidence
 * for bench.py's gpu_launches). */
int64_t sphemu_gpu_launch_count(void);

/* ======================================================================
 * Mixed-precision tiled Cholesky (replaces mpchol.hpp:18-148)
 * ====================================================================== */
#define SPHEMU_VARIANT_DP 0     /* PrecisionVariant::kDp     (mpchol.hpp:12) */
#define SPHEMU_VARIANT_DPSP 1   /* PrecisionVariant::kDpSp   */
#define SPHEMU_VARIANT_DPSPHP 2 /* PrecisionVariant::kDpSpHp */
#define SPHEMU_VARIANT_DPHP 3   /* PrecisionVariant::kDpHp   */

#define SPHEMU_PREC_DP 0 /* Precision::kDouble (mpchol.hpp:11) */
#define SPHEMU_PREC_SP 1 /* Precision::kSingle */
#define SPHEMU_PREC_HP 2 /* Precision::kHalf   */

#define SPHEMU_HP_FP16 0 /* IEEE binary16, saturating (half.hpp) — reference */
#define SPHEMU_HP_BF16 1 /* bfloat16 storage class — extension   */

#define SPHEMU_COMPUTE_TENSOR 0 /* per-class tensor cores: tcgen05 fp16/bf16, 3xTF32, FP64 DMMA */
#define SPHEMU_COMPUTE_FP64 1   /* every tile kernel in FP64 (mpchol.cpp:283-316 semantics) */

#define SPHEMU_SP_F16X3 0  /* SP-class updates: fp16 hi+lo split of row-scaled operands, kind::f16 */
#define SPHEMU_SP_TF32X3 1 /* SP-class updates: 3xTF32 on kind::tf32 */
#define SPHEMU_SP_FP64 2   /* SP-class panel + updates in FP64 DMMA: the oracle's arithmetic (mpchol.cpp:283-316)
                              on SP tiles, tensor cores for the HP class only */

/* MpCholConfig (mpchol.hpp:18-28) plus appended GPU fields whose zero values
 * keep reference behaviour. */
typedef struct {
  int variant;        /* SPHEMU_VARIANT_* */
  int tile_size;      /* default 128 */
  int band_width_dp;  /* default 1 */
  double sp_fraction; /* default 0.05 */
  int workers;        /* accepted for API parity; the GPU scheduler uses streams */
  int hp_format;      /* SPHEMU_HP_* */
  int compute;        /* SPHEMU_COMPUTE_* */
  int lookahead;      /* 0 = off, 1 = panel k+1 on a priority stream */
  int sp_compute;     /* SPHEMU_SP_* (tensor mode only) */
} sphemu_chol_config;

/* FactorizationStats (mpchol.hpp:104-120) + GPU timing. */
typedef struct {
  int n, tile_size, n_tiles, workers, variant;
  int64_t tasks_potrf, tasks_trsm, tasks_syrk, tasks_gemm;
  int64_t tiles_dp, tiles_sp, tiles_hp;
  int64_t bytes_dp, bytes_sp, bytes_hp;
  int64_t demotions_sp, demotions_hp, half_saturations;
  double wall_seconds;
  double device_ms;   /* factorization time on the device (CUDA events) */
  int64_t launches;   /* kernels launched by this factorization */
} sphemu_chol_stats;

/* MpCholConfig::validate (mpchol.cpp:55-61). */
int sphemu_gpu_chol_config_validate(const sphemu_chol_config* cfg);
/* assign_precisions (mpchol.cpp:67-93): out has n_tiles*(n_tiles+1)/2 bytes. */
int sphemu_gpu_assign_precisions(int n_tiles, const sphemu_chol_config* cfg, uint8_t* out);

/* tiled_cholesky_dense (mpchol.cpp:412-417): dense row-major n x n in, dense
 * lower factor (exact zeros above the diagonal) out. Host or device pointers.
 * On SPHEMU_ERR_NOT_SPD *failed_tile holds the diagonal tile index. */
int sphemu_gpu_tiled_cholesky_dense(const double* a, int where_a, int n,
                                    const sphemu_chol_config* cfg, double* factor,
                                    int where_factor, sphemu_chol_stats* stats, int* failed_tile);

/* The one-shot call keeps its device buffers cached for the next call with
 * the same n, configuration and device; this frees them. */
int sphemu_gpu_release_cache(void);

/* Host-only view of the 2D block-cyclic layout a rank would use (no GPU
 * needed): tiles it stores, its arena bytes, and xchg_bytes[k*P*Q + r] = the
 * panel bytes rank r receives at step k (nt*P*Q entries, may be NULL): each
 * panel tile (i, k) travels point to point from its owner to the owners of
 * row i and column i only. */
int sphemu_gpu_dist_layout(int n, const sphemu_chol_config* cfg, int P, int Q, int rank, int64_t* tiles_owned,
                           int64_t* arena_bytes, int64_t* xchg_bytes);

/* Tile-norm precision policy ("tile-centric" precision), an
 * opt-in next to the band rule of assign_precisions: tile Frobenius norms of
 * the dense row-major A (host or device) on the device, then, off the DP
 * band, tile (i, j) takes the lowest precision the variant allows with
 * u_p ||A_ij||_F <= tolerance ||A||_F / n_tiles (u: 2^-53, 2^-24, 2^-11 fp16 /
 * 2^-8 bf16) — the tiles' storage rounding then sums to <= tolerance ||A||_F.
 * map: n_tiles (n_tiles + 1) / 2 bytes, packed i(i+1)/2 + j, SPHEMU_PREC_*. */
int sphemu_gpu_tile_norm_precisions(const double* a, int where, int64_t lda, int n, const sphemu_chol_config* cfg,
                                    double tolerance, uint8_t* map);

/* Device-resident factorization handle (TiledMatrix + tiled_cholesky,
 * mpchol.hpp:47-71,135): tiles live in HBM at their storage precision. */
typedef struct sphemu_chol_s* sphemu_chol_t;
int sphemu_gpu_chol_create(int n, const sphemu_chol_config* cfg, sphemu_chol_t* out);
int sphemu_gpu_chol_destroy(sphemu_chol_t h);
/* The same handle with an explicit precision map (e.g. from
 * sphemu_gpu_tile_norm_precisions) in place of assign_precisions; diagonal
 * tiles must be SPHEMU_PREC_DP. */
int sphemu_gpu_chol_create_map(int n, const sphemu_chol_config* cfg, const uint8_t* map, sphemu_chol_t* out);
/* 2D block-cyclic distribution over a P x Q grid of GPUs (one process per
 * GPU, the caller sets the device first): off-diagonal tile (i, j) is
 * stored on rank (i mod P) * Q + (j mod Q), diagonal tile (i, i) on rank
 * i mod (P Q); panel tiles travel over NCCL point to point at their storage
 * precision, each only to the ranks that update with it. All ranks call every handle function collectively; the dense
 * factor of store_dense is gathered on rank 0. uid128 comes from
 * sphemu_gpu_nccl_unique_id on rank 0 (the caller distributes it). */
int sphemu_gpu_nccl_unique_id(void* out128);
int sphemu_gpu_chol_create_dist(int n, const sphemu_chol_config* cfg, int P, int Q, int rank,
                                const void* uid128, sphemu_chol_t* out);
/* TiledMatrix::from_dense (mpchol.cpp:124-138) + the input quantization of
 * mpchol.cpp:360-363; lda = row stride in elements. */
int sphemu_gpu_chol_load_dense(sphemu_chol_t h, const double* a, int where, int64_t lda);
/* make_spd_test_matrix(n, seed) (mpchol.cpp:419-435) generated tile by tile in
 * HBM, bitwise equal to the reference's values, then quantized. */
int sphemu_gpu_chol_generate_spd(sphemu_chol_t h, uint64_t seed);
/* tiled_cholesky (mpchol.cpp:351-410), enqueued on the handle's streams. */
int sphemu_gpu_chol_factor(sphemu_chol_t h);
/* Waits for the factorization; returns SPHEMU_ERR_NOT_SPD with *failed_tile. */
int sphemu_gpu_chol_wait(sphemu_chol_t h, sphemu_chol_stats* stats, int* failed_tile);
/* TiledMatrix::to_dense_lower (mpchol.cpp:140-154); ldf = row stride. */
int sphemu_gpu_chol_store_dense(sphemu_chol_t h, double* factor, int where, int64_t ldf);
/* ||A - L L^T||_F / ||A||_F against a dense row-major A (device or host),
 * computed on the device in FP64 (tests/support/reference.cpp:32-44). */
int sphemu_gpu_chol_residual(sphemu_chol_t h, const double* a, int where, int64_t lda,
                             double* out);
/* Size-independent check for sizes the host cannot hold: ||(A - L L^T) x|| /
 * ||A x|| for n_vec seeded random vectors x, against make_spd_test_matrix(seed). */
int sphemu_gpu_chol_residual_probe_spd(sphemu_chol_t h, uint64_t seed, int n_vec, double* out);
/* The same generator family with the 0.9 decay replaced by rho in (0, 1):
 * a_ii = 1.25 d_i^2, a_ij = 0.25 d_i d_j rho^|i-j| = D (I + K/4) D with K the
 * Kac-Murdock-Szego matrix (SPD). rho = 0.9 is make_spd_test_matrix; rho ->
 * 1 keeps every tile O(1) (0.999^512 = 0.6), the parity input where the
 * flops are. The probe regenerates A the same way. */
int sphemu_gpu_chol_generate_spd_decay(sphemu_chol_t h, uint64_t seed, double rho);
int sphemu_gpu_chol_residual_probe_spd_decay(sphemu_chol_t h, uint64_t seed, double rho, int n_vec, double* out);
/* Per-precision flop split of the factorization (BASELINE.md §4 units). */
int sphemu_gpu_chol_flops(sphemu_chol_t h, double* f_dp, double* f_sp, double* f_hp);
/* Phase profiling (CUDA events around every phase; off by default). Phases:
 * 0 POTRF+TRTRI, 1 panel TRSM, 2/3/4 trailing update of the DP/SP/HP
 * classes, 5 tile load, 6 panel exchange + import (process grids). ms/counts
 * have 7 entries. on = 1 records every phase; on = 0x100 | mask records only
 * the phases whose bit is set. */
int sphemu_gpu_chol_set_profiling(sphemu_chol_t h, int on);
int sphemu_gpu_chol_phase_times(sphemu_chol_t h, double* ms, int64_t* counts, int reset);
/* Timeline of the last profiled factorization: one span per phase launch
 * (phase as above; stream 0 = main/bulk, 1 = high-priority chain, 2 = the
 * chunked panel exchange of process grids), times in
 * ms from the factorization's start. Writes min(count, cap) entries. */
int sphemu_gpu_chol_timeline(sphemu_chol_t h, int* phase, int* stream, double* t0, double* t1, int cap,
                             int* count);
/* Trailing-update flops by output class (2 b_i b_j b_k per GEMM, b_i^2 b_k per SYRK),
 * over the tiles this rank stores. */
int sphemu_gpu_chol_update_flops(sphemu_chol_t h, double* f_dp, double* f_sp, double* f_hp);
/* Device stream the handle enqueues on (cudaStream_t as void*). */
void* sphemu_gpu_chol_stream(sphemu_chol_t h);

/* estimate_innovation_covariance (stochastic.cpp:109-172; stochastic.hpp:52-57):
 * resid is the n_rows x d innovation matrix (row-major; n_rows must equal
 * r_len*(t_len-order)). Writes u_hat (d x d, optional: NULL skips) and the
 * dense lower factor v (d x d) of u_hat + nugget*I, with the nugget escalated
 * as the reference does; every retry refactors on the device. Returns
 * SPHEMU_ERR_INVALID_ARG for bad shapes and SPHEMU_ERR_RUNTIME for a
 * non-positive mean diagonal or when the nugget passes 1e-2 * mean(diag). */
int sphemu_gpu_estimate_innovation_covariance(const double* resid, int where_resid, int64_t n_rows, int d,
                                              int r_len, int t_len, int order, const sphemu_chol_config* cfg,
                                              double* u_hat, int where_u, double* v, int where_v,
                                              double* nugget_out, sphemu_chol_stats* stats);

/* ======================================================================
 * Spherical harmonic transform (replaces sht.hpp:105-129, wigner.hpp:48-63)
 * ====================================================================== */
typedef struct sphemu_sht_s* sphemu_sht_t;
/* build_plan(GridSpec{n_theta, n_phi}, band_limit) (sht.cpp:111-171). The
 * Wigner tables are built with the memory cap of wigner.hpp:48-49 unless
 * wigner_cap_bytes is nonzero. SPHEMU_ERR_INVALID_ARG on an inadmissible grid
 * or a cap violation, with the reference's message. */
int sphemu_gpu_sht_create(int n_theta, int n_phi, int band_limit, size_t wigner_cap_bytes,
                          sphemu_sht_t* out);
int sphemu_gpu_sht_destroy(sphemu_sht_t p);
/* forward_sht_batch (sht.cpp:374-388): fields (n, n_theta, n_phi) ->
 * coefficients (n, L^2) in the packed layout of sht.hpp:24-45. */
int sphemu_gpu_sht_forward(sphemu_sht_t p, const double* fields, int where_in, int64_t n,
                           double* coeffs, int where_out);
/* inverse_sht_batch (sht.cpp:390-404). */
int sphemu_gpu_sht_inverse(sphemu_sht_t p, const double* coeffs, int where_in, int64_t n,
                           double* fields, int where_out);
/* synth_bandlimited (sht.cpp:435-466, declared sht.hpp:143): direct
 * Legendre synthesis of n packed L^2 coefficient vectors onto any
 * n_theta x n_phi equiangular grid, including grids that cannot resolve L
 * (the Python inverse_sht fallback, bindings/module.cpp:92-94). */
int sphemu_gpu_synth_bandlimited(const double* coeffs, int where_in, int64_t n, int band_limit,
                                 int n_theta, int n_phi, double* fields, int where_out);
void* sphemu_gpu_sht_stream(sphemu_sht_t p);
/* Seconds spent building the plan (Wigner recurrence + operator build). */
double sphemu_gpu_sht_plan_seconds(sphemu_sht_t p);
/* WignerTables::d_half_pi (wigner.cpp:136-150) over the tables of
 * build_wigner_tables(band_limit) (wigner.cpp:49-134), built on the device:
 * out[i] = d^{l[i]}_{m2[i], m[i]}(pi/2), with the reference's sign rules for
 * negative orders and 0 for |m2| or |m| > l. All arrays host, n entries.
 * SPHEMU_ERR_INVALID_ARG for a degree outside [0, band_limit) or a cap
 * violation (wigner_cap_bytes = 0: the 2 GiB default of wigner.hpp:48-49).
 * renorm_warnings (may be NULL) receives the guard count
 * (WignerTables::renorm_warnings). The Python wigner_d_half_pi(l, m2, m) of
 * bindings/module.cpp:201-207 calls this with band_limit = l + 1. */
int sphemu_gpu_wigner_d_half_pi(int band_limit, size_t wigner_cap_bytes, int64_t n, const int* l, const int* m2,
                                const int* m, double* out, int* renorm_warnings);

/* build_wigner_tables(band_limit, cap) (wigner.cpp:49-134) on the device,
 * copied out: offsets[m2 * band_limit + m] (band_limit^2 + 1 entries) is the
 * start of the d^l_{m2,m}(pi/2) chain for l = max(m2, m) .. band_limit - 1 in
 * d (d_count = offsets[band_limit^2] entries = sum_k (2k+1)(band_limit-k)),
 * the layout of WignerTables::d_ / d_offset_ (wigner.hpp:36-41). */
int sphemu_gpu_wigner_tables(int band_limit, size_t wigner_cap_bytes, int64_t* offsets, double* d, int64_t d_count,
                             int* renorm_warnings);

/* ======================================================================
 * Emulation generator (replaces stochastic.hpp:84-86 emulate)
 * ====================================================================== */
#define SPHEMU_RNG_REFERENCE 0 /* the reference's serial mt19937_64 stream, bit-exact order */
#define SPHEMU_RNG_PHILOX 1    /* counter-based normals generated on the device */

/* emulate(model, plan, forcing, t_out, seed, r_len) with the trend evaluated
 * by the caller: means (t_out x points), sigma (points), v2 (points), phi
 * (order x d), and the innovation factor v as a dense lower d x d matrix.
 * out is (r_len, t_out, n_theta, n_phi). All pointers host. */
int sphemu_gpu_emulate(sphemu_sht_t p, const double* v, int d, const double* phi, int order,
                       const double* means, const double* sigma, const double* v2, int t_out,
                       uint64_t seed, int r_len, int rng_mode, double* out);

/* emulate(model, plan, forcing, t_out, seed, r_len, threads, t_start)
 * (stochastic.hpp:84-86) with the model's trend given as TrendModel records
 * (points x (5 + 2*harmonics), trend.hpp:37-59) and the forcing as two
 * arrays: the mean table (stochastic.cpp:229) and sigma are evaluated on the
 * device (trend.cu) instead of crossing PCIe. */
int sphemu_gpu_emulate_trend(sphemu_sht_t p, const double* v, int d, const double* phi, int order,
                             const double* records, int harmonics, int period, const double* forcing_x, int64_t n_x,
                             const double* forcing_history, int64_t n_history, int64_t t_start, const double* v2,
                             int t_out, uint64_t seed, int r_len, int rng_mode, double* out);

/* Replicates [r_begin, r_begin + r_count) of the same emulation (out holds
 * r_count replicates): the draws of replicate r do not depend on the split,
 * so replicate ranges can run on different GPUs with no communication
 * (reference mode skips the earlier replicates' draws on the
 * host, Philox mode indexes the counter by replicate). */
int sphemu_gpu_emulate_range(sphemu_sht_t p, const double* v, int d, const double* phi, int order,
                             const double* means, const double* sigma, const double* v2, int t_out, uint64_t seed,
                             int r_begin, int r_count, int rng_mode, double* out);

/* emulate(model, plan, forcing, t_out, seed, r_len) (stochastic.hpp:84-86;
 * stochastic.cpp:217-277) with V = the device-resident tiled factor of h
 * (after sphemu_gpu_chol_factor + wait; no dense V anywhere): each step's
 * xi = V eta is a TRMM over the stored tiles at their storage precision —
 * FP64 DMMA for DP tiles, tcgen05 for SP (fp16 hi/lo of the tile x eta's
 * hi/lo) and HP tiles (the stored fp16/bf16 tile x eta's hi/lo), fp32 TMEM
 * partial sums over <= 2048 of K added into FP64. Replicates
 * [r_begin, r_begin + r_count) run in chunks that fit HBM. phi (order x d),
 * means (t_out x points), sigma, v2 (points) host; out (r_count, t_out,
 * n_theta, n_phi) host or device (where_out). Distributed handles: every rank
 * calls collectively; the replicates are split in world contiguous balanced
 * blocks (rank q: [r_begin + floor(q r_count / W), r_begin + floor((q+1) r_count / W))),
 * each rank computes the partial product over its own tiles for every rank's
 * chunk columns and the blocks are reduced onto their owners over NCCL; out
 * receives this rank's block (rng_mode must be SPHEMU_RNG_PHILOX). */
int sphemu_gpu_emulate_chol(sphemu_chol_t h, sphemu_sht_t plan, const double* phi, int order, const double* means,
                            const double* sigma, const double* v2, int t_out, uint64_t seed, int r_begin,
                            int r_count, int rng_mode, double* out, int where_out);
/* The innovation product alone: xi (S x n) = eta (S x n) L^T over the
 * handle's tiles (row-major, host or device); distributed handles all-reduce
 * the partial products so every rank receives the full xi. */
int sphemu_gpu_chol_trmm(sphemu_chol_t h, const double* eta, int where_in, int64_t S, double* xi, int where_out);

/* sphemu_gpu_emulate_chol with the model's trend as TrendModel records
 * (points x (5 + 2*harmonics)) and a forcing trajectory, evaluated on the
 * device like sphemu_gpu_emulate_trend (stochastic.cpp:229,262-273). */
int sphemu_gpu_emulate_chol_trend(sphemu_chol_t h, sphemu_sht_t plan, const double* phi, int order,
                                  const double* records, int harmonics, int period, const double* forcing_x,
                                  int64_t n_x, const double* forcing_history, int64_t n_history, int64_t t_start,
                                  const double* v2, int t_out, uint64_t seed, int r_begin, int r_count,
                                  int rng_mode, double* out, int where_out);
/* estimate_innovation_covariance keeping the factor on the device: *out is
 * a factored handle of u_hat + nugget*I (for sphemu_gpu_emulate_chol*,
 * sphemu_gpu_chol_store_dense, ...; destroy with sphemu_gpu_chol_destroy). */
int sphemu_gpu_innovation_factor(const double* resid, int where_resid, int64_t n_rows, int d, int r_len,
                                 int t_len, int order, const sphemu_chol_config* cfg, double* u_hat, int where_u,
                                 double* nugget_out, sphemu_chol_stats* stats, sphemu_chol_t* out);
/* Loads a stored lower factor (e.g. a model bundle's UCOV v, read_ucov,
 * stochastic.cpp:323-350) into the handle's tiles as its factor: the tiles
 * are quantized to the precision map like load_dense, no factorization runs. */
int sphemu_gpu_chol_load_factor(sphemu_chol_t h, const double* l, int where, int64_t ldl);

/* fit_trend(series, {}, TrendConfig{harmonics, period}) (trend.cpp:129-250)
 * without forcing — the Python Emulator.train path (module.cpp:145-157): the
 * pooled replicate mean and within-ensemble scatter, least squares on
 * [1, cos(k base), sin(k base)] (a host Householder QR of the t_len x p
 * design gives R^-1 Q^T; the projection and residual variance run per
 * location on the device). series (r_len, t_len, points) host or device;
 * records points x (5 + 2*harmonics) (trend.hpp:37-59) host or device. */
int sphemu_gpu_fit_trend(const double* series, int where_in, int r_len, int t_len, int64_t points, int harmonics,
                         int period, double* records, int where_out);
/* fit_noise_field (stochastic.cpp:176-196): v2[loc] = mean over the n_slices
 * (r, t) slices of (detrended - reconstructed)^2. */
int sphemu_gpu_noise_field(const double* detrended, const double* reconstructed, int where_in, int64_t n_slices,
                           int64_t points, double* v2, int where_out);

/* fit_var (stochastic.cpp:30-107, declared stochastic.hpp:41): per packed
 * coefficient AR(order) least squares over an (r_len, t_len, d) coefficient
 * series. phi / phi_se: order x d host (row p-1 = lag p; may be NULL);
 * residuals: (r_len * (t_len - order)) x d (r_len * t_len rows for order 0),
 * host or device — a device buffer feeds
 * sphemu_gpu_estimate_innovation_covariance directly. Counts and the residual
 * column-mean norm as VarModel::zeroed_count / unstable_count and
 * VarFit::residual_mean_norm. SPHEMU_ERR_INVALID_ARG for order < 0 or > 16
 * and t_len <= order (the reference's messages). */
int sphemu_gpu_fit_var(const double* coeffs, int where_in, int r_len, int t_len, int64_t d, int order, double* phi,
                       double* phi_se, double* residuals, int where_resid, int64_t* zeroed_count,
                       int64_t* unstable_count, double* residual_mean_norm);

/* ======================================================================
 * Trend mean structure (replaces trend.hpp:79-82 mean_table and
 * trend.hpp:71-76 detrend / retrend; trend.cpp:252-324)
 * ====================================================================== */
/* records: points x (5 + 2*harmonics) doubles, host or device (detected;
 * device records stay in HBM, only the lag column and rho are read back),
 * TrendModel::values
 * (beta0, beta1, beta2, rho, a_1..a_K, b_1..b_K, sigma; trend.hpp:37-59).
 * Forcing: ForcingTrajectory{x, history} (trend.hpp:24-35) as two host
 * arrays; n_x = n_history = 0 is the empty trajectory (no forcing terms).
 * SPHEMU_ERR_INVALID_ARG for t_start < 1 ("time steps are 1-based") and for a
 * missing lag history (require_lag_history, trend.cpp:21-25). Results are
 * bitwise those of the reference (no FMA contraction, same libm cos/sin). */
int sphemu_gpu_mean_table(const double* records, int64_t points, int harmonics, int period,
                          const double* forcing_x, int64_t n_x, const double* forcing_history, int64_t n_history,
                          int t_len, int64_t t_start, double* table, int where_out);
/* detrend (trend.cpp:289-305): out = (series - m_t) / sigma over an
 * (r_len, t_len, points) series. */
int sphemu_gpu_detrend(const double* series, int where_in, int r_len, int t_len, const double* records,
                       int64_t points, int harmonics, int period, const double* forcing_x, int64_t n_x,
                       const double* forcing_history, int64_t n_history, int64_t t_start, double* out,
                       int where_out);
/* retrend (trend.cpp:307-324): out = m_t + sigma * standardized. */
int sphemu_gpu_retrend(const double* standardized, int where_in, int r_len, int t_len, const double* records,
                       int64_t points, int harmonics, int period, const double* forcing_x, int64_t n_x,
                       const double* forcing_history, int64_t n_history, int64_t t_start, double* out,
                       int where_out);

#ifdef __cplusplus
}
#endif
#endif
