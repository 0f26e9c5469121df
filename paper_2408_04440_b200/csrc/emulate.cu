// emulate.cu — the emulation generator (replaces proj/src/stochastic.cpp:217-277)
// behind sphemu_gpu_emulate, plus the full-size residual probe of the
// Cholesky (sphemu_gpu_chol_residual_probe_spd).
//
// Reference loop per replicate: eta ~ N(0,1)^d, xi = V eta (dense GEMV),
// f = xi + sum_p phi_p * state_p, keep f after 10P burn-in steps; eps ~
// N(0,1)^points per kept step; y = m_t + sigma (inverse_sht(f_t) + sqrt(v2) eps).
// B200 form: all innovations of all replicates and steps in one FP64 GEMM
// Xi = H V^T (DMMA, zero tiles of the lower factor skipped), the AR(P)
// recursion as one pass per coefficient (serial in time, parallel over
// coefficients and replicates), one batched inverse SHT, and a fused retrend
// epilogue.
//
// RNG: SPHEMU_RNG_REFERENCE reproduces the reference's single serial
// mt19937_64 + Box-Muller stream in its exact draw order (rng.hpp:12-39,
// stochastic.cpp:230-259), generated on the host because that stream is
// serial by definition; SPHEMU_RNG_PHILOX draws counter-based normals on the
// device.
#include <algorithm>
#include <cmath>
#include <memory>
#include <random>
#include <vector>

#include "common.cuh"
#include "dgemm.cuh"
#include "dgemm2.cuh"
#include "emulate.cuh"

namespace sphemu_gpu {

struct Sht;  // sht.cu
void sht_inverse_device(void* plan, const double* coeffs, int64_t n, double* fields, cudaStream_t* s_out);

// Xi (S x d) = H (S x d) * V^T, V lower triangular dense (row-major d x d):
// output columns c0..c0+63 need V rows whose nonzeros stop at column c0+63.
__global__ void __launch_bounds__(D2_THREADS) k_emul_xi(const double* __restrict__ H, const double* __restrict__ V,
                                                         int64_t S, int d, double* __restrict__ Xi) {
  extern __shared__ __align__(16) uint8_t d2_smem[];
  D2Smem& sm = *reinterpret_cast<D2Smem*>(d2_smem);
  const int64_t r0 = (int64_t)blockIdx.y * D2_BM;
  const int c0 = blockIdx.x * D2_BN;
  const int kmax = min(d, c0 + D2_BN);
  D2Op A{H + r0 * d, d, (int)(S - r0 < D2_BM ? S - r0 : D2_BM), kmax};
  D2Op B{V + (int64_t)c0 * d, d, min(D2_BN, d - c0), kmax};
  double acc[4][4][2];
  dgemm2_128x64<D2B::kNT, false>(A, B, kmax, sm, acc);
  d2_for_each(acc, [&](int r, int c, double v0, double v1) {
    if (r0 + r >= S) return;
    if (c0 + c < d) Xi[(r0 + r) * d + c0 + c] = v0;
    if (c0 + c + 1 < d) Xi[(r0 + r) * d + c0 + c + 1] = v1;
  });
}

// AR(P) recursion (stochastic.cpp:247-253): f_t = xi_t + sum_p phi_p f_{t-p},
// state zero at the start of each replicate, burn-in steps dropped.
__global__ void k_emul_ar(const double* __restrict__ Xi, const double* __restrict__ phi, int order, int d,
                          int burn, int t_out, int r_len, double* __restrict__ draws) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (i >= d || r >= r_len) return;
  double st[16];
  double ph[16];
  for (int p = 0; p < order; ++p) {
    st[p] = 0.0;
    ph[p] = phi[(int64_t)p * d + i];
  }
  const int steps = burn + t_out;
  for (int s = 0; s < steps; ++s) {
    double f = Xi[((int64_t)r * steps + s) * d + i];
    for (int p = 0; p < order; ++p) f += ph[p] * st[p];
    for (int p = order - 1; p > 0; --p) st[p] = st[p - 1];
    if (order > 0) st[0] = f;
    if (s >= burn) draws[((int64_t)r * t_out + (s - burn)) * d + i] = f;
  }
}

// y = m_t + sigma (synth + sqrt(v2) eps)   (stochastic.cpp:266-273)
__global__ void k_emul_retrend(const double* __restrict__ synth, const double* __restrict__ eps,
                               const double* __restrict__ means, const double* __restrict__ sigma,
                               const double* __restrict__ v2, int64_t points, int t_out, int64_t total,
                               double* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t loc = e % points;
    const int64_t t = (e / points) % t_out;
    const double ep = sqrt(v2[loc]) * eps[e];
    out[e] = means[t * points + loc] + sigma[loc] * (synth[e] + ep);
  }
}

// Philox4x32-10 counter-based normals (Box-Muller on two 53-bit uniforms).
__device__ __forceinline__ void philox(uint32_t (&c)[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0], p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = (uint32_t)p1;
    c[2] = n2;
    c[3] = (uint32_t)p0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// Normals for replicates [r0, r0 + nrep), per_rep values each: replicate r's
// values depend only on (seed, stream, r), so any split of the replicates
// over calls or GPUs draws identical numbers.
__global__ void k_philox_normals(uint64_t seed, uint64_t stream, int64_t per_rep, int r0, int nrep, double* out) {
  const int64_t half = (per_rep + 1) / 2;
  const int64_t n = half * nrep;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = q / half, e = q - rr * half;
    const uint64_t st = stream + ((uint64_t)(r0 + rr) << 8);
    uint32_t c[4] = {(uint32_t)e, (uint32_t)(e >> 32), (uint32_t)st, (uint32_t)(st >> 32)};
    philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
    const double u1 = ((double)((((uint64_t)c[0] << 32) | c[1]) >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = ((double)((((uint64_t)c[2] << 32) | c[3]) >> 11) + 1.0) * 0x1.0p-53;
    const double rad = sqrt(-2.0 * log(u1));
    double s, co;
    sincospi(2.0 * u2, &s, &co);
    double* o = out + rr * per_rep;
    o[2 * e] = rad * co;
    if (2 * e + 1 < per_rep) o[2 * e + 1] = rad * s;
  }
}

// The reference's serial stream (rng.hpp:12-39): uniform (0,1] from
// mt19937_64 >> 11, Box-Muller with a cached spare.
struct RefGaussian {
  std::mt19937_64 eng;
  double spare = 0.0;
  bool has = false;
  explicit RefGaussian(uint64_t s) : eng(s) {}
  double uniform() { return static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53; }
  double normal() {
    if (has) {
      has = false;
      return spare;
    }
    const double u1 = uniform(), u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare = r * std::sin(a);
    has = true;
    return r * std::cos(a);
  }
};

void emulate_core(const EmulArgs& a, const XiFn& xi_fn) {
  if (a.r_begin < 0) throw std::invalid_argument("first replicate must be >= 0");
  if (a.t_out < 1 || a.r_len < 1) throw std::invalid_argument("need t_out, r_len >= 1");
  if (a.d != a.L * a.L) throw std::invalid_argument("transform plan does not match the model");
  if (a.order < 0 || a.order > 16) throw std::invalid_argument("lag order must lie in [0, 16]");
  const int W = std::max(1, a.world);
  if (W > 1 && a.rng_mode == SPHEMU_RNG_REFERENCE)
    throw std::invalid_argument("the reference's serial RNG stream cannot be split over ranks: use rng='philox'");
  const int d = a.d;
  const int burn = 10 * a.order;  // stochastic.cpp:17,227
  const int64_t steps = burn + a.t_out;
  const int64_t points = (int64_t)a.n_theta * a.n_phi;
  cudaStream_t s = nullptr;
  sht_inverse_device(a.plan, nullptr, 0, nullptr, &s);  // fetch the plan's stream
  std::vector<int> lo(W), cnt(W);
  int cnt_max = 0;
  for (int q = 0; q < W; ++q) {
    int l, h;
    emul_share(a.r_begin, a.r_len, W, q, l, h);
    lo[q] = l;
    cnt[q] = h - l;
    cnt_max = std::max(cnt_max, cnt[q]);
  }
  const int mine = cnt[a.rank];
  // Replicates run in chunks whose buffers fit the budget: per snapshot
  // column the normals of every rank (8 d W), the innovations and the
  // tiled product's padded operands (~32 d), the kept draws, fields and eps.
  const int64_t col_bytes = (int64_t)d * (8 * W + 32) + points * 8 * 2;
  // default chunk budget: half of the free HBM, at most 32 GB (each chunk re-reads the whole factor, and the
  // TRMM's 256-snapshot blocks fill better with more columns per chunk)
  int64_t budget = a.chunk_bytes;
  if (budget <= 0) {
    size_t fr = 0, tot = 0;
    budget = (cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr > 0)
                 ? std::min<int64_t>(int64_t{32} << 30, std::max<int64_t>(int64_t{1} << 30, (int64_t)(fr / 2)))
                 : (int64_t{8} << 30);
  }
  const int rc = (int)std::max<int64_t>(1, std::min<int64_t>(cnt_max, budget / std::max<int64_t>(1, col_bytes * steps)));
  const int n_chunks = (cnt_max + rc - 1) / rc;
  const int64_t ymax = (int64_t)rc * a.t_out * points;
  DevBuf<double> dH((size_t)W * rc * steps * d), dXi((size_t)rc * steps * d), dDraws((size_t)rc * a.t_out * d);
  DevBuf<double> dEps(ymax), dSynth(ymax), dMeans((size_t)a.t_out * points), dSigma(points), dV2(points),
      dPhi(a.order > 0 ? (size_t)a.order * d : 1);
  DevBuf<double> dTrendRec, dTrendRows;
  if (a.trend) {  // stochastic.cpp:229: mean_table(model.trend, forcing, t_out, t_start), on the device
    const TrendArgs& t = *a.trend;
    mean_table_device(t.records, points, t.harmonics, t.period, t.fx, t.nx, t.fh, t.nh, a.t_out, t.t_start,
                      dMeans.get(), dSigma.get(), s, dTrendRec, dTrendRows);
  } else {
    SPH_CUDA(cudaMemcpyAsync(dMeans.get(), a.means, (size_t)a.t_out * points * sizeof(double), cudaMemcpyHostToDevice,
                             s));
    SPH_CUDA(cudaMemcpyAsync(dSigma.get(), a.sigma, points * sizeof(double), cudaMemcpyHostToDevice, s));
  }
  SPH_CUDA(cudaMemcpyAsync(dV2.get(), a.v2, points * sizeof(double), cudaMemcpyHostToDevice, s));
  if (a.order > 0)
    SPH_CUDA(cudaMemcpyAsync(dPhi.get(), a.phi, (size_t)a.order * d * sizeof(double), cudaMemcpyHostToDevice, s));
  std::vector<double> hH, hE;
  std::unique_ptr<RefGaussian> g;
  if (a.rng_mode == SPHEMU_RNG_REFERENCE) {
    g.reset(new RefGaussian(a.seed));
    for (int r = 0; r < a.r_begin; ++r)  // one serial stream: skip the replicates drawn elsewhere
      for (int64_t e = 0; e < steps * d + (int64_t)a.t_out * points; ++e) g->normal();
    hH.resize((size_t)rc * steps * d);
    hE.resize(ymax);
  }
  std::vector<int64_t> col_off(W + 1);
  for (int c = 0; c < n_chunks; ++c) {
    col_off[0] = 0;
    for (int q = 0; q < W; ++q)
      col_off[q + 1] = col_off[q] + (int64_t)std::max(0, std::min(rc, cnt[q] - c * rc)) * steps;
    const int nr = (int)((col_off[a.rank + 1] - col_off[a.rank]) / steps);
    const int64_t ytot = (int64_t)nr * a.t_out * points;
    if (g) {
      // Exact reference order: per replicate, (burn + t_out) x d innovations,
      // then t_out x points small-scale normals.
      SPH_CUDA(cudaStreamSynchronize(s));  // the staging vectors are reused per chunk
      for (int r = 0; r < nr; ++r) {
        double* h = hH.data() + (size_t)r * steps * d;
        for (int64_t e = 0; e < steps * d; ++e) h[e] = g->normal();
        double* ep = hE.data() + (size_t)r * a.t_out * points;
        for (int64_t e = 0; e < (int64_t)a.t_out * points; ++e) ep[e] = g->normal();
      }
      SPH_CUDA(cudaMemcpyAsync(dH.get(), hH.data(), (size_t)nr * steps * d * sizeof(double), cudaMemcpyHostToDevice,
                               s));
      SPH_CUDA(cudaMemcpyAsync(dEps.get(), hE.data(), ytot * sizeof(double), cudaMemcpyHostToDevice, s));
    } else {
      for (int q = 0; q < W; ++q) {
        const int nq = (int)((col_off[q + 1] - col_off[q]) / steps);
        if (!nq) continue;
        k_philox_normals<<<4 * num_sms(), 256, 0, s>>>(a.seed, 1, steps * d, lo[q] + c * rc, nq,
                                                        dH.get() + col_off[q] * d);
        SPH_LAUNCH_CHECK();
      }
      if (nr) {
        k_philox_normals<<<4 * num_sms(), 256, 0, s>>>(a.seed, 2, (int64_t)a.t_out * points, lo[a.rank] + c * rc, nr,
                                                        dEps.get());
        SPH_LAUNCH_CHECK();
      }
    }
    xi_fn(dH.get(), col_off[W], col_off, dXi.get(), s);
    if (!nr) continue;
    k_emul_ar<<<dim3(ceil_div(d, 128), nr), 128, 0, s>>>(dXi.get(), dPhi.get(), a.order, d, burn, a.t_out, nr,
                                                          dDraws.get());
    SPH_LAUNCH_CHECK();
    sht_inverse_device(a.plan, dDraws.get(), (int64_t)nr * a.t_out, dSynth.get(), nullptr);
    k_emul_retrend<<<8 * num_sms(), 256, 0, s>>>(dSynth.get(), dEps.get(), dMeans.get(), dSigma.get(), dV2.get(),
                                                  points, a.t_out, ytot, dEps.get());
    SPH_LAUNCH_CHECK();
    double* dst = a.out + (int64_t)c * rc * a.t_out * points;
    SPH_CUDA(cudaMemcpyAsync(dst, dEps.get(), ytot * sizeof(double),
                             a.where_out == SPHEMU_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
  }
  (void)mine;
  SPH_CUDA(cudaStreamSynchronize(s));
}

// The dense-V form (sphemu_gpu_emulate*): V uploaded once per call, Xi = H V^T by DMMA.
void emulate(void* plan, int n_theta, int n_phi, int L, const double* v, int d, const double* phi, int order,
             const double* means, const double* sigma, const double* v2, int t_out, uint64_t seed, int r_len,
             int rng_mode, double* out, int r_begin, const TrendArgs* trend) {
  EmulArgs a{plan, n_theta, n_phi, L, d, phi, order, means, sigma, v2, t_out, seed, r_begin, r_len, rng_mode,
             out, SPHEMU_HOST, trend, 0};
  cudaStream_t s = nullptr;
  sht_inverse_device(plan, nullptr, 0, nullptr, &s);
  if (d != L * L) throw std::invalid_argument("transform plan does not match the model");
  DevBuf<double> dV((size_t)d * d);
  SPH_CUDA(cudaMemcpyAsync(dV.get(), v, (size_t)d * d * sizeof(double), cudaMemcpyHostToDevice, s));
  smem_optin(reinterpret_cast<const void*>(k_emul_xi), (int)sizeof(D2Smem));
  emulate_core(a, [&](const double* dH, int64_t S, const std::vector<int64_t>&, double* dXi, cudaStream_t st) {
    k_emul_xi<<<dim3(ceil_div(d, D2_BN), (unsigned)ceil_div(S, D2_BM)), D2_THREADS, sizeof(D2Smem), st>>>(
        dH, dV.get(), S, d, dXi);
    SPH_LAUNCH_CHECK();
  });
}

}  // namespace sphemu_gpu
