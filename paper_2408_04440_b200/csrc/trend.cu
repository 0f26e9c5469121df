// trend.cu — the deterministic mean structure either side of the emulator's
// hot path: mean_table / detrend / retrend of
// proj/src/trend.cpp:252-324 on the device.
//
// Work split. The per-step scalars (current-year forcing x_t, the lagged
// forcing average of the shared rho, and the K seasonal cos/sin pairs) are
// O(t_len) host work done here in the library (same libm, same operation
// order as trend.cpp:258-277). The O(t_len * points) evaluation runs in one
// HBM-bound kernel: a CTA owns 128 consecutive locations and 128 time rows;
// each thread loads its location record once into registers (compile-time
// harmonic count; runtime counts stage the records in shared memory), the
// rows' per-step scalars sit in shared memory (broadcast reads), eight rows'
// loads are in flight per thread, and each row's output is written (and for
// detrend/retrend its input read) fully coalesced. Algorithmic bytes per
// element: 8 (table) or 16 (detrend / retrend). All arithmetic is explicit
// round-to-nearest without FMA contraction, in the reference's expression
// order, so the results are bitwise those of the reference's x86-64 Release
// build (no FMA), which the oracle restates.
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "sphemu_gpu.h"

namespace sphemu_gpu {
namespace {

constexpr double kTwoPi = 2.0 * 3.14159265358979323846;  // trend.cpp:14
constexpr double kLagWeightCutoff = 1e-12;                // trend.cpp:15
constexpr int kTrendThreads = 128;
constexpr int kTrendRows = 128;

enum TrendMode { kTable = 0, kDetrend = 1, kRetrend = 2 };

// ForcingTrajectory (trend.hpp:24-35; trend.cpp:35-57).
struct Forcing {
  const double* x;
  int64_t nx;
  const double* hist;
  int64_t nh;
  bool empty() const { return nx == 0 && nh == 0; }
  bool has_year(int64_t year) const { return year >= 1 ? year <= nx : -year < nh; }
  double at_year(int64_t year) const {
    if (!has_year(year)) return 0.0;
    return year >= 1 ? x[year - 1] : hist[-year];
  }
  double lagged_mean(int64_t year, double rho) const {
    double acc = 0.0, w = 1.0;
    for (int64_t s = 1;; ++s) {
      if (!has_year(year - s)) break;
      acc += w * at_year(year - s);
      w *= rho;
      if (w < kLagWeightCutoff) break;
    }
    return (1.0 - rho) * acc;
  }
};

int64_t year_of(int64_t t, int period) { return (t + period - 1) / period; }  // trend.cpp:18

// One row of per-step scalars: {x_t, lagged, cos(base), sin(base), ..., cos(K base), sin(K base)}
// (trend.cpp:259-275). Throws like require_lag_history (trend.cpp:21-25).
std::vector<double> row_params(bool any_lag, double rho, int harmonics, int period, const Forcing& f, int t_len,
                               int64_t t_start) {
  const int rp = 2 + 2 * harmonics;
  std::vector<double> out((size_t)t_len * rp, 0.0);
  const bool with_forcing = !f.empty();
  for (int row = 0; row < t_len; ++row) {
    const int64_t t = t_start + row;
    double* o = out.data() + (size_t)row * rp;
    const double base = kTwoPi * static_cast<double>(t % period) / period;
    for (int k = 1; k <= harmonics; ++k) {
      o[2 + 2 * (k - 1)] = std::cos(base * k);
      o[2 + 2 * (k - 1) + 1] = std::sin(base * k);
    }
    if (with_forcing) {
      const int64_t year = year_of(t, period);
      if (any_lag && !f.has_year(year - 1))
        throw std::invalid_argument("lagged forcing term needs history before year " + std::to_string(year));
      o[0] = f.at_year(year);
      o[1] = f.lagged_mean(year, rho);  // rho is shared: record(0)[3]
    }
  }
  return out;
}

// m_t at one location (trend.cpp:270-279 order). K >= 0: compile-time
// harmonics, rec is a register array; K < 0: runtime count, rec in smem.
template <int K>
__device__ __forceinline__ double eval_mean(const double* rec, const double* p, int harmonics, int with_forcing) {
  const int hk = K >= 0 ? K : harmonics;
  double m = rec[0];
  if (with_forcing) m = __dadd_rn(m, __dadd_rn(__dmul_rn(rec[1], p[0]), __dmul_rn(rec[2], p[1])));
#pragma unroll
  for (int k = 0; k < (K >= 0 ? K : hk); ++k)
    m = __dadd_rn(m, __dadd_rn(__dmul_rn(rec[4 + k], p[2 + 2 * k]), __dmul_rn(rec[4 + hk + k], p[3 + 2 * k])));
  return m;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  if (pa.type != cudaMemoryTypeDevice) return false;  // not Managed: with HMM, pageable host memory reports as managed
  int dev = 0;
  SPH_CUDA(cudaGetDevice(&dev));
  if (pa.device != dev)
    throw std::invalid_argument("trend records live on device " + std::to_string(pa.device) +
                                ", not on the current device " + std::to_string(dev));
  return true;
}

// any(record[loc][2] != 0) over device records: one flag word back to the host.
__global__ void k_any_lag(const double* __restrict__ records, int64_t points, int64_t stride, int* flag) {
  int hit = 0;
  for (int64_t loc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; loc < points && !hit;
       loc += (int64_t)gridDim.x * blockDim.x)
    hit = records[loc * stride + 2] != 0.0;
  if (__syncthreads_or(hit) && threadIdx.x == 0) atomicOr(flag, 1);
}

// The two record columns the host needs for the per-step scalars: whether any
// location has a lag coefficient (require_lag_history) and the shared rho.
// Device records: only column 2 and record(0)[3] cross PCIe.
void lag_info(const double* records, bool dev, int64_t points, int64_t stride, bool with_forcing, bool& any_lag,
              double& rho) {
  any_lag = false;
  rho = 0.0;
  if (!with_forcing || points == 0) return;
  const double* c2 = records + 2;
  if (dev) {
    int* flag = scratch<int>(3, 4);
    SPH_CUDA(cudaMemset(flag, 0, sizeof(int)));
    k_any_lag<<<std::max(1, std::min(ceil_div(points, 256), 4 * num_sms())), 256>>>(records, points, stride, flag);
    SPH_LAUNCH_CHECK();
    int h = 0;
    SPH_CUDA(cudaMemcpy(&h, flag, sizeof(int), cudaMemcpyDeviceToHost));
    SPH_CUDA(cudaMemcpy(&rho, records + 3, sizeof(double), cudaMemcpyDeviceToHost));
    any_lag = h != 0;
  } else {
    rho = records[3];
    for (int64_t loc = 0; loc < points && !any_lag; ++loc) any_lag = c2[loc * stride] != 0.0;
  }
}

// grid: x = location blocks of kTrendThreads, y = blocks of kTrendRows (r, t) rows.
// Shared memory: the CTA's records (kTrendThreads x stride) then its rows'
// per-step scalars (kTrendRows x rp).
template <int MODE, int K>
__global__ void __launch_bounds__(kTrendThreads) k_trend(const double* __restrict__ records, int64_t points,
                                                         int harmonics, const double* __restrict__ rowp,
                                                         int with_forcing, int t_len, int64_t row_base,
                                                         int64_t n_rows, const double* __restrict__ in,
                                                         double* __restrict__ out) {
  extern __shared__ double s_mem[];
  const int hk = K >= 0 ? K : harmonics;
  const int stride = 5 + 2 * hk;
  const int rp = 2 + 2 * hk;
  // Compile-time K: each thread reads its own record straight into registers
  // (the warp's 15 loads cover one contiguous span, served from L1), so shared
  // memory only holds the rows' per-step scalars and occupancy stays high.
  // Runtime K: the records are staged in shared memory first.
  double* s_rec = s_mem;
  double* s_row = K >= 0 ? s_mem : s_mem + kTrendThreads * stride;
  const int64_t loc0 = (int64_t)blockIdx.x * kTrendThreads;
  const int nloc = (int)(points - loc0 < kTrendThreads ? points - loc0 : kTrendThreads);
  const int64_t r_begin = row_base + (int64_t)blockIdx.y * kTrendRows;
  const int nr = (int)(r_begin + kTrendRows < n_rows ? kTrendRows : n_rows - r_begin);
  const double* src = records + loc0 * stride;
  if (K < 0)
    for (int i = threadIdx.x; i < nloc * stride; i += kTrendThreads) s_rec[i] = src[i];
  for (int i = threadIdx.x; i < nr * rp; i += kTrendThreads)
    s_row[i] = rowp[((r_begin + i / rp) % t_len) * rp + i % rp];
  __syncthreads();
  if ((int)threadIdx.x >= nloc) return;
  const int64_t loc = loc0 + threadIdx.x;
  constexpr int kRegs = K >= 0 ? 5 + 2 * K : 1;
  double reg[kRegs];
  const double* rec = s_rec + threadIdx.x * stride;
  if constexpr (K >= 0) {
#pragma unroll
    for (int i = 0; i < kRegs; ++i) reg[i] = __ldg(src + threadIdx.x * stride + i);
    rec = reg;
  }
  const double sigma = rec[stride - 1];
  const double* pin = in + r_begin * points + loc;
  double* pout = out + r_begin * points + loc;
  constexpr int U = 8;  // rows in flight per thread
  for (int j = 0; j < nr; j += U) {
    double x[U];
    if (MODE != kTable) {
#pragma unroll
      for (int u = 0; u < U; ++u) x[u] = j + u < nr ? __ldcs(pin + (int64_t)(j + u) * points) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j + u >= nr) break;
      const double m = eval_mean<K>(rec, s_row + (j + u) * rp, hk, with_forcing);
      double v;
      if (MODE == kTable) v = m;
      else if (MODE == kDetrend) v = __ddiv_rn(__dsub_rn(x[u], m), sigma);  // trend.cpp:302
      else v = __dadd_rn(m, __dmul_rn(sigma, x[u]));                        // trend.cpp:320
      __stcs(pout + (int64_t)(j + u) * points, v);
    }
  }
}

template <int MODE>
void launch_trend(dim3 grid, size_t smem, const double* rec, int64_t points, int harmonics, const double* rowp,
                  int wf, int t_len, int64_t row_base, int64_t n_rows, const double* in, double* out,
                  cudaStream_t stream = nullptr) {
  const size_t smem_rows = (size_t)kTrendRows * (2 + 2 * harmonics) * sizeof(double);
#define SPH_TREND_CASE(KK)                                                                                  \
  case KK:                                                                                                   \
    k_trend<MODE, KK><<<grid, kTrendThreads, smem_rows, stream>>>(rec, points, harmonics, rowp, wf, t_len, row_base, \
                                                             n_rows,                                         \
                                                     in, out);                                               \
    break;
  switch (harmonics) {
    SPH_TREND_CASE(0)
    SPH_TREND_CASE(1)
    SPH_TREND_CASE(2)
    SPH_TREND_CASE(3)
    SPH_TREND_CASE(4)
    SPH_TREND_CASE(5)
    SPH_TREND_CASE(6)
    SPH_TREND_CASE(8)
    default:
      SPH_CUDA(cudaFuncSetAttribute(k_trend<MODE, -1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      k_trend<MODE, -1><<<grid, kTrendThreads, smem, stream>>>(rec, points, harmonics, rowp, wf, t_len, row_base,
                                                               n_rows, in, out);
  }
#undef SPH_TREND_CASE
  SPH_LAUNCH_CHECK();
}

template <int MODE>
void run_trend(const double* records, int64_t points, int harmonics, int period, const double* fx, int64_t nx,
               const double* fh, int64_t nh, int r_len, int t_len, int64_t t_start, const double* in, int where_in,
               double* out, int where_out) {
  if (t_start < 1) throw std::invalid_argument("time steps are 1-based");
  if (period < 1) throw std::invalid_argument("period must be positive");
  if (harmonics < 0) throw std::invalid_argument("harmonics must be non-negative");
  if (points < 0 || t_len < 0 || r_len < 0) throw std::invalid_argument("negative extent");
  if ((nx > 0 && !fx) || (nh > 0 && !fh) || nx < 0 || nh < 0)
    throw std::invalid_argument("forcing arrays missing");
  const Forcing f{fx, nx, fh, nh};
  if (points == 0 || t_len == 0 || r_len == 0) return;
  const int64_t stride = 5 + 2 * (int64_t)harmonics;
  const size_t smem = ((size_t)kTrendThreads * stride + (size_t)kTrendRows * (2 + 2 * harmonics)) * sizeof(double);
  if (smem > 200 * 1024) throw std::invalid_argument("harmonics too large for the device trend kernel");
  const bool rec_dev = is_device_ptr(records);
  bool any_lag;
  double rho;
  lag_info(records, rec_dev, points, stride, !f.empty(), any_lag, rho);
  std::vector<double> rp = row_params(any_lag, rho, harmonics, period, f, t_len, t_start);
  const int64_t n_rows = (int64_t)r_len * t_len;
  const size_t n_el = (size_t)n_rows * points;
  DevBuf<double> d_in, d_out;
  double* const d_rp = scratch<double>(1, rp.size());
  const double* drec = records;
  if (!rec_dev) {
    double* const d_rec = scratch<double>(2, (size_t)points * stride);
    SPH_CUDA(cudaMemcpy(d_rec, records, sizeof(double) * points * stride, cudaMemcpyHostToDevice));
    drec = d_rec;
  }
  SPH_CUDA(cudaMemcpy(d_rp, rp.data(), sizeof(double) * rp.size(), cudaMemcpyHostToDevice));
  const double* din = in;
  if (MODE != kTable && where_in == SPHEMU_HOST) {
    d_in.alloc(n_el);
    SPH_CUDA(cudaMemcpy(d_in.get(), in, sizeof(double) * n_el, cudaMemcpyHostToDevice));
    din = d_in.get();
  }
  double* dout = out;
  if (where_out == SPHEMU_HOST) {
    d_out.alloc(n_el);
    dout = d_out.get();
  }
  const int64_t gy = (n_rows + kTrendRows - 1) / kTrendRows;
  for (int64_t y0 = 0; y0 < gy; y0 += 65535) {
    const dim3 grid((unsigned)ceil_div(points, kTrendThreads), (unsigned)std::min<int64_t>(65535, gy - y0));
    launch_trend<MODE>(grid, smem, drec, points, harmonics, d_rp, !f.empty(), t_len, y0 * kTrendRows,
                       n_rows, din, dout);
  }
  if (where_out == SPHEMU_HOST)
    SPH_CUDA(cudaMemcpy(out, dout, sizeof(double) * n_el, cudaMemcpyDeviceToHost));
  SPH_CUDA(cudaDeviceSynchronize());
}

}  // namespace

__global__ void k_trend_sigma(const double* __restrict__ records, int64_t points, int stride,
                              double* __restrict__ sigma) {
  for (int64_t loc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; loc < points; loc += (int64_t)gridDim.x * blockDim.x)
    sigma[loc] = records[loc * stride + stride - 1];
}

// mean_table + the sigma column into device buffers on `stream` (emulate's
// trend-model overload, stochastic.cpp:262-273 with trend.cpp:252-287). The
// device records/row buffers live until the stream reaches them: the caller
// synchronizes the stream before returning.
void mean_table_device(const double* records, int64_t points, int harmonics, int period, const double* fx,
                       int64_t nx, const double* fh, int64_t nh, int t_len, int64_t t_start, double* d_table,
                       double* d_sigma, cudaStream_t stream, DevBuf<double>& d_rec, DevBuf<double>& d_rp) {
  if (t_start < 1) throw std::invalid_argument("time steps are 1-based");
  if (period < 1) throw std::invalid_argument("period must be positive");
  if (harmonics < 0) throw std::invalid_argument("harmonics must be non-negative");
  if ((nx > 0 && !fx) || (nh > 0 && !fh) || nx < 0 || nh < 0) throw std::invalid_argument("forcing arrays missing");
  const Forcing f{fx, nx, fh, nh};
  const int64_t stride = 5 + 2 * (int64_t)harmonics;
  const size_t smem = ((size_t)kTrendThreads * stride + (size_t)kTrendRows * (2 + 2 * harmonics)) * sizeof(double);
  if (smem > 200 * 1024) throw std::invalid_argument("harmonics too large for the device trend kernel");
  bool any_lag;
  double rho;
  // records may be host or device memory (detected as in the trend calls)
  const bool dev = is_device_ptr(records);
  lag_info(records, dev, points, stride, !f.empty(), any_lag, rho);
  std::vector<double> rp = row_params(any_lag, rho, harmonics, period, f, t_len, t_start);
  d_rp.alloc(rp.size());
  const double* rec = records;
  if (!dev) {
    d_rec.alloc((size_t)points * stride);
    SPH_CUDA(cudaMemcpyAsync(d_rec.get(), records, sizeof(double) * points * stride, cudaMemcpyHostToDevice, stream));
    rec = d_rec.get();
  }
  SPH_CUDA(cudaMemcpyAsync(d_rp.get(), rp.data(), sizeof(double) * rp.size(), cudaMemcpyHostToDevice, stream));
  const int64_t gy = (t_len + kTrendRows - 1) / kTrendRows;
  for (int64_t y0 = 0; y0 < gy; y0 += 65535) {
    const dim3 grid((unsigned)ceil_div(points, kTrendThreads), (unsigned)std::min<int64_t>(65535, gy - y0));
    launch_trend<kTable>(grid, smem, rec, points, harmonics, d_rp.get(), !f.empty(), t_len, y0 * kTrendRows,
                         t_len, nullptr, d_table, stream);
  }
  k_trend_sigma<<<2 * num_sms(), 256, 0, stream>>>(rec, points, (int)stride, d_sigma);
  SPH_LAUNCH_CHECK();
  // rp is a pageable host vector: the async copy above is staged before it returns.
}

// ---- fit_trend (trend.cpp:129-250) without forcing ---------------------------
// Pooled ensemble mean (trend.cpp:144-150, replicates summed in order then
// divided) and the within-ensemble scatter (trend.cpp:151-159), one thread
// per location, every (r, t) row read coalesced.
__global__ void k_trend_pool(const double* __restrict__ s, int r_len, int t_len, int64_t points,
                             double* __restrict__ ybar, double* __restrict__ within) {
  const int64_t loc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (loc >= points) return;
  for (int t = 0; t < t_len; ++t) {
    double acc = 0.0;
    for (int r = 0; r < r_len; ++r) acc = __dadd_rn(acc, s[((int64_t)r * t_len + t) * points + loc]);
    ybar[(int64_t)t * points + loc] = acc / r_len;
  }
  double w = 0.0;
  for (int r = 0; r < r_len; ++r)
    for (int t = 0; t < t_len; ++t) {
      const double d = s[((int64_t)r * t_len + t) * points + loc] - ybar[(int64_t)t * points + loc];
      w = __dadd_rn(w, __dmul_rn(d, d));
    }
  within[loc] = w;
}

// beta = Pinv ybar (Pinv = R^-1 Q^T of the design, p x t_len, broadcast reads),
// then the residual sum of squares and the record (trend.cpp:230-249).
template <int PMAX>
__global__ void k_trend_solve(const double* __restrict__ ybar, int t_len, int64_t points, int p,
                              const double* __restrict__ pinv, const double* __restrict__ x, const double* within,
                              int r_len, int harmonics, double* __restrict__ rec) {
  const int64_t loc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (loc >= points) return;
  double beta[PMAX];
#pragma unroll
  for (int c = 0; c < PMAX; ++c) beta[c] = 0.0;
  for (int t = 0; t < t_len; ++t) {
    const double y = ybar[(int64_t)t * points + loc];
#pragma unroll
    for (int c = 0; c < PMAX; ++c)
      if (c < p) beta[c] = fma(__ldg(pinv + (int64_t)c * t_len + t), y, beta[c]);
  }
  double rss = 0.0;
  for (int t = 0; t < t_len; ++t) {
    double fit = 0.0;
#pragma unroll
    for (int c = 0; c < PMAX; ++c)
      if (c < p) fit = fma(__ldg(x + (int64_t)t * p + c), beta[c], fit);
    const double e = ybar[(int64_t)t * points + loc] - fit;
    rss = fma(e, e, rss);
  }
  const int stride = 5 + 2 * harmonics;
  double* o = rec + loc * stride;
  o[0] = beta[0];
  o[1] = o[2] = o[3] = 0.0;
#pragma unroll
  for (int k = 0; k < (PMAX - 1) / 2; ++k)
    if (k < harmonics) {
      o[4 + k] = beta[1 + 2 * k];
      o[4 + harmonics + k] = beta[2 + 2 * k];
    }
  const double var = (r_len * rss + within[loc]) / (static_cast<double>(r_len) * t_len);
  o[stride - 1] = sqrt(fmax(var, 1e-12));  // kSigmaFloor (trend.cpp:16)
}

// fit_noise_field (stochastic.cpp:176-196): mean over slices of (a - b)^2.
__global__ void k_noise_field(const double* __restrict__ a, const double* __restrict__ b, int64_t n_slices,
                              int64_t points, double* __restrict__ v2) {
  const int64_t loc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (loc >= points) return;
  double acc = 0.0;
  for (int64_t sl = 0; sl < n_slices; ++sl) {
    const double e = a[sl * points + loc] - b[sl * points + loc];
    acc = __dadd_rn(acc, __dmul_rn(e, e));
  }
  v2[loc] = acc * (1.0 / static_cast<double>(n_slices));
}

// Householder QR of the t_len x p design (column-major work copy), giving
// Pinv = R^-1 Q^T (p x t_len) — the least-squares solve of
// Eigen::HouseholderQR::solve (trend.cpp:231-232) as one matrix.
std::vector<double> design_pinv(const std::vector<double>& x, int m, int p) {
  std::vector<double> a(x);  // row-major m x p
  std::vector<double> qt((size_t)m * m, 0.0);  // accumulate Q^T applied to I, only first p rows needed
  std::vector<std::vector<double>> vs;
  std::vector<double> taus;
  for (int k = 0; k < p; ++k) {
    double nrm = 0.0;
    for (int i = k; i < m; ++i) nrm += a[(size_t)i * p + k] * a[(size_t)i * p + k];
    nrm = std::sqrt(nrm);
    const double alpha = a[(size_t)k * p + k] >= 0 ? -nrm : nrm;
    std::vector<double> v(m, 0.0);
    for (int i = k; i < m; ++i) v[i] = a[(size_t)i * p + k];
    v[k] -= alpha;
    double vn = 0.0;
    for (int i = k; i < m; ++i) vn += v[i] * v[i];
    const double tau = vn > 0.0 ? 2.0 / vn : 0.0;
    for (int j = k; j < p; ++j) {
      double d = 0.0;
      for (int i = k; i < m; ++i) d += v[i] * a[(size_t)i * p + j];
      d *= tau;
      for (int i = k; i < m; ++i) a[(size_t)i * p + j] -= d * v[i];
    }
    vs.push_back(std::move(v));
    taus.push_back(tau);
  }
  // rows 0..p-1 of Q^T: apply H_{p-1} ... H_0 to e_i^T from the left, i.e. Q^T = H_{p-1} .. H_0
  std::vector<double> pinv((size_t)p * m, 0.0);
  std::vector<double> col(m);
  for (int t = 0; t < m; ++t) {  // column t of Q^T = Q^T e_t
    std::fill(col.begin(), col.end(), 0.0);
    col[t] = 1.0;
    for (int k = 0; k < p; ++k) {
      double d = 0.0;
      for (int i = k; i < m; ++i) d += vs[k][i] * col[i];
      d *= taus[k];
      for (int i = k; i < m; ++i) col[i] -= d * vs[k][i];
    }
    // back-substitute R z = (Q^T e_t)[0:p]
    for (int c = p - 1; c >= 0; --c) {
      double acc = col[c];
      for (int j = c + 1; j < p; ++j) acc -= a[(size_t)c * p + j] * pinv[(size_t)j * m + t];
      pinv[(size_t)c * m + t] = acc / a[(size_t)c * p + c];
    }
  }
  return pinv;
}

void fit_trend_device(const double* series, int where_in, int r_len, int t_len, int64_t points, int harmonics,
                      int period, double* records, int where_out) {
  if (period != 12 && period != 365 && period != 8760)
    throw std::invalid_argument("period must be 12, 365 or 8760 steps per year");  // trend.cpp:28-34
  if (harmonics < 0) throw std::invalid_argument("harmonics must be non-negative");
  if (2 * harmonics >= period) throw std::invalid_argument("harmonics must stay below half the period");
  if (r_len < 1 || t_len < 1 || points < 1) throw std::invalid_argument("series needs t_len, r_len >= 1");
  if (t_len < 4 + 2 * harmonics)
    throw std::invalid_argument("need at least 4 + 2*harmonics time steps to fit the trend");
  if (harmonics > 7) throw std::invalid_argument("harmonics above 7 are not supported by the device trend fit");
  const int p = 1 + 2 * harmonics;
  // design rows t = 1..t_len: 1, cos(k base), sin(k base) (trend.cpp:96-111)
  std::vector<double> x((size_t)t_len * p);
  for (int row = 0; row < t_len; ++row) {
    const int64_t t = row + 1;
    double* o = x.data() + (size_t)row * p;
    o[0] = 1.0;
    const double base = kTwoPi * static_cast<double>(t % period) / period;
    for (int k = 1; k <= harmonics; ++k) {
      o[1 + 2 * (k - 1)] = std::cos(base * k);
      o[2 + 2 * (k - 1)] = std::sin(base * k);
    }
  }
  const std::vector<double> pinv = design_pinv(x, t_len, p);
  const size_t n = (size_t)r_len * t_len * points;
  DevBuf<double> d_in, ybar((size_t)t_len * points), within(points), d_x(x.size()), d_p(pinv.size()), d_rec;
  const double* s = series;
  if (where_in == SPHEMU_HOST) {
    d_in.alloc(n);
    SPH_CUDA(cudaMemcpy(d_in.get(), series, n * sizeof(double), cudaMemcpyHostToDevice));
    s = d_in.get();
  }
  SPH_CUDA(cudaMemcpy(d_x.get(), x.data(), x.size() * sizeof(double), cudaMemcpyHostToDevice));
  SPH_CUDA(cudaMemcpy(d_p.get(), pinv.data(), pinv.size() * sizeof(double), cudaMemcpyHostToDevice));
  const int stride = 5 + 2 * harmonics;
  double* rec = records;
  if (where_out == SPHEMU_HOST) {
    d_rec.alloc((size_t)points * stride);
    rec = d_rec.get();
  }
  const unsigned grid = (unsigned)ceil_div(points, 128);
  k_trend_pool<<<grid, 128>>>(s, r_len, t_len, points, ybar.get(), within.get());
  SPH_LAUNCH_CHECK();
  k_trend_solve<15><<<grid, 128>>>(ybar.get(), t_len, points, p, d_p.get(), d_x.get(), within.get(), r_len,
                                   harmonics, rec);
  SPH_LAUNCH_CHECK();
  if (where_out == SPHEMU_HOST)
    SPH_CUDA(cudaMemcpy(records, rec, (size_t)points * stride * sizeof(double), cudaMemcpyDeviceToHost));
  SPH_CUDA(cudaDeviceSynchronize());
}

}  // namespace sphemu_gpu

extern "C" int sphemu_gpu_fit_trend(const double* series, int where_in, int r_len, int t_len, int64_t points,
                                    int harmonics, int period, double* records, int where_out) {
  using namespace sphemu_gpu;
  return guard([&] { fit_trend_device(series, where_in, r_len, t_len, points, harmonics, period, records, where_out); });
}

extern "C" int sphemu_gpu_noise_field(const double* detrended, const double* reconstructed, int where_in,
                                      int64_t n_slices, int64_t points, double* v2, int where_out) {
  using namespace sphemu_gpu;
  return guard([&] {
    if (n_slices < 1 || points < 1) throw std::invalid_argument("empty series");
    const size_t n = (size_t)n_slices * points;
    DevBuf<double> da, db, dv;
    const double* a = detrended;
    const double* b = reconstructed;
    if (where_in == SPHEMU_HOST) {
      da.alloc(n);
      db.alloc(n);
      SPH_CUDA(cudaMemcpy(da.get(), detrended, n * sizeof(double), cudaMemcpyHostToDevice));
      SPH_CUDA(cudaMemcpy(db.get(), reconstructed, n * sizeof(double), cudaMemcpyHostToDevice));
      a = da.get();
      b = db.get();
    }
    double* v = v2;
    if (where_out == SPHEMU_HOST) {
      dv.alloc(points);
      v = dv.get();
    }
    k_noise_field<<<(unsigned)ceil_div(points, 128), 128>>>(a, b, n_slices, points, v);
    SPH_LAUNCH_CHECK();
    if (where_out == SPHEMU_HOST) SPH_CUDA(cudaMemcpy(v2, v, points * sizeof(double), cudaMemcpyDeviceToHost));
    SPH_CUDA(cudaDeviceSynchronize());
  });
}


extern "C" int sphemu_gpu_mean_table(const double* records, int64_t points, int harmonics, int period,
                                     const double* forcing_x, int64_t n_x, const double* forcing_history,
                                     int64_t n_history, int t_len, int64_t t_start, double* table, int where_out) {
  using namespace sphemu_gpu;
  return guard([&] {
    run_trend<kTable>(records, points, harmonics, period, forcing_x, n_x, forcing_history, n_history, 1, t_len,
                      t_start, nullptr, SPHEMU_HOST, table, where_out);
  });
}

extern "C" int sphemu_gpu_detrend(const double* series, int where_in, int r_len, int t_len, const double* records,
                                  int64_t points, int harmonics, int period, const double* forcing_x, int64_t n_x,
                                  const double* forcing_history, int64_t n_history, int64_t t_start, double* out,
                                  int where_out) {
  using namespace sphemu_gpu;
  return guard([&] {
    run_trend<kDetrend>(records, points, harmonics, period, forcing_x, n_x, forcing_history, n_history, r_len,
                        t_len, t_start, series, where_in, out, where_out);
  });
}

extern "C" int sphemu_gpu_retrend(const double* standardized, int where_in, int r_len, int t_len,
                                  const double* records, int64_t points, int harmonics, int period,
                                  const double* forcing_x, int64_t n_x, const double* forcing_history,
                                  int64_t n_history, int64_t t_start, double* out, int where_out) {
  using namespace sphemu_gpu;
  return guard([&] {
    run_trend<kRetrend>(records, points, harmonics, period, forcing_x, n_x, forcing_history, n_history, r_len,
                        t_len, t_start, standardized, where_in, out, where_out);
  });
}
