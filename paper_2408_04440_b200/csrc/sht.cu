// sht.cu — B200 spherical harmonic transform behind the C-ABI of
// include/sphemu_gpu.h (replaces proj/src/sht.cpp:111-404).
//
// The reference analysis per order m is  ring FFT -> parity extension ->
// FFT(2 n_theta - 2) -> J = K * I -> Wigner contraction  (sht.cpp:226-263),
// and synthesis is  K = sum_l q z -> spectrum -> FFT(2 n_theta - 2) -> ring
// FFT  (sht.cpp:304-357). Everything after the ring FFT is linear and fixed
// per m, so the plan composes it once into real operators:
//   forward  f_{l,m} = sum_i Psi_m[l, i] g_m(theta_i)
//            Psi_m = Re(2 pi i^{-m} Q_m V_par(m)),
//            V_par(m2, i) = W(m2, i) + par W(-m2, i),
//            W(m2, i) = (1/n_ext) sum_{m'} I(m' + m2) (w^{-i m'} + par [interior] w^{i m'})
//   inverse  g_m(theta_i) = sum_l Y_m[i, l] z_{l,m},
//            Y_m = s_m (Q_m T_par)^T, T_+ = (1, 2cos m' theta), T_- = (0, 2sin m' theta)
// with Q_m[l, m2] = q(l, m, m2) (wigner.cpp:152-163). Both are the exact
// linear maps of the reference on every input (band-limited or not). Psi_m,
// Y_m are built on the GPU by FP64 DMMA GEMMs; a transform is then one
// batched ring FFT (HBM-bound) plus one grouped FP64 Legendre GEMM over m.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "hostio.cuh"
#include "dgemm.cuh"
#include "dgemm2.cuh"

namespace sphemu_gpu {

// ===========================================================================
// Wigner d(pi/2) tables (wigner.cpp:49-134), built on the device.
// Layout as the reference: chain (a, b) = (m2, m) >= 0 holds l = max(a,b)..L-1
// contiguously, starting at off[a * L + b]. One thread per chain runs the
// degree recurrence; one thread per (l, b) runs the renormalization guard
// (every guard column touches its own entries, so the columns are
// independent). The recurrence and the guard use explicitly rounded
// operations in the reference's evaluation order (no FMA contraction), so
// they match the host arithmetic of wigner.cpp; the chain seed
// 2^-l0 sqrt(prod (l0+lo+k)/k) (wigner.cpp:18-28, long double there) is a
// double-double product with power-of-two rescaling.
// ===========================================================================

static size_t wigner_bytes(int L) {
  size_t d_entries = 0;
  for (int a = 0; a < L; ++a)
    for (int b = 0; b < L; ++b) d_entries += static_cast<size_t>(L - std::max(a, b));
  const size_t q_entries = static_cast<size_t>(L) * L * (L + 1) / 2;
  return (d_entries + q_entries) * sizeof(double) + (static_cast<size_t>(L) * L + 1) * sizeof(size_t);
}

__device__ __forceinline__ void dd_mul(double& h, double& lo, double bh, double bl) {
  const double p = h * bh;
  double e = fma(h, bh, -p);
  e += h * bl + lo * bh;
  const double s = p + e;
  lo = e - (s - p);
  h = s;
}

__device__ double wigner_seed(int a, int b) {
  const int l0 = max(a, b), lo = min(a, b);
  double h = 1.0, hl = 0.0;
  int e2 = 0;  // product = (h + hl) * 2^e2, e2 even
  for (int k = 1; k <= l0 - lo; ++k) {
    const double num = (double)(l0 + lo + k), den = (double)k;
    const double q = num / den;
    const double r = fma(-q, den, num) / den;
    dd_mul(h, hl, q, r);
    if (h > 0x1p600) { h *= 0x1p-600; hl *= 0x1p-600; e2 += 600; }
  }
  const double s = sqrt(h);
  const double t = (fma(-s, s, h) + hl) / (2.0 * s);
  const double v = ldexp(s + t, e2 / 2 - l0);
  return ((l0 - b) & 1) ? -v : v;
}

__global__ void k_wigner_chains(int L, const int64_t* __restrict__ off, double* __restrict__ d) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)L * L) return;
  const int a = (int)(t / L), b = (int)(t % L);
  const int l0 = max(a, b);
  double* chain = d + off[t];
  const double seed = wigner_seed(a, b);
  chain[0] = seed;
  if (l0 + 1 >= L) return;
  const double da = (double)a, db = (double)b;
  double prev = 0.0, cur = seed;
  double c0 = __dmul_rn(__dmul_rn(__dmul_rn(sqrt((double)(l0 + a)), sqrt((double)(l0 - a))), sqrt((double)(l0 + b))),
                        sqrt((double)(l0 - b)));
  for (int l = l0; l + 1 < L; ++l) {
    double next;
    const double c1 = __dmul_rn(__dmul_rn(__dmul_rn(sqrt((double)(l + 1 + a)), sqrt((double)(l + 1 - a))),
                                          sqrt((double)(l + 1 + b))),
                                sqrt((double)(l + 1 - b)));
    if (l == 0) {
      next = 0.0;
    } else {
      const double dl = (double)l;
      const double t1 = __dmul_rn(__dmul_rn(__dmul_rn(-(2.0 * dl + 1.0), da), db), cur);
      const double t2 = __dmul_rn(__dmul_rn(dl + 1.0, c0), prev);
      next = __ddiv_rn(__dsub_rn(t1, t2), __dmul_rn(dl, c1));
    }
    chain[l + 1 - l0] = next;
    prev = cur;
    cur = next;
    c0 = c1;
  }
}

__global__ void k_wigner_renorm(int L, const int64_t* __restrict__ off, double* __restrict__ d, int* renorm) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)L * (L + 1) / 2) return;
  int l = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((int64_t)l * (l + 1) / 2 > t) --l;
  while ((int64_t)(l + 1) * (l + 2) / 2 <= t) ++l;
  const int b = (int)(t - (int64_t)l * (l + 1) / 2);
  bool bad = false;
  double s = 0.0;
  for (int a = 0; a <= l; ++a) {
    const double v = d[off[(int64_t)a * L + b] + l - max(a, b)];
    if (fabs(v) > 1.0 + 1e-9) bad = true;
    s = __dadd_rn(s, __dmul_rn(__dmul_rn(a == 0 ? 1.0 : 2.0, v), v));
  }
  if (!bad) return;
  atomicAdd(renorm, 1);
  const double scale = __ddiv_rn(1.0, sqrt(s));
  for (int a = 0; a <= l; ++a) {
    double* e = d + off[(int64_t)a * L + b] + l - max(a, b);
    *e = __dmul_rn(*e, scale);
  }
}

struct WignerDev {
  int L = 0;
  int renorm = 0;
  DevBuf<double> d;
  DevBuf<int64_t> off;
};

static void check_wigner_cap(int L, size_t cap) {
  if (L < 1) throw std::invalid_argument("band limit must be positive");
  const size_t bytes = wigner_bytes(L);
  if (bytes > cap)
    throw std::invalid_argument("Wigner tables for band limit " + std::to_string(L) + " need " +
                                std::to_string(bytes) + " bytes, over the cap of " +
                                std::to_string(cap));
}

static void build_wigner_device(WignerDev& w, int L, size_t cap, cudaStream_t stream) {
  check_wigner_cap(L, cap);
  w.L = L;
  std::vector<int64_t> off(static_cast<size_t>(L) * L + 1, 0);
  int64_t o = 0;
  for (int a = 0; a < L; ++a)
    for (int b = 0; b < L; ++b) {
      off[(size_t)a * L + b] = o;
      o += L - std::max(a, b);
    }
  off.back() = o;
  w.d.alloc((size_t)o);
  w.off.alloc(off.size());
  SPH_CUDA(cudaMemcpyAsync(w.off.get(), off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice, stream));
  DevBuf<int> cnt(1);
  SPH_CUDA(cudaMemsetAsync(cnt.get(), 0, sizeof(int), stream));
  const int64_t chains = (int64_t)L * L, cols = (int64_t)L * (L + 1) / 2;
  k_wigner_chains<<<(unsigned)ceil_div(chains, (int64_t)128), 128, 0, stream>>>(L, w.off.get(), w.d.get());
  SPH_LAUNCH_CHECK();
  k_wigner_renorm<<<(unsigned)ceil_div(cols, (int64_t)128), 128, 0, stream>>>(L, w.off.get(), w.d.get(), cnt.get());
  SPH_LAUNCH_CHECK();
  SPH_CUDA(cudaMemcpyAsync(&w.renorm, cnt.get(), sizeof(int), cudaMemcpyDeviceToHost, stream));
  SPH_CUDA(cudaStreamSynchronize(stream));
}

// Gather d^l_{m2,m}(pi/2) with the sign rules of WignerTables::d_half_pi
// (wigner.cpp:136-150): zero for |m2| or |m| > l.
__global__ void k_wigner_gather(int L, const int64_t* __restrict__ off, const double* __restrict__ d, int64_t n,
                                const int* __restrict__ ls, const int* __restrict__ m2s, const int* __restrict__ ms,
                                double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int l = ls[i];
  int m2 = m2s[i], m = ms[i];
  if (abs(m2) > l || abs(m) > l) { out[i] = 0.0; return; }
  int sign = 1;
  if (m2 < 0) { sign *= ((l + m) & 1) ? -1 : 1; m2 = -m2; }
  if (m < 0) { sign *= ((l + m2) & 1) ? -1 : 1; m = -m; }
  out[i] = sign * d[off[(int64_t)m2 * L + m] + l - max(m2, m)];
}

// ===========================================================================
// Device: operator build
// ===========================================================================
// Q_m accessor: element (r, k) = q(m + r, m, k) = norm_l d^l_{k,0} d^l_{k,m}
// (wigner.cpp:152-163), zero for k > l. Used as A (forward) and as B (inverse).
struct QAcc {
  static constexpr bool kKContig = true;
  const double* d;
  const int64_t* off;
  int L, m, rows;
  __device__ double operator()(int r, int k) const {
    const int l = m + r;
    if (r >= rows || k >= L || k > l) return 0.0;
    const double norm = sqrt((2.0 * l + 1.0) / (4.0 * 3.14159265358979323846));
    const double d0 = d[off[(int64_t)k * L + 0] + l - k];
    const double dm = d[off[(int64_t)k * L + m] + l - max(k, m)];
    return norm * d0 * dm;
  }
};

// Q_m rows shifted by an output-tile origin.
struct QShift {
  static constexpr bool kKContig = true;
  QAcc q;
  int r0;
  __device__ double operator()(int r, int k) const { return q(r0 + r, k); }
};

// V tables: vre_p = Re V_+(m2, i), vim_m = Im V_-(m2, i), L x n_theta.
__global__ void k_sht_vtables(int L, int n_theta, const double2* __restrict__ tw_ext, double* vre_p,
                              double* vim_m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int m2 = blockIdx.y;
  if (i >= n_theta) return;
  const int n_ext = 2 * n_theta - 2;
  const bool interior = i > 0 && i < n_theta - 1;
  // W_par(+-m2, i) accumulated for both parities.
  double wr_p[2] = {0, 0}, wi_p[2] = {0, 0}, wr_m[2] = {0, 0}, wi_m[2] = {0, 0};
  for (int mp = -(L - 1); mp <= L - 1; ++mp) {
    // w^{-i mp} = tw_ext[(i*mp) mod n_ext] (tw = exp(-2 pi i t / n_ext))
    int t = (int)(((int64_t)i * mp) % n_ext);
    if (t < 0) t += n_ext;
    const double2 e_neg = tw_ext[t];                 // exp(-i theta mp)
    const double2 e_pos = make_double2(e_neg.x, -e_neg.y);  // exp(+i theta mp)
    // c_par = e_neg + par * [interior] e_pos
    double cp_r = e_neg.x, cp_i = e_neg.y, cm_r = e_neg.x, cm_i = e_neg.y;
    if (interior) {
      cp_r += e_pos.x; cp_i += e_pos.y;
      cm_r -= e_pos.x; cm_i -= e_pos.y;
    }
#pragma unroll
    for (int sgn = 0; sgn < 2; ++sgn) {
      const int q = mp + (sgn == 0 ? m2 : -m2);
      double Ir = 0.0, Ii = 0.0;
      if (q & 1) {
        if (q == 1) Ii = 3.14159265358979323846 / 2.0;
        else if (q == -1) Ii = -3.14159265358979323846 / 2.0;
        else continue;
      } else {
        Ir = 2.0 / (1.0 - (double)q * (double)q);
      }
      wr_p[sgn] += Ir * cp_r - Ii * cp_i;
      wi_p[sgn] += Ir * cp_i + Ii * cp_r;
      wr_m[sgn] += Ir * cm_r - Ii * cm_i;
      wi_m[sgn] += Ir * cm_i + Ii * cm_r;
    }
  }
  const double inv = 1.0 / n_ext;
  double vp, vm;
  if (m2 == 0) {
    vp = wr_p[0] * inv;
    vm = wi_m[0] * inv;
  } else {
    vp = (wr_p[0] + wr_p[1]) * inv;   // W_+(m2) + W_+(-m2)
    vm = (wi_m[0] - wi_m[1]) * inv;   // W_-(m2) - W_-(-m2)
  }
  vre_p[(int64_t)m2 * n_theta + i] = vp;
  vim_m[(int64_t)m2 * n_theta + i] = vm;
}

// Psi_m (L-m x n_theta) = s_m 2 pi Q_m Vsel, grid (n_theta/64, L/64, L).
__global__ void __launch_bounds__(DG_THREADS) k_sht_build_psi(const double* d, const int64_t* off, int L,
                                                               int n_theta, const double* vre_p,
                                                               const double* vim_m, const int64_t* psi_off,
                                                               double* psi) {
  __shared__ DgSmem sm;
  const int m = blockIdx.z;
  const int rows = L - m;
  const int r0 = blockIdx.y * DG_BM, c0 = blockIdx.x * DG_BN;
  if (r0 >= rows) return;
  QShift As{QAcc{d, off, L, m, rows}, r0};
  const double* vs = (m & 1) ? vim_m : vre_p;
  KMajor B{vs + c0, n_theta, min(DG_BN, n_theta - c0), L};
  double acc[4][4][2];
  dgemm_64x64(As, B, L, sm, acc);
  const double sgn = ((m >> 1) & 1) ? -1.0 : 1.0;
  const double scale = sgn * 2.0 * 3.14159265358979323846;
  double* out = psi + psi_off[m];
  const int ntp = (n_theta + 1) & ~1;  // even row stride (16-byte rows for the Legendre GEMM loader)
  dg_for_each(acc, [&](int r, int c, double v) {
    if (r0 + r < rows && c0 + c < n_theta) out[(int64_t)(r0 + r) * ntp + c0 + c] = scale * v;
  });
}

// Y_m (n_theta x L-m) = s_m (Q_m Tsel)^T: A(i, m') = Tsel(m', i), B(l', m') = Q_m.
__global__ void __launch_bounds__(DG_THREADS) k_sht_build_y(const double* d, const int64_t* off, int L,
                                                             int n_theta, const double* tcos,
                                                             const double* tsin, const int64_t* y_off,
                                                             double* y) {
  __shared__ DgSmem sm;
  const int m = blockIdx.z;
  const int cols = L - m;
  const int r0 = blockIdx.x * DG_BM, c0 = blockIdx.y * DG_BN;
  if (c0 >= cols) return;
  const double* ts = (m & 1) ? tsin : tcos;
  KMajor A{ts + r0, n_theta, min(DG_BM, n_theta - r0), L};
  QShift Bs{QAcc{d, off, L, m, cols}, c0};
  double acc[4][4][2];
  dgemm_64x64(A, Bs, L, sm, acc);
  const double sgn = ((m >> 1) & 1) ? -1.0 : 1.0;
  double* out = y + y_off[m];
  const int colsp = (cols + 1) & ~1;
  dg_for_each(acc, [&](int r, int c, double v) {
    if (r0 + r < n_theta && c0 + c < cols) out[(int64_t)(r0 + r) * colsp + c0 + c] = sgn * v;
  });
}

// ===========================================================================
// Device: batched ring FFT (in-place mixed-radix DIF in shared memory)
// ===========================================================================
constexpr int FFT_MAX_STAGES = 24;
struct FftPlan {
  int n;
  int stages;
  int radix[FFT_MAX_STAGES];
  const double2* tw;  // exp(-2 pi i t / n), t in [0, n)
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Generic radix p (O(p^2), p <= 64): kept out of line so the common
// radix-2/3/4/5 path does not carry its register and local-memory footprint.
template <int SIGN>
__device__ __noinline__ void fft_generic_bfly(double2* base, int span, int p, int j, int tstep, const FftPlan& P) {
  const int n = P.n;
  double2 in[64];
  const int pp = p <= 64 ? p : 64;
  for (int r = 0; r < pp; ++r) in[r] = base[r * span];
  for (int q = 0; q < pp; ++q) {
    double2 acc = make_double2(0.0, 0.0);
    for (int r = 0; r < pp; ++r) {
      double2 w = P.tw[((int64_t)((r * q) % p) * (n / p)) % n];
      if (SIGN > 0) w.y = -w.y;
      const double2 v = cmul(in[r], w);
      acc.x += v.x;
      acc.y += v.y;
    }
    double2 w = P.tw[((int64_t)j * q * tstep) % n];
    if (SIGN > 0) w.y = -w.y;
    base[q * span] = cmul(acc, w);
  }
}

// Exact t / d for t < 2^24 through a float reciprocal plus one correction step.
__device__ __forceinline__ int fdiv(int t, int d, float inv) {
  int q = static_cast<int>(static_cast<float>(t) * inv);
  if (q * d > t) --q;
  else if ((q + 1) * d <= t) ++q;
  return q;
}

// One DIF pass over R rings held in x (R * n complex), sign -1 (analysis) or
// +1 (synthesis, conjugated twiddles). Twiddle indices of radix 2..5 stay
// below n, so no modulo; butterfly coordinates use reciprocal divisions.
template <int SIGN>
__device__ void fft_dif_rings(double2* x, int R, const FftPlan& P) {
  const int n = P.n;
  int len = n;
  for (int s = 0; s < P.stages; ++s) {
    const int p = P.radix[s];
    const int span = len / p;
    const int nb = n / p;  // butterflies per ring
    const int bfly = R * nb;
    const int tstep = n / len;
    const float inv_nb = 1.0f / nb, inv_span = 1.0f / span;
    for (int t = threadIdx.x; t < bfly; t += blockDim.x) {
      const int ring = fdiv(t, nb, inv_nb);
      const int rem = t - ring * nb;
      const int g = fdiv(rem, span, inv_span), j = rem - g * span;
      double2* base = x + (int64_t)ring * n + g * len + j;
      if (p == 2) {
        const double2 a = base[0], b = base[span];
        double2 y1 = make_double2(a.x - b.x, a.y - b.y);
        base[0] = make_double2(a.x + b.x, a.y + b.y);
        double2 w = P.tw[j * tstep];
        if (SIGN > 0) w.y = -w.y;
        base[span] = cmul(y1, w);
      } else if (p == 4) {
        const double2 a0 = base[0], a1 = base[span], a2 = base[2 * span], a3 = base[3 * span];
        const double2 s02 = make_double2(a0.x + a2.x, a0.y + a2.y), d02 = make_double2(a0.x - a2.x, a0.y - a2.y);
        const double2 s13 = make_double2(a1.x + a3.x, a1.y + a3.y), d13 = make_double2(a1.x - a3.x, a1.y - a3.y);
        // -i * d13 for analysis, +i * d13 for synthesis
        const double2 rd13 = SIGN < 0 ? make_double2(d13.y, -d13.x) : make_double2(-d13.y, d13.x);
        double2 y0 = make_double2(s02.x + s13.x, s02.y + s13.y);
        double2 y2 = make_double2(s02.x - s13.x, s02.y - s13.y);
        double2 y1 = make_double2(d02.x + rd13.x, d02.y + rd13.y);
        double2 y3 = make_double2(d02.x - rd13.x, d02.y - rd13.y);
        double2 w1 = P.tw[j * tstep], w2 = P.tw[2 * j * tstep], w3 = P.tw[3 * j * tstep];
        if (SIGN > 0) { w1.y = -w1.y; w2.y = -w2.y; w3.y = -w3.y; }
        base[0] = y0;
        base[span] = cmul(y1, w1);
        base[2 * span] = cmul(y2, w2);
        base[3 * span] = cmul(y3, w3);
      } else if (p == 3) {
        // W3 = exp(-+2 pi i / 3): y1,2 = a0 - (a1+a2)/2 -+ i s (sqrt3/2)(a1-a2)
        const double2 a0 = base[0], a1 = base[span], a2 = base[2 * span];
        const double2 t = make_double2(a1.x + a2.x, a1.y + a2.y), d = make_double2(a1.x - a2.x, a1.y - a2.y);
        const double h = 0.86602540378443864676 * (SIGN < 0 ? 1.0 : -1.0);
        const double2 m = make_double2(a0.x - 0.5 * t.x, a0.y - 0.5 * t.y);
        const double2 rd = make_double2(h * d.y, -h * d.x);  // -i s (sqrt3/2) d
        double2 w1 = P.tw[j * tstep], w2 = P.tw[2 * j * tstep];
        if (SIGN > 0) { w1.y = -w1.y; w2.y = -w2.y; }
        base[0] = make_double2(a0.x + t.x, a0.y + t.y);
        base[span] = cmul(make_double2(m.x + rd.x, m.y + rd.y), w1);
        base[2 * span] = cmul(make_double2(m.x - rd.x, m.y - rd.y), w2);
      } else if (p == 5) {
        const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
        const double s1 = 0.95105651629515357212 * (SIGN < 0 ? 1.0 : -1.0);
        const double s2 = 0.58778525229247312917 * (SIGN < 0 ? 1.0 : -1.0);
        const double2 a0 = base[0], a1 = base[span], a2 = base[2 * span], a3 = base[3 * span], a4 = base[4 * span];
        const double2 b1 = make_double2(a1.x + a4.x, a1.y + a4.y), b2 = make_double2(a2.x + a3.x, a2.y + a3.y);
        const double2 d1 = make_double2(a1.x - a4.x, a1.y - a4.y), d2 = make_double2(a2.x - a3.x, a2.y - a3.y);
        const double2 r1 = make_double2(a0.x + c1 * b1.x + c2 * b2.x, a0.y + c1 * b1.y + c2 * b2.y);
        const double2 r2 = make_double2(a0.x + c2 * b1.x + c1 * b2.x, a0.y + c2 * b1.y + c1 * b2.y);
        const double2 e1 = make_double2(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y);
        const double2 e2 = make_double2(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y);
        // -i e = (e.y, -e.x)
        double2 w1 = P.tw[j * tstep], w2 = P.tw[2 * j * tstep], w3 = P.tw[3 * j * tstep], w4 = P.tw[4 * j * tstep];
        if (SIGN > 0) { w1.y = -w1.y; w2.y = -w2.y; w3.y = -w3.y; w4.y = -w4.y; }
        base[0] = make_double2(a0.x + b1.x + b2.x, a0.y + b1.y + b2.y);
        base[span] = cmul(make_double2(r1.x + e1.y, r1.y - e1.x), w1);
        base[4 * span] = cmul(make_double2(r1.x - e1.y, r1.y + e1.x), w4);
        base[2 * span] = cmul(make_double2(r2.x + e2.y, r2.y - e2.x), w2);
        base[3 * span] = cmul(make_double2(r2.x - e2.y, r2.y + e2.x), w3);
      } else {
        fft_generic_bfly<SIGN>(base, span, p, j, tstep, P);
      }
    }
    __syncthreads();
    len = span;
  }
}

__device__ __forceinline__ int fft_pos(int k, const FftPlan& P) {
  int pos = 0, len = P.n;
  for (int s = 0; s < P.stages; ++s) {
    const int p = P.radix[s];
    len /= p;
    pos += (k % p) * len;
    k /= p;
  }
  return pos;
}

// Ring stages work on one latitude ring of R consecutive snapshots per CTA, so
// the staging G[m][i][s] (s = 2 t + {re, im} contiguous) is written and read
// in runs of 2R doubles per (m, i).
//
// Forward ring stage (sht.cpp:211-222): fields (T, n_theta, n_phi) ->
// G[m][i][s] scaled by 1/n_phi. grid (n_theta, ceil(T / R)).
__global__ void k_ring_fft_fwd(const double* __restrict__ fields, int n_theta, int L, int R, FftPlan P,
                               int T, double* __restrict__ G) {
  extern __shared__ double2 xs[];
  const int n = P.n;
  const int i = blockIdx.x, t0 = blockIdx.y * R;
  const int nr = min(R, T - t0);
  for (int e = threadIdx.x; e < nr * n; e += blockDim.x) {
    const int r = e / n, j = e - r * n;
    xs[e] = make_double2(fields[((int64_t)(t0 + r) * n_theta + i) * n + j], 0.0);
  }
  __syncthreads();
  fft_dif_rings<-1>(xs, nr, P);
  const double inv = 1.0 / n;
  const int ntp = (n_theta + 1) & ~1;
  const int64_t mstride = (int64_t)ntp * 2 * T;
  double* g = G + (int64_t)i * 2 * T + 2 * t0;
  for (int e = threadIdx.x; e < L * 2 * nr; e += blockDim.x) {
    const int m = e / (2 * nr), q = e - m * 2 * nr;  // q = 2 r + c
    const double2 v = xs[(q >> 1) * n + fft_pos(m, P)];
    g[m * mstride + q] = ((q & 1) ? v.y : v.x) * inv;
  }
}

// Inverse ring stage (sht.cpp:345-356): Hermitian fill, unnormalized
// synthesis, real part. G[m][i][s] -> fields (T, n_theta, n_phi).
__global__ void k_ring_fft_inv(const double* __restrict__ G, int n_theta, int L, int R, FftPlan P, int T,
                               double* __restrict__ fields) {
  extern __shared__ double2 xs[];
  const int n = P.n;
  const int i = blockIdx.x, t0 = blockIdx.y * R;
  const int nr = min(R, T - t0);
  const int ntp = (n_theta + 1) & ~1;
  const int64_t mstride = (int64_t)ntp * 2 * T;
  const double* g = G + (int64_t)i * 2 * T + 2 * t0;
  for (int e = threadIdx.x; e < nr * n; e += blockDim.x) xs[e] = make_double2(0.0, 0.0);
  __syncthreads();
  for (int e = threadIdx.x; e < L * nr; e += blockDim.x) {
    const int m = e / nr, r = e - m * nr;
    const double2 z = *reinterpret_cast<const double2*>(g + m * mstride + 2 * r);
    if (m == 0) {
      xs[r * n] = z;
    } else {
      xs[r * n + m] = z;
      xs[r * n + n - m] = make_double2(z.x, -z.y);
    }
  }
  __syncthreads();
  fft_dif_rings<+1>(xs, nr, P);
  for (int e = threadIdx.x; e < nr * n; e += blockDim.x) {
    const int r = e / n, j = e - r * n;
    fields[((int64_t)(t0 + r) * n_theta + i) * n + j] = xs[r * n + fft_pos(j, P)].x;
  }
}

// Real-input rings (n_phi even): a ring of n reals is one complex FFT of
// N = n / 2 points on z_j = x_2j + i x_2j+1, then
//   X_m = E_m + w^m O_m,  E_m = (Z_m + conj Z_{N-m}) / 2,  O_m = (Z_m - conj Z_{N-m}) / 2i
// (w = exp(-2 pi i / n)); synthesis builds Z'_k = (X_k + conj X_{N-k}) +
// i w^-k (X_k - conj X_{N-k}) and one inverse FFT of N points yields
// x_2j + i x_2j+1. Half the butterflies and half the shared memory of the
// complex path.
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

__global__ void k_ring_rfft_fwd(const double* __restrict__ fields, int n_theta, int L, int R, FftPlan H,
                                const double2* __restrict__ twn, int T, double* __restrict__ G) {
  extern __shared__ double2 xs[];
  const int N = H.n;
  const int i = blockIdx.x, t0 = blockIdx.y * R;
  const int nr = min(R, T - t0);
  for (int e = threadIdx.x; e < nr * N; e += blockDim.x) {
    const int r = e / N, j = e - r * N;
    xs[e] = reinterpret_cast<const double2*>(fields + ((int64_t)(t0 + r) * n_theta + i) * 2 * N)[j];
  }
  __syncthreads();
  fft_dif_rings<-1>(xs, nr, H);
  const double inv = 0.5 / (2 * N);  // the 1/2 of E and O folded into the 1/n_phi scaling
  const int ntp = (n_theta + 1) & ~1;
  const int64_t mstride = (int64_t)ntp * 2 * T;
  double* g = G + (int64_t)i * 2 * T + 2 * t0;
  for (int e = threadIdx.x; e < L * nr; e += blockDim.x) {
    const int m = e / nr, r = e - m * nr;
    const double2 zk = xs[r * N + fft_pos(m, H)];
    const double2 zc = cconj(xs[r * N + fft_pos(m == 0 ? 0 : N - m, H)]);
    const double2 e2 = make_double2(zk.x + zc.x, zk.y + zc.y);                 // 2 E
    const double2 d = make_double2(zk.x - zc.x, zk.y - zc.y);
    const double2 o2 = make_double2(d.y, -d.x);                                // 2 O = -i d
    const double2 wo = cmul(twn[m], o2);
    *reinterpret_cast<double2*>(g + m * mstride + 2 * r) = make_double2((e2.x + wo.x) * inv, (e2.y + wo.y) * inv);
  }
}

__global__ void k_ring_rfft_inv(const double* __restrict__ G, int n_theta, int L, int R, FftPlan H,
                                const double2* __restrict__ twn, int T, double* __restrict__ fields) {
  extern __shared__ double2 xs[];
  const int N = H.n;
  const int i = blockIdx.x, t0 = blockIdx.y * R;
  const int nr = min(R, T - t0);
  const int ntp = (n_theta + 1) & ~1;
  const int64_t mstride = (int64_t)ntp * 2 * T;
  const double* g = G + (int64_t)i * 2 * T + 2 * t0;
  for (int e = threadIdx.x; e < nr * N; e += blockDim.x) {
    const int r = e / N, k = e - r * N;
    const double2 xk = k < L ? *reinterpret_cast<const double2*>(g + k * mstride + 2 * r) : make_double2(0.0, 0.0);
    const int km = N - k;  // k = 0 -> X_N = 0 (L <= N)
    const double2 xm = km < L ? cconj(*reinterpret_cast<const double2*>(g + km * mstride + 2 * r)) : make_double2(0.0, 0.0);
    const double2 a = make_double2(xk.x + xm.x, xk.y + xm.y);
    const double2 bv = make_double2(xk.x - xm.x, xk.y - xm.y);
    const double2 wb = cmul(cconj(twn[k]), bv);
    xs[r * N + k] = make_double2(a.x - wb.y, a.y + wb.x);  // a + i (w^-k b)
  }
  __syncthreads();
  fft_dif_rings<+1>(xs, nr, H);
  for (int e = threadIdx.x; e < nr * N; e += blockDim.x) {
    const int r = e / N, j = e - r * N;
    reinterpret_cast<double2*>(fields + ((int64_t)(t0 + r) * n_theta + i) * 2 * N)[j] = xs[r * N + fft_pos(j, H)];
  }
}

// ===========================================================================
// Device: Legendre stages (grouped FP64 GEMMs over m)
// ===========================================================================
// Forward: F_m (L-m x 2T) = Psi_m (L-m x n_theta) * G_m^T; scattered into the
// packed layout (sht.hpp:38-45): m = 0 keeps the real part only.
__global__ void __launch_bounds__(D2_THREADS) k_legendre_fwd(const double* __restrict__ psi,
                                                              const int64_t* psi_off, const double* __restrict__ G,
                                                              int L, int n_theta, int T, double* coeffs) {
  extern __shared__ __align__(16) uint8_t d2_smem[];
  D2Smem& sm = *reinterpret_cast<D2Smem*>(d2_smem);
  const int m = blockIdx.z;
  const int rows = L - m;
  const int r0 = blockIdx.y * D2_BM, c0 = blockIdx.x * D2_BN;
  if (r0 >= rows) return;
  const int ncols = 2 * T;
  const int ntp = (n_theta + 1) & ~1;  // Psi rows padded with a zero column to an even stride: 16-byte cp.async
  D2Op A{psi + psi_off[m] + (int64_t)r0 * ntp, ntp, min(D2_BM, rows - r0), ntp};
  D2Op B{G + (int64_t)m * ntp * ncols + c0, ncols, ntp, min(D2_BN, ncols - c0)};  // G_m[i][s], K = i
  double acc[4][4][2];
  dgemm2_128x64<D2B::kNN, true>(A, B, ntp, sm, acc);
  const int64_t nc = (int64_t)L * L;
  d2_for_each(acc, [&](int r, int c, double v0, double v1) {
    const int l = m + r0 + r, s = c0 + c;  // s even: (re, im) of snapshot s/2
    if (r0 + r >= rows || s >= ncols) return;
    const int t = s >> 1;
    if (m == 0) {
      coeffs[(int64_t)t * nc + (int64_t)l * l] = v0;
    } else {
      double2* q = reinterpret_cast<double2*>(coeffs + (int64_t)t * nc + (int64_t)l * l + 2 * m - 1);
      // l*l + 2m - 1 is even when l*l is odd; use scalar stores to stay aligned-agnostic
      double* qq = reinterpret_cast<double*>(q);
      qq[0] = v0;
      qq[1] = v1;
    }
  });
}

// Z[m][s][l - m] from packed coefficients (m = 0 imaginary part is zero).
__global__ void k_gather_z(const double* __restrict__ coeffs, int L, int T, const int64_t* z_off, double* Z) {
  const int m = blockIdx.y;
  const int s = blockIdx.x;
  const int t = s >> 1, part = s & 1;
  const int cols = L - m;
  const int colsp = (cols + 1) & ~1;
  const int64_t nc = (int64_t)L * L;
  double* dst = Z + z_off[m] * 2 * T + (int64_t)s * colsp;
  for (int r = threadIdx.x; r < cols; r += blockDim.x) {
    const int l = m + r;
    double v;
    if (m == 0) v = part ? 0.0 : coeffs[(int64_t)t * nc + (int64_t)l * l];
    else v = coeffs[(int64_t)t * nc + (int64_t)l * l + 2 * m - 1 + part];
    dst[r] = v;
  }
}

// Inverse: G_m^T (2T x n_theta) = Z_m (2T x L-m) * Y_m^T, G[m][s][i].
__global__ void __launch_bounds__(D2_THREADS) k_legendre_inv(const double* __restrict__ y, const int64_t* y_off,
                                                              const double* __restrict__ Z, const int64_t* z_off,
                                                              int L, int n_theta, int T, double* G) {
  // G_m[i][s] (n_theta x 2T) = Y_m (n_theta x L-m) * Z_m^T, Z_m[s][l - m].
  extern __shared__ __align__(16) uint8_t d2_smem[];
  D2Smem& sm = *reinterpret_cast<D2Smem*>(d2_smem);
  const int m = blockIdx.z;
  const int cols = L - m;
  const int ncols = 2 * T;
  const int r0 = blockIdx.y * D2_BM, c0 = blockIdx.x * D2_BN;
  if (r0 >= n_theta) return;
  const int colsp = (cols + 1) & ~1, ntp = (n_theta + 1) & ~1;
  D2Op A{y + y_off[m] + (int64_t)r0 * colsp, colsp, min(D2_BM, n_theta - r0), colsp};
  D2Op B{Z + z_off[m] * ncols + (int64_t)c0 * colsp, colsp, min(D2_BN, ncols - c0), colsp};
  double acc[4][4][2];
  dgemm2_128x64<D2B::kNT, true>(A, B, colsp, sm, acc);
  double* out = G + (int64_t)m * ntp * ncols;
  d2_for_each(acc, [&](int r, int c, double v0, double v1) {
    if (r0 + r >= n_theta || c0 + c >= ncols) return;  // ncols even, c even: the pair is in range
    *reinterpret_cast<double2*>(out + (int64_t)(r0 + r) * ncols + c0 + c) = make_double2(v0, v1);
  });
}

// ===========================================================================
// Host plan
// ===========================================================================
struct Sht {
  int n_theta = 0, n_phi = 0, L = 0;
  cudaStream_t stream = nullptr;
  DevBuf<double> psi, y;
  DevBuf<int64_t> d_psi_off, d_y_off, d_z_off;
  std::vector<int64_t> psi_off, y_off, z_off;
  DevBuf<double2> tw_phi, tw_half;
  FftPlan fplan{}, hplan{};
  bool real_rings = false;
  int rings_per_cta = 1;
  size_t fft_smem = 0;
  int chunk = 64;
  DevBuf<double> G, Z, fields_buf, coeffs_buf;
  double plan_seconds = 0.0;

  Sht(int nt, int np, int L_, size_t cap) : n_theta(nt), n_phi(np), L(L_) {
    auto t0 = std::chrono::steady_clock::now();
    if (n_theta < 2) throw std::invalid_argument("grid needs at least two latitude rings");
    if (n_phi < 1) throw std::invalid_argument("grid needs at least one longitude point");
    const int maxL = std::min(n_theta - 1, (n_phi + 1) / 2);
    if (L < 1 || L > maxL)
      throw std::invalid_argument("grid " + std::to_string(n_theta) + "x" + std::to_string(n_phi) +
                                  " does not resolve band limit " + std::to_string(L));
    check_wigner_cap(L, cap ? cap : (size_t{2} << 30));  // before any CUDA call
    SPH_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    WignerDev wigner;  // freed once the operators below are built
    build_wigner_device(wigner, L, cap ? cap : (size_t{2} << 30), stream);
    // Offsets of the per-m operators.
    psi_off.resize(L + 1);
    y_off.resize(L + 1);
    z_off.resize(L + 1);
    // Per-m operators with even row strides (zero padding), so every
    // operand row of the Legendre GEMMs starts 16-byte aligned.
    const int64_t ntp = (n_theta + 1) & ~1;
    int64_t po = 0, yo = 0, zo = 0;
    for (int m = 0; m < L; ++m) {
      psi_off[m] = po;
      y_off[m] = yo;
      z_off[m] = zo;
      const int64_t colsp = (L - m + 1) & ~1;
      po += (int64_t)(L - m) * ntp;
      yo += (int64_t)n_theta * colsp;
      zo += colsp;
    }
    psi_off[L] = po;
    y_off[L] = yo;
    z_off[L] = zo;
    psi.alloc(po);
    y.alloc(yo);
    SPH_CUDA(cudaMemsetAsync(psi.get(), 0, sizeof(double) * po, stream));
    SPH_CUDA(cudaMemsetAsync(y.get(), 0, sizeof(double) * yo, stream));
    d_psi_off.alloc(L + 1);
    d_y_off.alloc(L + 1);
    d_z_off.alloc(L + 1);
    SPH_CUDA(cudaMemcpy(d_psi_off.get(), psi_off.data(), (L + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    SPH_CUDA(cudaMemcpy(d_y_off.get(), y_off.data(), (L + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    SPH_CUDA(cudaMemcpy(d_z_off.get(), z_off.data(), (L + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    const double* dd_p = wigner.d.get();
    const int64_t* doff_p = wigner.off.get();
    // Twiddles of the extended line and the T_+/- tables (host, exact angles).
    const int n_ext = 2 * n_theta - 2;
    std::vector<double2> tw_ext(n_ext);
    for (int t = 0; t < n_ext; ++t) {
      const double a = 2.0 * M_PI * t / n_ext;
      tw_ext[t] = make_double2(std::cos(a), -std::sin(a));
    }
    std::vector<double> tcos((size_t)L * n_theta), tsin((size_t)L * n_theta);
    for (int mp = 0; mp < L; ++mp)
      for (int i = 0; i < n_theta; ++i) {
        const int64_t tt = ((int64_t)mp * i) % n_ext;
        const double a = 2.0 * M_PI * tt / n_ext;
        tcos[(size_t)mp * n_theta + i] = mp == 0 ? 1.0 : 2.0 * std::cos(a);
        tsin[(size_t)mp * n_theta + i] = mp == 0 ? 0.0 : 2.0 * std::sin(a);
      }
    DevBuf<double2> dtw(n_ext);
    DevBuf<double> dtc(tcos.size()), dts(tsin.size()), vre((size_t)L * n_theta), vim((size_t)L * n_theta);
    SPH_CUDA(cudaMemcpy(dtw.get(), tw_ext.data(), n_ext * sizeof(double2), cudaMemcpyHostToDevice));
    SPH_CUDA(cudaMemcpy(dtc.get(), tcos.data(), tcos.size() * sizeof(double), cudaMemcpyHostToDevice));
    SPH_CUDA(cudaMemcpy(dts.get(), tsin.data(), tsin.size() * sizeof(double), cudaMemcpyHostToDevice));
    k_sht_vtables<<<dim3(ceil_div(n_theta, 128), L), 128, 0, stream>>>(L, n_theta, dtw.get(), vre.get(), vim.get());
    SPH_LAUNCH_CHECK();
    k_sht_build_psi<<<dim3(ceil_div(n_theta, DG_BN), ceil_div(L, DG_BM), L), DG_THREADS, 0, stream>>>(
        dd_p, doff_p, L, n_theta, vre.get(), vim.get(), d_psi_off.get(), psi.get());
    SPH_LAUNCH_CHECK();
    k_sht_build_y<<<dim3(ceil_div(n_theta, DG_BM), ceil_div(L, DG_BN), L), DG_THREADS, 0, stream>>>(
        dd_p, doff_p, L, n_theta, dtc.get(), dts.get(), d_y_off.get(), y.get());
    SPH_LAUNCH_CHECK();
    // Ring FFT plan.
    fplan.n = n_phi;
    fplan.stages = 0;
    int rem = n_phi;
    auto push = [&](int p) {
      if (fplan.stages >= FFT_MAX_STAGES) throw std::invalid_argument("n_phi has too many factors");
      fplan.radix[fplan.stages++] = p;
    };
    while (rem % 4 == 0) { push(4); rem /= 4; }
    while (rem % 2 == 0) { push(2); rem /= 2; }
    for (int p = 3; rem > 1; p += 2)
      while (rem % p == 0) { push(p); rem /= p; }
    for (int s = 0; s < fplan.stages; ++s)
      if (fplan.radix[s] > 64)
        throw std::invalid_argument("n_phi has a prime factor above 64 (" + std::to_string(fplan.radix[s]) + ")");
    std::vector<double2> twp(n_phi);
    for (int t = 0; t < n_phi; ++t) {
      const double a = 2.0 * M_PI * t / n_phi;
      twp[t] = make_double2(std::cos(a), -std::sin(a));
    }
    tw_phi.alloc(n_phi);
    SPH_CUDA(cudaMemcpy(tw_phi.get(), twp.data(), n_phi * sizeof(double2), cudaMemcpyHostToDevice));
    fplan.tw = tw_phi.get();
    // Half-length plan for real rings (n_phi even and L <= n_phi / 2).
    real_rings = (n_phi % 2 == 0) && L <= n_phi / 2 && !(std::getenv("SPHEMU_SHT_COMPLEX_RINGS"));
    if (real_rings) {
      const int N = n_phi / 2;
      hplan.n = N;
      hplan.stages = 0;
      int r2 = N;
      auto hpush = [&](int p) { hplan.radix[hplan.stages++] = p; };
      while (r2 % 4 == 0) { hpush(4); r2 /= 4; }
      while (r2 % 2 == 0) { hpush(2); r2 /= 2; }
      for (int p = 3; r2 > 1; p += 2)
        while (r2 % p == 0) { hpush(p); r2 /= p; }
      std::vector<double2> twh(N);
      for (int t = 0; t < N; ++t) {
        const double a = 2.0 * M_PI * t / N;
        twh[t] = make_double2(std::cos(a), -std::sin(a));
      }
      tw_half.alloc(N);
      SPH_CUDA(cudaMemcpy(tw_half.get(), twh.data(), N * sizeof(double2), cudaMemcpyHostToDevice));
      hplan.tw = tw_half.get();
    }
    // snapshots per FFT CTA: runs of >= 64 bytes per (m, ring) in G, within ~200 KB of smem
    {
      const char* e = std::getenv("SPHEMU_FFT_R");
      const int cap = e ? std::max(1, std::atoi(e)) : 16;
      // ~48 KB of rings per CTA (measured best for n_phi = 360 and 1440)
      const int pts_ring = real_rings ? n_phi / 2 : n_phi;
      rings_per_cta = std::max(1, std::min(cap, (48 * 1024) / (16 * pts_ring)));
    }
    fft_smem = (size_t)rings_per_cta * (real_rings ? n_phi / 2 : n_phi) * sizeof(double2);
    if (fft_smem > 48 * 1024) {
      SPH_CUDA(cudaFuncSetAttribute(k_ring_fft_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fft_smem));
      SPH_CUDA(cudaFuncSetAttribute(k_ring_fft_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fft_smem));
      SPH_CUDA(cudaFuncSetAttribute(k_ring_rfft_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fft_smem));
      SPH_CUDA(cudaFuncSetAttribute(k_ring_rfft_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fft_smem));
    }
    SPH_CUDA(cudaFuncSetAttribute(k_legendre_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(D2Smem)));
    SPH_CUDA(cudaFuncSetAttribute(k_legendre_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(D2Smem)));
    // Snapshot chunk: bound the G staging to ~1 GiB.
    const double per = 16.0 * L * n_theta + 16.0 * L * L;
    chunk = (int)std::max(1.0, std::min(1024.0, (1024.0 * 1024 * 1024) / per));
    SPH_CUDA(cudaStreamSynchronize(stream));
    plan_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }

  ~Sht() {
    if (stream) {
      cudaStreamSynchronize(stream);
      cudaStreamDestroy(stream);
    }
    for (auto st : {hcs, hds})
      if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
      }
    for (int r = 0; r < kRing; ++r)
      for (auto e : {ev_h2d[r], ev_comp[r], ev_d2h[r]})
        if (e) cudaEventDestroy(e);
  }

  // ---- host-buffer batches (the 8 760-snapshot year of C4) ----------------
  // Chunks of hchunk snapshots stream through a ring of kRing pinned + device
  // slots: host threads copy the caller's (pageable) array into the pinned
  // slot, H2D on hcs, the transform on `stream`, D2H on hds, and the host
  // drains chunk c-1 while the GPU works on chunk c; pinned memory is kept
  // (grow-only) for the next call.
  static constexpr int kRing = 3;
  cudaStream_t hcs = nullptr, hds = nullptr;
  cudaEvent_t ev_h2d[kRing] = {}, ev_comp[kRing] = {}, ev_d2h[kRing] = {};
  PinnedBuf pin_in, pin_out;
  DevBuf<double> ring_in, ring_out;
  std::unique_ptr<HostPool> hpool;

  void run_host(bool fwd, const double* in, int win, int64_t n, double* out, int wout) {
    const int64_t pts = (int64_t)n_theta * n_phi, nc = (int64_t)L * L;
    const int64_t isz = fwd ? pts : nc, osz = fwd ? nc : pts;
    const bool hin = win == SPHEMU_HOST, hout = wout == SPHEMU_HOST;
    const int64_t T = std::max<int64_t>(1, std::min<int64_t>(chunk, (int64_t{512} << 20) / (8 * std::max(isz, osz))));
    const int64_t nch = (n + T - 1) / T;
    if (!hcs) {
      SPH_CUDA(cudaStreamCreateWithFlags(&hcs, cudaStreamNonBlocking));
      SPH_CUDA(cudaStreamCreateWithFlags(&hds, cudaStreamNonBlocking));
      for (int r = 0; r < kRing; ++r) {
        SPH_CUDA(cudaEventCreateWithFlags(&ev_h2d[r], cudaEventDisableTiming));
        SPH_CUDA(cudaEventCreateWithFlags(&ev_comp[r], cudaEventDisableTiming));
        SPH_CUDA(cudaEventCreateWithFlags(&ev_d2h[r], cudaEventDisableTiming));
      }
      const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
      hpool.reset(new HostPool(static_cast<int>(std::min(16u, hw))));
    }
    const size_t in_b = (size_t)T * isz * sizeof(double), out_b = (size_t)T * osz * sizeof(double);
    if (hin) {
      pin_in.ensure(kRing * in_b);
      if (ring_in.n < (size_t)kRing * T * isz) ring_in.alloc((size_t)kRing * T * isz);
    }
    if (hout) {
      pin_out.ensure(kRing * out_b);
      if (ring_out.n < (size_t)kRing * T * osz) ring_out.alloc((size_t)kRing * T * osz);
    }
    auto host_copy = [&](char* dst, const char* src, size_t bytes) {
      hpool->run([&](int t, int nt) {
        const size_t per = (bytes / nt + 4095) & ~size_t{4095};
        const size_t a = std::min(bytes, per * t), b = std::min(bytes, a + per);
        if (b > a) std::memcpy(dst + a, src + a, b - a);
      });
    };
    auto drain = [&](int64_t c) {
      const int slot = static_cast<int>(c % kRing);
      const int64_t Tc = std::min(T, n - c * T);
      SPH_CUDA(cudaEventSynchronize(ev_d2h[slot]));
      host_copy(reinterpret_cast<char*>(out + c * T * osz), pin_out.p + slot * out_b, (size_t)Tc * osz * 8);
    };
    for (int64_t c = 0; c < nch; ++c) {
      const int slot = static_cast<int>(c % kRing);
      const int64_t Tc = std::min(T, n - c * T);
      const double* src = in + c * T * isz;
      if (hin) {
        SPH_CUDA(cudaEventSynchronize(ev_h2d[slot]));  // the slot's previous H2D has read the pinned copy
        host_copy(pin_in.p + slot * in_b, reinterpret_cast<const char*>(src), (size_t)Tc * isz * 8);
        double* d = ring_in.get() + (size_t)slot * T * isz;
        SPH_CUDA(cudaStreamWaitEvent(hcs, ev_comp[slot], 0));  // the slot's previous transform has read it
        SPH_CUDA(cudaMemcpyAsync(d, pin_in.p + slot * in_b, (size_t)Tc * isz * 8, cudaMemcpyHostToDevice, hcs));
        SPH_CUDA(cudaEventRecord(ev_h2d[slot], hcs));
        SPH_CUDA(cudaStreamWaitEvent(stream, ev_h2d[slot], 0));
        src = d;
      }
      double* dst = hout ? ring_out.get() + (size_t)slot * T * osz : out + c * T * osz;
      if (hout) SPH_CUDA(cudaStreamWaitEvent(stream, ev_d2h[slot], 0));  // the slot's previous D2H is done
      if (fwd) forward_dev(src, Tc, dst);
      else inverse_dev(src, Tc, dst);
      SPH_CUDA(cudaEventRecord(ev_comp[slot], stream));
      if (hout) {
        SPH_CUDA(cudaStreamWaitEvent(hds, ev_comp[slot], 0));
        SPH_CUDA(cudaMemcpyAsync(pin_out.p + slot * out_b, dst, (size_t)Tc * osz * 8, cudaMemcpyDeviceToHost, hds));
        SPH_CUDA(cudaEventRecord(ev_d2h[slot], hds));
      }
      if (hout && c >= 1) drain(c - 1);
    }
    if (hout && nch >= 1) drain(nch - 1);
    SPH_CUDA(cudaStreamSynchronize(stream));
    SPH_CUDA(cudaStreamSynchronize(hcs));
    SPH_CUDA(cudaStreamSynchronize(hds));
  }

  void ensure(int64_t tchunk) {
    const size_t g = (size_t)L * 2 * tchunk * ((n_theta + 1) & ~1);
    if (G.n < g) {  // zero: the padding column is never written
      G.alloc(g);
      SPH_CUDA(cudaMemsetAsync(G.get(), 0, sizeof(double) * g, stream));
    }
    const size_t z = (size_t)z_off[L] * 2 * tchunk;
    if (Z.n < z) {
      Z.alloc(z);
      SPH_CUDA(cudaMemsetAsync(Z.get(), 0, sizeof(double) * z, stream));
    }
  }

  // Device-resident batched transforms.
  void forward_dev(const double* fields, int64_t n, double* coeffs) {
    const int64_t pts = (int64_t)n_theta * n_phi, nc = (int64_t)L * L;
    for (int64_t t0 = 0; t0 < n; t0 += chunk) {
      const int T = (int)std::min<int64_t>(chunk, n - t0);
      ensure(T);
      if (real_rings)
        k_ring_rfft_fwd<<<dim3(n_theta, ceil_div(T, rings_per_cta)), 256, fft_smem, stream>>>(
            fields + t0 * pts, n_theta, L, rings_per_cta, hplan, tw_phi.get(), T, G.get());
      else
        k_ring_fft_fwd<<<dim3(n_theta, ceil_div(T, rings_per_cta)), 256, fft_smem, stream>>>(
            fields + t0 * pts, n_theta, L, rings_per_cta, fplan, T, G.get());
      SPH_LAUNCH_CHECK();
      k_legendre_fwd<<<dim3(ceil_div(2 * T, D2_BN), ceil_div(L, D2_BM), L), D2_THREADS, sizeof(D2Smem), stream>>>(
          psi.get(), d_psi_off.get(), G.get(), L, n_theta, T, coeffs + t0 * nc);
      SPH_LAUNCH_CHECK();
    }
  }

  void inverse_dev(const double* coeffs, int64_t n, double* fields) {
    const int64_t pts = (int64_t)n_theta * n_phi, nc = (int64_t)L * L;
    for (int64_t t0 = 0; t0 < n; t0 += chunk) {
      const int T = (int)std::min<int64_t>(chunk, n - t0);
      ensure(T);
      k_gather_z<<<dim3(2 * T, L), 128, 0, stream>>>(coeffs + t0 * nc, L, T, d_z_off.get(), Z.get());
      SPH_LAUNCH_CHECK();
      k_legendre_inv<<<dim3(ceil_div(2 * T, D2_BN), ceil_div(n_theta, D2_BM), L), D2_THREADS, sizeof(D2Smem), stream>>>(
          y.get(), d_y_off.get(), Z.get(), d_z_off.get(), L, n_theta, T, G.get());
      SPH_LAUNCH_CHECK();
      if (real_rings)
        k_ring_rfft_inv<<<dim3(n_theta, ceil_div(T, rings_per_cta)), 256, fft_smem, stream>>>(
            G.get(), n_theta, L, rings_per_cta, hplan, tw_phi.get(), T, fields + t0 * pts);
      else
        k_ring_fft_inv<<<dim3(n_theta, ceil_div(T, rings_per_cta)), 256, fft_smem, stream>>>(
            G.get(), n_theta, L, rings_per_cta, fplan, T, fields + t0 * pts);
      SPH_LAUNCH_CHECK();
    }
  }

  void forward(const double* in, int win, int64_t n, double* out, int wout) {
    if (n <= 0) return;
    if (win == SPHEMU_DEVICE && wout == SPHEMU_DEVICE) {
      forward_dev(in, n, out);
      SPH_CUDA(cudaStreamSynchronize(stream));
      return;
    }
    run_host(true, in, win, n, out, wout);
  }

  void inverse(const double* in, int win, int64_t n, double* out, int wout) {
    if (n <= 0) return;
    if (win == SPHEMU_DEVICE && wout == SPHEMU_DEVICE) {
      inverse_dev(in, n, out);
      SPH_CUDA(cudaStreamSynchronize(stream));
      return;
    }
    run_host(false, in, win, n, out, wout);
  }
};

}  // namespace sphemu_gpu

using namespace sphemu_gpu;

struct sphemu_sht_s {
  Sht* p;
};

namespace sphemu_gpu {
void emulate(void* plan, int n_theta, int n_phi, int L, const double* v, int d, const double* phi, int order,
             const double* means, const double* sigma, const double* v2, int t_out, uint64_t seed, int r_len,
             int rng_mode, double* out, int r_begin, const TrendArgs* trend = nullptr);

void sht_plan_dims(void* plan, int* n_theta, int* n_phi, int* L) {
  Sht* p = static_cast<sphemu_sht_s*>(plan)->p;
  *n_theta = p->n_theta;
  *n_phi = p->n_phi;
  *L = p->L;
}

// Bridge for emulate.cu: the plan's stream, and a device-resident inverse.
void sht_inverse_device(void* plan, const double* coeffs, int64_t n, double* fields, cudaStream_t* s_out) {
  Sht* p = static_cast<sphemu_sht_s*>(plan)->p;
  if (s_out) *s_out = p->stream;
  if (n > 0) p->inverse_dev(coeffs, n, fields);
}
}  // namespace sphemu_gpu

extern "C" {

int sphemu_gpu_sht_create(int n_theta, int n_phi, int band_limit, size_t wigner_cap_bytes, sphemu_sht_t* out) {
  return guard([&] {
    *out = nullptr;
    auto* h = new sphemu_sht_s{nullptr};
    try {
      h->p = new Sht(n_theta, n_phi, band_limit, wigner_cap_bytes);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int sphemu_gpu_sht_destroy(sphemu_sht_t p) {
  return guard([&] {
    if (!p) return;
    delete p->p;
    delete p;
  });
}

int sphemu_gpu_sht_forward(sphemu_sht_t p, const double* fields, int where_in, int64_t n, double* coeffs,
                           int where_out) {
  return guard([&] { p->p->forward(fields, where_in, n, coeffs, where_out); });
}

int sphemu_gpu_sht_inverse(sphemu_sht_t p, const double* coeffs, int where_in, int64_t n, double* fields,
                           int where_out) {
  return guard([&] { p->p->inverse(coeffs, where_in, n, fields, where_out); });
}

void* sphemu_gpu_sht_stream(sphemu_sht_t p) { return p ? p->p->stream : nullptr; }
double sphemu_gpu_sht_plan_seconds(sphemu_sht_t p) { return p ? p->p->plan_seconds : 0.0; }

int sphemu_gpu_wigner_d_half_pi(int band_limit, size_t wigner_cap_bytes, int64_t n, const int* l, const int* m2,
                                const int* m, double* out, int* renorm_warnings) {
  return guard([&] {
    using namespace sphemu_gpu;
    if (n < 0) throw std::invalid_argument("negative entry count");
    for (int64_t i = 0; i < n; ++i)
      if (l[i] < 0 || l[i] >= band_limit) throw std::invalid_argument("degree outside the table");
    const size_t cap = wigner_cap_bytes ? wigner_cap_bytes : (size_t{2} << 30);
    check_wigner_cap(band_limit, cap);
    cudaStream_t s = nullptr;
    SPH_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    } sg{s};
    WignerDev w;
    build_wigner_device(w, band_limit, cap, s);
    if (renorm_warnings) *renorm_warnings = w.renorm;
    if (n == 0) return;
    DevBuf<int> idx((size_t)n * 3);
    DevBuf<double> dout((size_t)n);
    SPH_CUDA(cudaMemcpyAsync(idx.get(), l, n * sizeof(int), cudaMemcpyHostToDevice, s));
    SPH_CUDA(cudaMemcpyAsync(idx.get() + n, m2, n * sizeof(int), cudaMemcpyHostToDevice, s));
    SPH_CUDA(cudaMemcpyAsync(idx.get() + 2 * n, m, n * sizeof(int), cudaMemcpyHostToDevice, s));
    k_wigner_gather<<<(unsigned)ceil_div(n, (int64_t)256), 256, 0, s>>>(band_limit, w.off.get(), w.d.get(), n,
                                                                         idx.get(), idx.get() + n, idx.get() + 2 * n,
                                                                         dout.get());
    SPH_LAUNCH_CHECK();
    SPH_CUDA(cudaMemcpyAsync(out, dout.get(), n * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPH_CUDA(cudaStreamSynchronize(s));
  });
}

int sphemu_gpu_wigner_tables(int band_limit, size_t wigner_cap_bytes, int64_t* offsets, double* d, int64_t d_count,
                             int* renorm_warnings) {
  return guard([&] {
    using namespace sphemu_gpu;
    const size_t cap = wigner_cap_bytes ? wigner_cap_bytes : (size_t{2} << 30);
    check_wigner_cap(band_limit, cap);
    cudaStream_t s = nullptr;
    SPH_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    } sg{s};
    WignerDev w;
    build_wigner_device(w, band_limit, cap, s);
    const size_t n_off = static_cast<size_t>(band_limit) * band_limit + 1;
    std::vector<int64_t> off(n_off);
    SPH_CUDA(cudaMemcpyAsync(off.data(), w.off.get(), n_off * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPH_CUDA(cudaStreamSynchronize(s));
    if (d_count != off.back()) throw std::invalid_argument("d buffer size does not match the table");
    std::copy(off.begin(), off.end(), offsets);
    SPH_CUDA(cudaMemcpyAsync(d, w.d.get(), static_cast<size_t>(d_count) * sizeof(double), cudaMemcpyDeviceToHost, s));
    SPH_CUDA(cudaStreamSynchronize(s));
    if (renorm_warnings) *renorm_warnings = w.renorm;
  });
}

int sphemu_gpu_emulate(sphemu_sht_t p, const double* v, int d, const double* phi, int order, const double* means,
                       const double* sigma, const double* v2, int t_out, uint64_t seed, int r_len, int rng_mode,
                       double* out) {
  return guard([&] {
    emulate(p, p->p->n_theta, p->p->n_phi, p->p->L, v, d, phi, order, means, sigma, v2, t_out, seed, r_len,
            rng_mode, out, 0);
  });
}

int sphemu_gpu_emulate_trend(sphemu_sht_t p, const double* v, int d, const double* phi, int order,
                             const double* records, int harmonics, int period, const double* forcing_x, int64_t n_x,
                             const double* forcing_history, int64_t n_history, int64_t t_start, const double* v2,
                             int t_out, uint64_t seed, int r_len, int rng_mode, double* out) {
  return guard([&] {
    const TrendArgs ta{records, harmonics, period, forcing_x, n_x, forcing_history, n_history, t_start};
    emulate(p, p->p->n_theta, p->p->n_phi, p->p->L, v, d, phi, order, nullptr, nullptr, v2, t_out, seed, r_len,
            rng_mode, out, 0, &ta);
  });
}

int sphemu_gpu_emulate_range(sphemu_sht_t p, const double* v, int d, const double* phi, int order,
                             const double* means, const double* sigma, const double* v2, int t_out, uint64_t seed,
                             int r_begin, int r_count, int rng_mode, double* out) {
  return guard([&] {
    emulate(p, p->p->n_theta, p->p->n_phi, p->p->L, v, d, phi, order, means, sigma, v2, t_out, seed, r_count,
            rng_mode, out, r_begin);
  });
}

}  // extern "C"

// ===========================================================================
// Direct synthesis onto grids that cannot resolve L (sht.cpp:406-466,
// synth_bandlimited; the Python inverse_sht fallback of module.cpp:92-94).
// ===========================================================================
namespace sphemu_gpu {

// Fully normalized P~_lm(cos theta_i) (normalized_legendre_all, sht.cpp:406-427):
// P[i][l(l+1)/2 + m]. One CTA per ring: thread 0 runs the sectoral chain,
// then each thread walks the l-recurrence of its m columns.
__global__ void k_legendre_table(int L, int n_theta, double* P) {
  const int i = blockIdx.x;
  const double th = 3.14159265358979323846 * i / (n_theta - 1);
  const double ct = cos(th), st = sin(th);
  double* p = P + (int64_t)i * L * (L + 1) / 2;
  auto at = [&](int l, int m) -> double& { return p[(int64_t)l * (l + 1) / 2 + m]; };
  if (threadIdx.x == 0) {
    at(0, 0) = 1.0 / sqrt(4.0 * 3.14159265358979323846);
    for (int m = 1; m < L; ++m) at(m, m) = -sqrt((2.0 * m + 1.0) / (2.0 * m)) * st * at(m - 1, m - 1);
  }
  __syncthreads();
  for (int m = threadIdx.x; m < L; m += blockDim.x) {
    if (m + 1 < L) at(m + 1, m) = sqrt(2.0 * m + 3.0) * ct * at(m, m);
    for (int l = m + 2; l < L; ++l) {
      const double a = sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)m * m));
      const double b = sqrt(((double)(l - 1) * (l - 1) - (double)m * m) / (4.0 * (double)(l - 1) * (l - 1) - 1.0));
      at(l, m) = a * (ct * at(l - 1, m) - b * at(l - 2, m));
    }
  }
}

// One CTA per (ring i, snapshot t): s_m = sum_l P_lm z_lm, then
// f(theta_i, phi_j) = Re s_0 + 2 sum_{m>=1} Re(s_m e^{i m phi_j}).
__global__ void k_synth_direct(const double* __restrict__ coeffs, const double* __restrict__ P, int L, int n_theta,
                               int n_phi, double* __restrict__ fields) {
  extern __shared__ double2 sm_s[];
  const int i = blockIdx.x, t = blockIdx.y;
  const double* z = coeffs + (int64_t)t * L * L;
  const double* p = P + (int64_t)i * L * (L + 1) / 2;
  for (int m = threadIdx.x; m < L; m += blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int l = m; l < L; ++l) {
      const double pl = p[(int64_t)l * (l + 1) / 2 + m];
      if (m == 0) {
        re += pl * z[(int64_t)l * l];
      } else {
        re += pl * z[(int64_t)l * l + 2 * m - 1];
        im += pl * z[(int64_t)l * l + 2 * m];
      }
    }
    sm_s[m] = make_double2(re, im);
  }
  __syncthreads();
  double* out = fields + ((int64_t)t * n_theta + i) * n_phi;
  for (int j = threadIdx.x; j < n_phi; j += blockDim.x) {
    double v = sm_s[0].x;
    for (int m = 1; m < L; ++m) {
      double s, c;
      sincospi(2.0 * (double)((int64_t)m * j % n_phi) / n_phi, &s, &c);  // phi_j = 2 pi j / n_phi
      v += 2.0 * (sm_s[m].x * c - sm_s[m].y * s);
    }
    out[j] = v;
  }
}

}  // namespace sphemu_gpu

extern "C" int sphemu_gpu_synth_bandlimited(const double* coeffs, int where_in, int64_t n, int band_limit,
                                            int n_theta, int n_phi, double* fields, int where_out) {
  using namespace sphemu_gpu;
  return guard([&] {
    if (band_limit < 1) throw std::invalid_argument("band limit must be positive");
    if (n_theta < 2) throw std::invalid_argument("grid needs at least two latitude rings");
    if (n_phi < 1) throw std::invalid_argument("grid needs at least one longitude point");
    if (n <= 0) return;
    const int L = band_limit;
    const int64_t nc = (int64_t)L * L, pts = (int64_t)n_theta * n_phi;
    DevBuf<double> dP((size_t)n_theta * L * (L + 1) / 2), dc, df;
    const double* cin = coeffs;
    double* fout = fields;
    if (where_in == SPHEMU_HOST) {
      dc.alloc((size_t)n * nc);
      SPH_CUDA(cudaMemcpy(dc.get(), coeffs, sizeof(double) * n * nc, cudaMemcpyHostToDevice));
      cin = dc.get();
    }
    if (where_out == SPHEMU_HOST) {
      df.alloc((size_t)n * pts);
      fout = df.get();
    }
    k_legendre_table<<<n_theta, 128>>>(L, n_theta, dP.get());
    SPH_LAUNCH_CHECK();
    for (int64_t t0 = 0; t0 < n; t0 += 65535) {
      const int64_t T = std::min<int64_t>(65535, n - t0);
      k_synth_direct<<<dim3(n_theta, (unsigned)T), 128, L * sizeof(double2)>>>(cin + t0 * nc, dP.get(), L, n_theta,
                                                                              n_phi, fout + t0 * pts);
      SPH_LAUNCH_CHECK();
    }
    if (where_out == SPHEMU_HOST)
      SPH_CUDA(cudaMemcpy(fields, fout, sizeof(double) * n * pts, cudaMemcpyDeviceToHost));
    SPH_CUDA(cudaDeviceSynchronize());
  });
}
