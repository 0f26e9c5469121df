// chol.cu — host side of the tiled mixed-precision Cholesky: precision map,
// HBM tile arena, the CUDA-stream tile scheduler that replaces the reference's
// DAG worker pool (proj/src/mpchol.cpp:254-347), statistics, and the C-ABI
// entry points of include/sphemu_gpu.h.
//
// Schedule (right-looking, the same k-ordered update chains as
// build_task_graph, mpchol.cpp:156-205, so every tile sees its updates in
// k order exactly like the reference's serialized chains):
//   for k: POTRF+TRTRI(k,k) -> panel TRSM-as-GEMM (all i > k) -> scatter
//          -> trailing update grouped by output precision class.
#include <algorithm>
#include <atomic>
#include <emmintrin.h>
#include <condition_variable>
#include <functional>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include <nccl.h>

#include "chol_kernels.cuh"
#include "cov_kernels.cuh"
#include "potrf_coop.cuh"
#include "emulate.cuh"
#include "hostio.cuh"
#include "ozaki.cuh"
#include "tc_gemm.cuh"
#include "tcgen05.cuh"
#include "trmm.cuh"

namespace sphemu_gpu {
void sht_plan_dims(void* plan, int* n_theta, int* n_phi, int* L);  // sht.cu

#define SPH_NCCL(call)                                                                              \
  do {                                                                                              \
    ncclResult_t r__ = (call);                                                                      \
    if (r__ != ncclSuccess)                                                                         \
      throw ::sphemu_gpu::Error(SPHEMU_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r__)); \
  } while (0)

namespace {
thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
void note_launch(int64_t n) { g_launches += n; }
bool sync_check() {
  static const bool on = [] {
    const char* e = std::getenv("SPHEMU_SYNC_CHECK");
    return e && e[0] == '1';
  }();
  return on;
}
int64_t launch_count() { return g_launches.load(); }

namespace {
struct ScratchKey {
  std::thread::id tid;
  int dev, slot;
  bool operator<(const ScratchKey& o) const {
    return std::tie(tid, dev, slot) < std::tie(o.tid, o.dev, o.slot);
  }
};
std::mutex g_scratch_mu;
std::map<ScratchKey, DevBuf<char>>& scratch_map() {
  static auto* m = new std::map<ScratchKey, DevBuf<char>>();  // never destroyed: no CUDA calls at exit
  return *m;
}
}  // namespace

void* scratch_bytes(int slot, size_t bytes) {
  if (slot < 0 || slot >= 8) throw Error(SPHEMU_ERR_RUNTIME, "scratch slot out of range");
  int dev = 0;
  SPH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  DevBuf<char>& b = scratch_map()[ScratchKey{std::this_thread::get_id(), dev, slot}];
  if (b.n < bytes) b.alloc(bytes);
  return b.get();
}

void smem_optin(const void* kernel, int bytes) {
  static std::mutex mu;
  static auto* done = new std::map<std::pair<const void*, int>, int>();
  int dev = 0;
  SPH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  int& have = (*done)[{kernel, dev}];
  if (have >= bytes) return;
  SPH_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  have = bytes;
}

void scratch_release_all() {
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  scratch_map().clear();
}

int num_sms() {
  static int sms = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return sms;
}

// MpCholConfig::validate (mpchol.cpp:55-61), same messages.
void validate_config(const sphemu_chol_config& c) {
  if (c.tile_size < 1) throw std::invalid_argument("tile size must be positive");
  if (c.band_width_dp < 1) throw std::invalid_argument("double-precision band must be at least 1");
  if (c.sp_fraction < 0.0 || c.sp_fraction > 1.0)
    throw std::invalid_argument("sp fraction must lie in [0, 1]");
  if (c.workers < 1) throw std::invalid_argument("worker count must be positive");
  if (c.variant < 0 || c.variant > 3) throw std::invalid_argument("unknown precision variant");
  if (c.hp_format != SPHEMU_HP_FP16 && c.hp_format != SPHEMU_HP_BF16)
    throw std::invalid_argument("unknown half-precision format");
  if (c.compute != SPHEMU_COMPUTE_TENSOR && c.compute != SPHEMU_COMPUTE_FP64)
    throw std::invalid_argument("unknown compute mode");
  if (c.sp_compute < SPHEMU_SP_F16X3 || c.sp_compute > SPHEMU_SP_FP64)
    throw std::invalid_argument("unknown single-precision compute");
}

// assign_precisions (mpchol.cpp:67-93): band tiles double; off-band tiles
// ordered by (distance, i, j); dpsp all single, dpsphp the first
// ceil(sp_fraction * off) single and the rest half, dphp all half.
std::vector<uint8_t> assign_precisions(int nt, const sphemu_chol_config& c) {
  validate_config(c);
  if (nt < 1) throw std::invalid_argument("need at least one tile");
  std::vector<uint8_t> map(static_cast<size_t>(nt) * (nt + 1) / 2, SPHEMU_PREC_DP);
  if (c.variant == SPHEMU_VARIANT_DP) return map;
  int64_t n_off = 0;
  for (int d = c.band_width_dp; d < nt; ++d) n_off += nt - d;
  int64_t n_sp = n_off;
  if (c.variant == SPHEMU_VARIANT_DPSPHP)
    n_sp = static_cast<int64_t>(std::ceil(c.sp_fraction * static_cast<double>(n_off)));
  else if (c.variant == SPHEMU_VARIANT_DPHP)
    n_sp = 0;
  int64_t t = 0;
  for (int d = c.band_width_dp; d < nt; ++d)
    for (int j = 0; j + d < nt; ++j, ++t) {
      const int i = j + d;
      map[static_cast<size_t>(i) * (i + 1) / 2 + j] = t < n_sp ? SPHEMU_PREC_SP : SPHEMU_PREC_HP;
    }
  return map;
}

// Squared Frobenius norm of every b x b tile of a dense row-major A (both
// triangles; the lower ones feed the tile-norm precision policy). One CTA per
// tile, coalesced row reads, warp-shuffle + smem reduction.
__global__ void k_tile_sqnorms(const double* __restrict__ a, int64_t lda, int n, int b, double* sq) {
  const int ti = blockIdx.y, tj = blockIdx.x;
  const int r0 = ti * b, c0 = tj * b;
  const int rows = min(b, n - r0), cols = min(b, n - c0);
  double acc = 0.0;
  for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
    const double v = a[(int64_t)(r0 + e / cols) * lda + c0 + e % cols];
    acc = fma(v, v, acc);
  }
  __shared__ double red[32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    acc = warp_sum(acc);
    if (threadIdx.x == 0) sq[(int64_t)ti * gridDim.x + tj] = acc;
  }
}

// The tile-norm ("tile-centric") precision rule, opt-in next to
// the band rule of mpchol.cpp:67-93: off the DP band, tile (i, j) takes the
// lowest precision the variant allows with u_p ||A_ij||_F <= tol ||A||_F / nt,
// so the storage rounding of all tiles sums to <= tol ||A||_F (Frobenius).
void tile_norm_map(const std::vector<double>& sq, int nt, const sphemu_chol_config& c, double tol, uint8_t* map) {
  double total = 0.0;
  for (double v : sq) total += v;
  total = std::sqrt(total);
  const double u_dp = 0x1.0p-53, u_sp = 0x1.0p-24, u_hp = c.hp_format == SPHEMU_HP_BF16 ? 0x1.0p-8 : 0x1.0p-11;
  std::vector<std::pair<int, double>> allowed;
  switch (c.variant) {
    case SPHEMU_VARIANT_DP: allowed = {{SPHEMU_PREC_DP, u_dp}}; break;
    case SPHEMU_VARIANT_DPSP: allowed = {{SPHEMU_PREC_SP, u_sp}, {SPHEMU_PREC_DP, u_dp}}; break;
    case SPHEMU_VARIANT_DPSPHP: allowed = {{SPHEMU_PREC_HP, u_hp}, {SPHEMU_PREC_SP, u_sp}, {SPHEMU_PREC_DP, u_dp}}; break;
    default: allowed = {{SPHEMU_PREC_HP, u_hp}, {SPHEMU_PREC_DP, u_dp}}; break;
  }
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j <= i; ++j) {
      uint8_t p = SPHEMU_PREC_DP;
      if (i - j >= c.band_width_dp) {
        const double t = std::sqrt(sq[static_cast<size_t>(i) * nt + j]);
        for (const auto& a : allowed)
          if (a.second * t <= tol * total / nt) {
            p = static_cast<uint8_t>(a.first);
            break;
          }
      }
      map[static_cast<size_t>(i) * (i + 1) / 2 + j] = p;
    }
}

// Row scale exponents for the FP16x3 path: |L_rj| <= sqrt(A_rr), so with
// sqrt(A_rr) = m 2^E (m in [0.5, 1)) every operand of row r times 2^(14-E)
// stays below 2^14 in magnitude.
__global__ void k_rowexp(TileStore ts, int* rowexp) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= ts.n) return;
  const int t = r / ts.lb, o = r % ts.lb;
  if (!ts.owned(t, t)) {  // another rank owns this diagonal tile (max-reduced later)
    rowexp[r] = -0x40000000;
    return;
  }
  const double a = load_elem(ts.tile(t, t), ts.tprec(t, t), (int64_t)o * ts.b + o);
  int e = 0;
  if (a > 0.0 && a < INFINITY) {
    int E;
    frexp(sqrt(a), &E);
    e = 14 - E;
  }
  rowexp[r] = e;
}

// 2D block-cyclic exchange: a panel tile received at its storage precision
// (xbuf slot i-k-1) -> FP64 mirror P64 and the tensor-core mirrors, exactly as
// the owner's panel epilogue writes them. blockIdx.y indexes the import list.
// need[i] (per panel row block, this rank's consumers): bit 0 the FP64 mirror
// (FP64-class updates / the INT8 digit cut), bit 1 the 16-bit HP mirror, bit 2
// the SP class's split; mirrors nobody here reads are not written.
__global__ void k_panel_import(TileStore ts, int k, const int2* __restrict__ list, const int64_t* __restrict__ xoff,
                               const uint8_t* __restrict__ xbuf, double* p64, float* p_hi, float* p_lo, uint16_t* p16, uint16_t* h_hi, uint16_t* h_lo,
                               const int* rowexp, int hp_format, const uint8_t* __restrict__ need, const int* fail) {
  if (*(volatile const int*)fail >= 0) return;
  const int b = ts.b;
  const int64_t bb = (int64_t)b * b;
  const int i = list[blockIdx.y].x;
  const int nd = need ? need[i] : 7;
  if (!(nd & 1)) p64 = nullptr;
  if (!(nd & 2)) p16 = nullptr;
  if (!(nd & 4)) p_hi = p_lo = nullptr, h_hi = h_lo = nullptr;
  if (!p64 && !p16 && !p_hi && !h_hi) return;
  const int p = ts.tprec(i, k);
  const int64_t base = (int64_t)(i - k - 1) * bb;
  const uint8_t* src = xbuf + xoff[blockIdx.y];
  // 8 consecutive elements (one row segment) per thread: 16-byte loads of the
  // packed tile, 16-byte stores of every mirror
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < bb / 8; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = g * 8;
    double x[8];
    if (p == kDP) {
      const double2* q = reinterpret_cast<const double2*>(src) + g * 4;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 v = q[u];
        x[2 * u] = v.x;
        x[2 * u + 1] = v.y;
      }
    } else if (p == kSP) {
      const float4* q = reinterpret_cast<const float4*>(src) + g * 2;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float4 v = q[u];
        x[4 * u] = v.x;
        x[4 * u + 1] = v.y;
        x[4 * u + 2] = v.z;
        x[4 * u + 3] = v.w;
      }
    } else {
      const uint4 v = reinterpret_cast<const uint4*>(src)[g];
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (p == kHP) {
          const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[u]));
          x[2 * u] = f.x;
          x[2 * u + 1] = f.y;
        } else {
          x[2 * u] = __uint_as_float(w[u] << 16);
          x[2 * u + 1] = __uint_as_float(w[u] & 0xffff0000u);
        }
      }
    }
    if (p64) {
      double2* q = reinterpret_cast<double2*>(p64 + base + e);
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = make_double2(x[2 * u], x[2 * u + 1]);
    }
    if (p_hi) {
      float hi[8], lo[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) tf32_split(__double2float_rn(x[u]), hi[u], lo[u]);
      float4* qh = reinterpret_cast<float4*>(p_hi + base + e);
      float4* ql = reinterpret_cast<float4*>(p_lo + base + e);
      qh[0] = make_float4(hi[0], hi[1], hi[2], hi[3]);
      qh[1] = make_float4(hi[4], hi[5], hi[6], hi[7]);
      ql[0] = make_float4(lo[0], lo[1], lo[2], lo[3]);
      ql[1] = make_float4(lo[4], lo[5], lo[6], lo[7]);
    }
    if (p16) {
      uint16_t h[8];
      unsigned dummy = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        h[u] = hp_format == SPHEMU_HP_BF16 ? __bfloat16_as_ushort(to_bf16_sat(x[u], dummy))
                                           : __half_as_ushort(to_half_sat(x[u], dummy));
      *reinterpret_cast<uint4*>(p16 + base + e) = *reinterpret_cast<const uint4*>(h);
    }
    if (h_hi) {
      const int r = (int)(e / b);
      const int er = rowexp[min(i * ts.lb + r, ts.n - 1)];
      uint16_t hh[8], hl[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) f16_split(x[u], er, hh[u], hl[u]);
      *reinterpret_cast<uint4*>(h_hi + base + e) = *reinterpret_cast<const uint4*>(hh);
      *reinterpret_cast<uint4*>(h_lo + base + e) = *reinterpret_cast<const uint4*>(hl);
    }
  }
}

// Sender side of the panel exchange: the owned panel tiles of step k, at
// storage precision, packed root-contiguously into the exchange buffer so
// each root sends one broadcast per step.
__global__ void k_panel_pack(TileStore ts, int k, const int2* __restrict__ list, const int64_t* __restrict__ xoff,
                             uint8_t* __restrict__ xbuf, const int* fail) {
  if (*(volatile const int*)fail >= 0) return;
  const int i = list[blockIdx.y].x;
  const int64_t words = (int64_t)ts.b * ts.b * prec_bytes(ts.tprec(i, k)) / 16;
  const uint4* src = static_cast<const uint4*>(ts.tile(i, k));
  uint4* dst = reinterpret_cast<uint4*>(xbuf + xoff[blockIdx.y]);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < words; e += (int64_t)gridDim.x * blockDim.x)
    dst[e] = src[e];
}

// ---- residual probe kernels -------------------------------------------------
__global__ void k_probe_vec(int n, uint64_t seed, double* x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  x[i] = ((double)(z >> 11) * 0x1.0p-53) * 2.0 - 1.0;
}

// y = A x with A = make_spd_test_matrix regenerated from (d, pw); warp per row.
__global__ void k_spd_matvec(int n, const double* __restrict__ d, const double* __restrict__ pw,
                             const double* __restrict__ x, double* y) {
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double acc = 0.0;
  for (int j = lane; j < n; j += 32) {
    double a;
    if (j == row) a = __dmul_rn(__dmul_rn(d[row], d[row]), 1.25);
    else if (j < row) a = __dmul_rn(__dmul_rn(__dmul_rn(d[row], d[j]), 0.25), pw[row - j]);
    else a = __dmul_rn(__dmul_rn(__dmul_rn(d[j], d[row]), 0.25), pw[j - row]);
    acc += a * x[j];
  }
  acc = warp_sum(acc);
  if (lane == 0) y[row] = acc;
}

// trans = 1: z_j += L_ij^T x_i ; trans = 0: y_i += L_ij z_j  (block per tile).
__global__ void k_tile_matvec(TileStore ts, const double* __restrict__ x, double* y, int trans) {
  int i, j;
  pair_from_index(blockIdx.x, i, j);
  if (!ts.owned(i, j)) return;
  const void* tp = ts.tile(i, j);
  const int p = ts.tprec(i, j);
  const int ri = ts.rows(i), rj = ts.rows(j);
  if (trans) {
    for (int c = threadIdx.x; c < rj; c += blockDim.x) {
      double acc = 0.0;
      for (int r = 0; r < ri; ++r) acc += load_elem(tp, p, (int64_t)r * ts.b + c) * x[i * ts.lb + r];
      atomicAdd(&y[j * ts.lb + c], acc);
    }
  } else {
    for (int r = threadIdx.x; r < ri; r += blockDim.x) {
      double acc = 0.0;
      for (int c = 0; c < rj; ++c) acc += load_elem(tp, p, (int64_t)r * ts.b + c) * x[j * ts.lb + c];
      atomicAdd(&y[i * ts.lb + r], acc);
    }
  }
}

__global__ void k_diff_norms(int n, const double* a, const double* b, double* sums) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double num = 0.0, den = 0.0;
  if (i < n) {
    num = (a[i] - b[i]) * (a[i] - b[i]);
    den = a[i] * a[i];
  }
  num = warp_sum(num);
  den = warp_sum(den);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&sums[0], num);
    atomicAdd(&sums[1], den);
  }
}

// Owner of tile (i, j) on a P x Q process grid: off-diagonal tiles are 2D
// block-cyclic, (i mod P, j mod Q), so row i lives on process row i mod P and
// column i on process column i mod Q; diagonal tiles — the FP64 band, whose
// SYRK updates cost ~50x a BF16 tile's — go round-robin over all P Q ranks
// (the plain map would give them only to the ranks with i mod P == i mod Q).
inline int block_cyclic_owner(int i, int j, int P, int Q) {
  // SPHEMU_MAP=shift (A/B): round 1's row-shifted map, ((i + s (j div Q)) mod P, j mod Q) with the
  // smallest s making gcd(Q + s, P) = 1
  static const bool shift = [] {
    const char* e = std::getenv("SPHEMU_MAP");
    return e && std::string(e) == "shift";
  }();
  if (shift) {
    int sh = 0;
    while (std::gcd(Q + sh, P) != 1) ++sh;
    return ((i + sh * (j / Q)) % P) * Q + (j % Q);
  }
  return i == j ? i % (P * Q) : (i % P) * Q + (j % Q);
}

// Host-only 2D block-cyclic layout (no CUDA calls): this rank's tile offsets
// in its arena and the per-step panel exchange plan. Panel tile (i, k) goes
// from its owner to exactly the ranks whose updates read it — the owners of
// row i's tiles (i, j), k < j <= i (process row i mod P + the owner of the
// diagonal tile) and of column i's tiles (j, i), j > i (process column
// i mod Q): P + Q ranks at most instead of all P Q.
// Chol builds its device state from it; sphemu_gpu_dist_layout exposes it to
// host-side tests.
struct BlockCyclic {
  struct Xfer {
    int i;      // panel tile row
    int peer;   // destination (sends) or source (recvs)
    int64_t pos, bytes;
  };
  int nt = 0, b = 0, P = 1, Q = 1, rank = 0;
  std::vector<int64_t> off;                 // per packed tile; -1 = stored elsewhere; back() = arena bytes
  std::vector<std::vector<Xfer>> sends, recvs;  // this rank's, per step k
  std::vector<std::vector<Xfer>> roots;         // per step k: (-, root, pos, bytes) owner blocks (broadcast mode)
  std::vector<std::vector<int>> others;         // per step k: panel rows this rank does not own
  std::vector<std::vector<int64_t>> xpos;   // per step k: byte position of panel tile i at [i - k - 1]
  std::vector<std::vector<int64_t>> recv_bytes;  // per step k, per rank: bytes that rank receives
  int64_t xmax = 0;
  int owner(int i, int j) const { return block_cyclic_owner(i, j, P, Q); }
  bool mine(int i, int j) const { return owner(i, j) == rank; }
  // ranks that read panel tile (i, k) in step k, its owner excluded
  std::vector<int> needers(int i, int k) const {
    std::vector<char> need(static_cast<size_t>(P) * Q, 0);
    for (int j = k + 1; j <= i; ++j) need[owner(i, j)] = 1;
    for (int j = i + 1; j < nt; ++j) need[owner(j, i)] = 1;
    need[owner(i, k)] = 0;
    std::vector<int> r;
    for (int q = 0; q < P * Q; ++q)
      if (need[q]) r.push_back(q);
    return r;
  }

  BlockCyclic(int nt_, int b_, const std::vector<uint8_t>& sprec, int P_, int Q_, int rank_)
      : nt(nt_), b(b_), P(P_), Q(Q_), rank(rank_) {
    off.assign(sprec.size() + 1, 0);
    int64_t o = 0;
    size_t t = 0;
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j <= i; ++j, ++t) {
        if (!mine(i, j)) {
          off[t] = -1;
          continue;
        }
        off[t] = o;
        o += static_cast<int64_t>(b) * b * prec_bytes(sprec[t]);
        o = (o + 255) & ~int64_t{255};
      }
    off.back() = o;
    if (P * Q == 1) return;
    sends.assign(nt, {});
    recvs.assign(nt, {});
    roots.assign(nt, {});
    others.assign(nt, {});
    xpos.assign(nt, {});
    recv_bytes.assign(nt, std::vector<int64_t>(static_cast<size_t>(P) * Q, 0));
    for (int k = 0; k + 1 < nt; ++k) {
      xpos[k].assign(nt - k - 1, 0);
      int64_t x = 0;
      for (int root = 0; root < P * Q; ++root)  // grouped by owner: each owner packs one contiguous block
        for (int i = k + 1; i < nt; ++i)
          if (owner(i, k) == root) {
            xpos[k][i - k - 1] = x;
            x += static_cast<int64_t>(b) * b * prec_bytes(sprec[static_cast<size_t>(i) * (i + 1) / 2 + k]);
          }
      xmax = std::max(xmax, x);
      for (int root = 0; root < P * Q; ++root) {
        int64_t lo = -1, hi = -1;
        for (int i = k + 1; i < nt; ++i)
          if (owner(i, k) == root) {
            const int64_t a = xpos[k][i - k - 1];
            const int64_t e = a + static_cast<int64_t>(b) * b *
                                      prec_bytes(sprec[static_cast<size_t>(i) * (i + 1) / 2 + k]);
            lo = lo < 0 ? a : std::min(lo, a);
            hi = std::max(hi, e);
          }
        if (lo >= 0) roots[k].push_back({-1, root, lo, hi - lo});
      }
      for (int i = k + 1; i < nt; ++i)
        if (owner(i, k) != rank) others[k].push_back(i);
      for (int i = k + 1; i < nt; ++i) {
        const int src = owner(i, k);
        const int64_t bytes = static_cast<int64_t>(b) * b * prec_bytes(sprec[static_cast<size_t>(i) * (i + 1) / 2 + k]);
        for (int r : needers(i, k)) {
          recv_bytes[k][r] += bytes;
          if (src == rank) sends[k].push_back({i, r, xpos[k][i - k - 1], bytes});
          if (r == rank) recvs[k].push_back({i, src, xpos[k][i - k - 1], bytes});
        }
      }
    }
  }
};

// fp64 <-> fp32 row conversion with streaming (non-temporal) stores: the
// destination is written once and read by the DMA engine or the caller, so
// skipping the read-for-ownership cuts the host memory traffic per element
// from 16 (20) to 12 bytes.
static void narrow_row(float* dst, const double* src, int cw) {
  int c = 0;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)
    for (; c + 4 <= cw; c += 4) {
      const __m128 lo = _mm_cvtpd_ps(_mm_loadu_pd(src + c));
      const __m128 hi = _mm_cvtpd_ps(_mm_loadu_pd(src + c + 2));
      _mm_stream_ps(dst + c, _mm_movelh_ps(lo, hi));
    }
  for (; c < cw; ++c) dst[c] = static_cast<float>(src[c]);
}

static void zero_row(double* dst, int64_t cnt) {
  int64_t c = 0;
  for (; c < cnt && (reinterpret_cast<uintptr_t>(dst + c) & 15); ++c) dst[c] = 0.0;
  const __m128d z = _mm_setzero_pd();
  for (; c + 2 <= cnt; c += 2) _mm_stream_pd(dst + c, z);
  for (; c < cnt; ++c) dst[c] = 0.0;
}

static void widen_row(double* dst, const float* src, int cw) {
  int c = 0;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)
    for (; c + 4 <= cw; c += 4) {
      const __m128 v = _mm_loadu_ps(src + c);
      _mm_stream_pd(dst + c, _mm_cvtps_pd(v));
      _mm_stream_pd(dst + c + 2, _mm_cvtps_pd(_mm_movehl_ps(v, v)));
    }
  for (; c < cw; ++c) dst[c] = static_cast<double>(src[c]);
}



struct Chol {
  static constexpr int kChainCtas = 32;  // SMs reserved for the critical chain under lookahead
  int potrf_cap = kChainCtas;            // cooperative POTRF grid cap (follows the step's reserve)
  int n = 0, b = 0, nt = 0;  // b = storage pitch (padded), lb = logical tile size
  int lb = 0;
  // 2D block-cyclic distribution over a P x Q process grid (one GPU per
  // rank): tile (i, j) lives on rank (i mod P) * Q + (j mod Q).
  int P = 1, Q = 1, rank = 0;
  ncclComm_t comm = nullptr;
  bool dist() const { return P * Q > 1; }
  int owner(int i, int j) const { return block_cyclic_owner(i, j, P, Q); }
  bool mine(int i, int j) const { return owner(i, j) == rank; }
  // Panel exchange buffer: per step the panel tiles at storage precision at
  // fixed positions (grouped by owner); xsend / ilists list this rank's packed
  // / received tiles with their byte positions, xsends / xrecvs the
  // point-to-point transfers of each step (BlockCyclic).
  DevBuf<uint8_t> xbuf;
  // Copy-engine panel exchange ("ipc", the default on a process grid): every
  // rank maps its peers' exchange buffers and sync words (CUDA IPC); an owner
  // packs its panel tiles into its own buffer (double-buffered by step
  // parity) and publishes the step with a stream memory write, readers wait
  // for it with cuStreamWaitValue32 and pull each owner's block with one
  // device-to-device copy over NVLink — copy engines, no SMs taken from the
  // bulk update (the NCCL broadcast kernels had to fit in the chain's reserve
  // next to a persistent bulk and crawled) — then acknowledge into the
  // owner's sync words before it reuses that parity.
  bool xipc = false;
  int64_t xhalf = 0;                        // bytes per parity half of xbuf
  DevBuf<uint32_t> xsync;                   // [0] = published step, [1 + r] = acks from rank r
  DevBuf<int> xbar;                         // device-side barrier word at the start of a factorization
  std::vector<uint8_t*> peer_xbuf;
  std::vector<uint32_t*> peer_sync;
  uint32_t xepoch = 0;                      // advanced by nt per factorization (stream-ordered words never go back)
  // Early exchange (lookahead on a process grid): tile k+1's panel row goes
  // first (its own TRSM, pack, publish, pull, import on the chain) so the
  // chain's next diagonal SYRK and POTRF start while the rest of the panel is
  // still being solved / pulled / imported on xstream; xlate[k] marks steps
  // whose panel completes on xstream.
  std::vector<uint8_t> xlate;
  cudaEvent_t ev_trdone = nullptr;
  void record_panel(int k) { SPH_CUDA(cudaEventRecord(ev_panel[k], (xlate.size() > size_t(k) && xlate[k]) ? xstream : pstream)); }
  DevBuf<int2> ilists, xsend;
  DevBuf<int64_t> ioffs, xsoffs;
  std::vector<int64_t> ilist_off, ilist_cnt, xsend_off, xsend_cnt;
  using Xfer = BlockCyclic::Xfer;
  std::vector<std::vector<Xfer>> xsends, xrecvs, xroots;
  // Chunked panel exchange (broadcast mode): the panel TRSM runs in xchunks
  // slices of the column on the chain stream while the previous slice is
  // packed, broadcast (second communicator) and imported on xstream.
  ncclComm_t comm2 = nullptr;
  cudaStream_t xstream = nullptr;
  // Process grids: the merged pair's big update (part 5) on its own stream
  // with fewer CTAs, so the next pair's critical column updates (part 2) are
  // not queued behind it (SPHEMU_SPLIT5, default on for process grids).
  cudaStream_t bstream = nullptr;
  std::vector<cudaEvent_t> ev_p4, ev_p5;
  std::vector<cudaEvent_t> ev_tr;
  cudaEvent_t ev_xdone = nullptr;
  int xchunks = 1;
  std::vector<std::vector<int64_t>> xpos_h;  // layout.xpos
  std::vector<int> pl_i, xs_i, il_i;         // host copies of the plist / xsend / ilist tile rows
  // Panel exchange: one grouped ncclBroadcast per owner block to every rank
  // (default), or with SPHEMU_XCHG=p2p point to point to the readers only
  // (BlockCyclic::needers: (P+Q)/(PQ) of the bytes per rank, but the owner
  // sends one copy per reader over its NVLink port). Measured on C3 (2x2):
  // broadcast 429 ms vs point-to-point 510 ms; 2x1: 677 vs 694 ms.
  static bool xchg_bcast() {
    static const bool on = [] {
      const char* e = std::getenv("SPHEMU_XCHG");
      return !(e && std::string(e) == "p2p");
    }();
    return on;
  }
  sphemu_chol_config cfg{};
  std::vector<uint8_t> pmap, sprec;
  std::vector<int64_t> off;
  DevBuf<char> arena;
  DevBuf<int64_t> d_off;
  DevBuf<uint8_t> d_prec;
  // Panel buffers rotate over kSets steps: with lookahead the chain writes
  // panel k+1 while the bulk reads panel k, and the merged schedule reads
  // panels k and k+1 while the chain writes k+2.
  static constexpr int kSets = 3;
  static int set_of(int k) { return k % kSets; }
  DevBuf<double> linv_[kSets], p64_[kSets];
  // DP-class updates on the INT8 tensor cores (ozaki.cuh): the digit planes
  // of each panel set. Block 0 (tile k+1, the chain's diagonal SYRK) is cut
  // on the panel's stream right after the panel; the rest by the main stream
  // before its first DP-class update of the step (oz_rest[k]).
  OzSlices oz_[kSets];
  bool oz = false;
  std::vector<uint8_t> oz_rest;
  std::vector<uint8_t> oz_fused;  // step k's digits were written by its panel epilogue
  // One GPU, opt-in (SPHEMU_OZ_FUSE = fraction): the panel epilogue writes the
  // digits of steps k < fraction * nt itself instead of the FP64 mirror; the
  // integer digit work on the chain's few SMs costs more than the bulk's
  // separate cut saves, so the default is 0.
  static double oz_fuse_frac() {
    static const double f = [] {
      const char* e = std::getenv("SPHEMU_OZ_FUSE");
      return e ? std::atof(e) : 0.0;  // measured: 0 / 0.25 / 0.5 / 1 -> C2 46.4 / 47.4 / 48.2 / 48.8 ms
    }();
    return f;
  }
  // Tiles whose panel rows some DP-class update on this rank reads (every
  // diagonal tile on one GPU; the owned DP tiles' rows and columns on a
  // process grid), ascending: the digits are cut for these rows only.
  std::vector<int> oz_tiles;
  std::vector<uint8_t> oz_need;
  DevBuf<int> d_oz_tiles;
  // SPHEMU_DP_EMU=0: DP-class updates on FP64 DMMA instead.
  static bool dp_emu_env() {
    static const bool on = [] {
      const char* e = std::getenv("SPHEMU_DP_EMU");
      return !(e && e[0] == '0');
    }();
    return on;
  }
  void oz_slice_rest(int k, cudaStream_t s) {
    if (oz_rest[k]) return;
    oz_rest[k] = 1;
    // the needed tiles below k+1 (block 0, tile k+1, is cut with the panel)
    const auto first = std::lower_bound(oz_tiles.begin(), oz_tiles.end(), k + 2);
    const int64_t cnt = oz_tiles.end() - first;
    if (cnt)
      oz_slice_tiles(store(), k, oz_src(k), d_oz_tiles.get() + (first - oz_tiles.begin()), cnt,
                     rowexp.get(), oz_[set_of(k)], fail.get(), s);
  }
  void oz_slice_next(int k, cudaStream_t s) {  // tile k+1's rows, for the chain's diagonal SYRK
    if (oz && k + 1 < nt && oz_need[k + 1])
      oz_slice(store(), k, oz_src(k), 0, b, rowexp.get(), oz_[set_of(k)], fail.get(), s);
  }
  // Where the digits are cut from: one GPU reads the panel tiles themselves
  // (their rounded values at 2-8 bytes; the panel epilogue then skips the FP64
  // mirror of SP/HP rows, which nothing else reads); process grids read the
  // FP64 mirror the import rebuilt (imported tiles are not in the arena).
  const double* oz_src(int k) { return dist() ? p64_[set_of(k)].get() : nullptr; }
  DevBuf<double> dinv, spd_d, spd_pw;
  uint64_t spd_seed = 0;
  double spd_rho = -1.0;  // (seed, rho) of the factors in spd_d / spd_pw
  DevBuf<int> rowexp;  // per-row power-of-two operand scale (FP16x3 SP path)
  DevBuf<int> fail;
  DevBuf<unsigned> sat;
  DevBuf<int2> lists;
  DevBuf<uint8_t> d_import_need;  // distributed: per panel row block, the mirrors this rank reads (k_panel_import)
  DevBuf<int> lrows;  // per update-list entry: the C tile's arena row (see constructor)
  // Dynamic work claiming for the persistent tcgen05 kernels: one counter per
  // (stream, class) (kernels on one stream run in order; the memset precedes
  // each launch, a resumed launch continues from its class's counter).
  // SPHEMU_TC_DYN=0 falls back to static striding.
  DevBuf<int> sched_ctr;
  DevBuf<unsigned> pc_bar;  // k_potrf_coop's split-barrier arrival counter (zero between launches)
  int* ctr(cudaStream_t s, int cls) {
    static const bool on = [] {
      const char* e = std::getenv("SPHEMU_TC_DYN");
      return !(e && e[0] == '0');
    }();
    return on ? sched_ctr.get() + (s == pstream ? 4 : (s == bstream && bstream ? 8 : 0)) + cls : nullptr;
  }
  // Bulk yield: the chain raises the flag when the next panel is ready; the
  // bulk's persistent CTAs stop claiming items so the panel gets the SMs, and
  // the bulk resumes after it (SPHEMU_YIELD=0 disables).
  DevBuf<int> yield_flag;
  static bool yield_on() {
    static const bool on = [] {
      const char* e = std::getenv("SPHEMU_YIELD");
      return !(e && e[0] == '0');
    }();
    return on;
  }
  // Update lists per (step k, part, class): part 0 = next column (k+1, the
  // critical chain), part 1 = the rest (columns >= k+2, the bulk).
  // Parts: 0 = the next diagonal tile (k+1, k+1) (feeds POTRF(k+1), the
  // critical chain), 1 = columns >= k+2 (the bulk), 2 = column k+1 below the
  // diagonal (feeds panel(k+1), runs ahead of the bulk on the main stream).
  // Merged schedule (pairs of steps k, k+1): part 3 = column k+2 (i >= k+2,
  // by panel k alone), part 4 = column k+3 and part 5 = columns >= k+4, both
  // updated by panels k and k+1 in one pass (parts 3+4+5 = part 1).
  static constexpr int kParts = 6;
  std::vector<int64_t> list_off, list_cnt;  // [(k * kParts + part) * 3 + class]
  DevBuf<int2> plists;                      // panel tiles per step: DP class, then SP/HP
  std::vector<int64_t> plist_off, plist_dp, plist_lo, plist_bf;
  bool panel_bf = false;  // BF16-class panel tiles listed after the others (plist_bf)
  PanelFormats panel_[kSets];               // tensor-core operand mirrors per set
  cudaStream_t stream = nullptr;            // main stream: bulk trailing updates
  cudaStream_t pstream = nullptr;           // high-priority stream: POTRF + panel chain
  std::vector<cudaEvent_t> ev_panel, ev_bulk, ev_colrest, ev_bulkdp;
  cudaEvent_t ev_start_p = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int64_t launches_at_start = 0, launches = 0;
  // Phase profiling (tracing subsystem): CUDA events around every phase
  // launch, folded into per-phase totals at wait().
  enum Phase { kPotrf = 0, kPanel = 1, kUpdDp = 2, kUpdSp = 3, kUpdHp = 4, kLoad = 5, kXchg = 6, kNumPhases = 7 };
  bool profiling = false;
  unsigned prof_mask = 0x7f;  // phases recorded while profiling
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, int>> ev_marks;  // (phase, start event index)
  struct Span {
    int phase, stream;
    double t0, t1;  // ms since the factorization's start event
  };
  std::vector<Span> timeline;  // last factorization
  double phase_ms[kNumPhases] = {0};
  int64_t phase_n[kNumPhases] = {0};
  int prof_begin(int phase, cudaStream_t s = nullptr) {
    if (!s) s = stream;
    if (!profiling || !(prof_mask & (1u << phase))) return -1;
    const size_t idx = ev_marks.size() * 2;
    while (ev_pool.size() < idx + 2) {
      cudaEvent_t e;
      SPH_CUDA(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    ev_marks.push_back({phase | (s == pstream ? 0x100 : (s == xstream && xstream ? 0x200 : 0)), static_cast<int>(idx)});
    SPH_CUDA(cudaEventRecord(ev_pool[idx], s));
    return static_cast<int>(idx);
  }
  void prof_end(int idx, cudaStream_t s = nullptr) {
    if (!s) s = stream;
    if (idx >= 0) SPH_CUDA(cudaEventRecord(ev_pool[idx + 1], s));
  }
  void prof_fold() {
    if (!ev_marks.empty()) timeline.clear();
    for (auto& m : ev_marks) {
      float ms = 0.f, a = 0.f, z = 0.f;
      const int phase = m.first & 0xff;
      SPH_CUDA(cudaEventElapsedTime(&ms, ev_pool[m.second], ev_pool[m.second + 1]));
      if (factored && cudaEventElapsedTime(&a, ev0, ev_pool[m.second]) == cudaSuccess &&
          cudaEventElapsedTime(&z, ev0, ev_pool[m.second + 1]) == cudaSuccess)
        timeline.push_back({phase, (m.first >> 8) & 3, a, z});
      phase_ms[phase] += ms;
      phase_n[phase] += 1;
    }
    ev_marks.clear();
  }
  std::chrono::steady_clock::time_point t_start;
  bool factored = false;

  // Host I/O pipeline. Host input is streamed by tile rows (row block i
  // needs only columns [0, (i+1) lb): the lower triangle, half the bytes)
  // through a ring of device slabs on a copy stream, and each slab is
  // quantized into its tiles on the main stream as soon as it lands. The
  // factor is streamed out by tile columns on a D2H stream as soon as each
  // column is final (after POTRF(k) + panel(k)), overlapping the rest of the
  // factorization; host threads write the zeros above the diagonal
  // meanwhile.
  static constexpr int kSlabs = 3;
  cudaStream_t cstream = nullptr, dstream = nullptr;
  DevBuf<double> islab, oslab;
  cudaEvent_t ev_in_full[kSlabs] = {}, ev_in_free[kSlabs] = {}, ev_col = nullptr;
  double* hout = nullptr;
  int64_t hldo = 0;
  std::vector<std::thread> zeroers;

  // Packed host I/O (single GPU, host buffers; SPHEMU_PACKED_IO=0 disables):
  // tile rows cross the link at storage width (k_load_packed), the factor
  // comes back the same way by column groups (k_store_cols_packed) and host
  // threads widen it into the caller's fp64 buffer while the factorization
  // continues. Halves the PCIe bytes of an SP-dominated matrix.
  std::unique_ptr<HostPool> iopool;
  PinnedBuf pin_in, pin_out;
  DevBuf<int64_t> d_grp_off, d_grp_rb;
  std::vector<int64_t> grp_off, grp_rb, grp_base;
  std::vector<cudaEvent_t> ev_grp;
  std::thread expander;
  std::mutex out_mu;
  std::condition_variable out_cv;
  int groups_issued = 0, groups_total = 0;
  bool out_abort = false, packed_out = false;
  std::exception_ptr out_err;

  bool packed_io() const {
    static const bool on = [] {
      const char* e = std::getenv("SPHEMU_PACKED_IO");
      return !(e && std::atoi(e) == 0);
    }();
    return on && !dist();
  }
  HostPool& pool() {
    if (!iopool) {
      const char* e = std::getenv("SPHEMU_IO_THREADS");
      const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
      const int T = e ? std::max(1, std::atoi(e)) : static_cast<int>(std::min(24u, std::max(1u, hw - 1)));
      iopool = std::make_unique<HostPool>(T);
    }
    return *iopool;
  }
  int64_t seg_bytes(int i, int j) const { return packed_seg_bytes(std::min(lb, n - j * lb), sprec[tix(i, j)]); }

  void load_host_packed(const double* a, int64_t lda, double diag_shift) {
    std::vector<int64_t> rbytes(nt), boff(nt + 1, 0);
    for (int i = 0; i < nt; ++i) {
      int64_t w = 0;
      for (int j = 0; j <= i; ++j) w += seg_bytes(i, j);
      rbytes[i] = w;
      boff[i + 1] = boff[i] + w * rows(i);
    }
    pin_in.ensure(static_cast<size_t>(boff[nt]));
    const size_t slab_bytes = sizeof(double) * static_cast<size_t>(lb) * n;  // >= any packed row block
    if (islab.n < kSlabs * static_cast<size_t>(lb) * n) islab.alloc(kSlabs * static_cast<size_t>(lb) * n);
    char* dslab = reinterpret_cast<char*>(islab.get());
    const unsigned gy = static_cast<unsigned>(std::max(1, b * b / (256 * 64)));
    HostPool& P = pool();
    for (int i = 0; i < nt; ++i) {
      char* hb = pin_in.p + boff[i];
      const int nr = rows(i);
      const int64_t rbi = rbytes[i];
      P.run([&](int t, int T) {
        const int r0 = static_cast<int>(static_cast<int64_t>(nr) * t / T);
        const int r1 = static_cast<int>(static_cast<int64_t>(nr) * (t + 1) / T);
        for (int r = r0; r < r1; ++r) {
          const double* src = a + static_cast<int64_t>(i * lb + r) * lda;
          char* dst = hb + static_cast<int64_t>(r) * rbi;
          for (int j = 0; j <= i; ++j) {
            const int cw = std::min(lb, n - j * lb);
            const double* sj = src + static_cast<int64_t>(j) * lb;
            if (sprec[tix(i, j)] == kDP) {
              std::memcpy(dst, sj, sizeof(double) * cw);
            } else {
              narrow_row(reinterpret_cast<float*>(dst), sj, cw);
            }
            dst += seg_bytes(i, j);
          }
        }
        _mm_sfence();
      });
      const int s = i % kSlabs;
      if (i >= kSlabs) SPH_CUDA(cudaStreamWaitEvent(cstream, ev_in_free[s], 0));
      char* dst = dslab + s * slab_bytes;
      SPH_CUDA(cudaMemcpyAsync(dst, hb, static_cast<size_t>(rbi) * nr, cudaMemcpyHostToDevice, cstream));
      SPH_CUDA(cudaEventRecord(ev_in_full[s], cstream));
      SPH_CUDA(cudaStreamWaitEvent(stream, ev_in_full[s], 0));
      k_load_packed<<<dim3(static_cast<unsigned>(i + 1), gy), 256, 0, stream>>>(store(), dst, rbi, sat.get(), i,
                                                                                 diag_shift);
      SPH_LAUNCH_CHECK();
      SPH_CUDA(cudaEventRecord(ev_in_free[s], stream));
    }
  }

  void begin_packed_out() {
    const int G = col_group();
    groups_total = (nt + G - 1) / G;
    grp_off.assign(static_cast<size_t>(groups_total) * nt, 0);
    grp_rb.assign(static_cast<size_t>(groups_total) * nt, 0);
    grp_base.assign(groups_total + 1, 0);
    for (int g = 0; g < groups_total; ++g) {
      const int k0 = g * G, k1 = std::min(nt, k0 + G);
      int64_t o = 0;
      for (int i = k0; i < nt; ++i) {
        int64_t w = 0;
        for (int j = k0; j < k1 && j <= i; ++j) w += seg_bytes(i, j);
        grp_off[static_cast<size_t>(g) * nt + i] = o;
        grp_rb[static_cast<size_t>(g) * nt + i] = w;
        o += w * rows(i);
      }
      grp_base[g + 1] = grp_base[g] + o;
    }
    pin_out.ensure(static_cast<size_t>(grp_base[groups_total]));
    d_grp_off.alloc(grp_off.size());
    d_grp_rb.alloc(grp_rb.size());
    SPH_CUDA(cudaMemcpy(d_grp_off.get(), grp_off.data(), grp_off.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    SPH_CUDA(cudaMemcpy(d_grp_rb.get(), grp_rb.data(), grp_rb.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    while (static_cast<int>(ev_grp.size()) < groups_total) {
      cudaEvent_t e;
      SPH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev_grp.push_back(e);
    }
    groups_issued = 0;
    out_abort = false;
    out_err = nullptr;
    packed_out = true;
    expander = std::thread([this, G] {
      try {
        for (int g = 0; g < groups_total; ++g) {
          {
            std::unique_lock<std::mutex> lk(out_mu);
            out_cv.wait(lk, [&] { return out_abort || groups_issued > g; });
            if (groups_issued <= g) return;
          }
          SPH_CUDA(cudaEventSynchronize(ev_grp[g]));
          widen_group(g, G);
        }
      } catch (...) {
        out_err = std::current_exception();
      }
    });
  }

  void widen_group(int g, int G) {
    const int k0 = g * G, k1 = std::min(nt, k0 + G);
    const int R0 = k0 * lb, nr = n - R0;
    const char* base = pin_out.p + grp_base[g];
    pool().run([&](int t, int T) {
      const int a0 = R0 + static_cast<int>(static_cast<int64_t>(nr) * t / T);
      const int a1 = R0 + static_cast<int>(static_cast<int64_t>(nr) * (t + 1) / T);
      for (int R = a0; R < a1; ++R) {
        const int i = R / lb;
        const size_t gi = static_cast<size_t>(g) * nt + i;
        const char* src = base + grp_off[gi] + static_cast<int64_t>(R - i * lb) * grp_rb[gi];
        double* dst = hout + static_cast<int64_t>(R) * hldo + static_cast<int64_t>(k0) * lb;
        for (int j = k0; j < k1 && j <= i; ++j) {
          const int cw = std::min(lb, n - j * lb);
          if (sprec[tix(i, j)] == kDP) {
            std::memcpy(dst, src, sizeof(double) * cw);
          } else {
            widen_row(dst, reinterpret_cast<const float*>(src), cw);
          }
          dst += cw;
          src += seg_bytes(i, j);
        }
      }
      _mm_sfence();
    });
  }

  void stop_expander() {
    if (!expander.joinable()) return;
    {
      std::lock_guard<std::mutex> lk(out_mu);
      out_abort = true;
    }
    out_cv.notify_all();
    expander.join();
  }

  void ensure_io() {
    if (cstream) return;
    SPH_CUDA(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking));
    SPH_CUDA(cudaStreamCreateWithFlags(&dstream, cudaStreamNonBlocking));
    for (int s = 0; s < kSlabs; ++s) {
      SPH_CUDA(cudaEventCreateWithFlags(&ev_in_full[s], cudaEventDisableTiming));
      SPH_CUDA(cudaEventCreateWithFlags(&ev_in_free[s], cudaEventDisableTiming));
    }
    SPH_CUDA(cudaEventCreateWithFlags(&ev_col, cudaEventDisableTiming));
  }

  void load_host(const double* a, int64_t lda, double diag_shift = 0.0) {
    ensure_io();
    if (packed_io()) {
      load_host_packed(a, lda, diag_shift);
      return;
    }
    const size_t slab = static_cast<size_t>(lb) * n;
    if (islab.n < kSlabs * slab) islab.alloc(kSlabs * slab);
    std::vector<char> row_has(nt, 0);  // rows holding at least one tile of this rank
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j <= i && !row_has[i]; ++j) row_has[i] = mine(i, j);
    const unsigned gy = static_cast<unsigned>(std::max(1, b * b / (256 * 64)));
    int used = 0;
    for (int i = 0; i < nt; ++i) {
      if (dist() && !row_has[i]) continue;
      const int s = used % kSlabs;
      if (used >= kSlabs) SPH_CUDA(cudaStreamWaitEvent(cstream, ev_in_free[s], 0));
      double* dst = islab.get() + s * slab;
      const int w = std::min(n, (i + 1) * lb);
      if (!dist()) {
        SPH_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * n, a + static_cast<int64_t>(i) * lb * lda,
                                   sizeof(double) * lda, sizeof(double) * w, rows(i), cudaMemcpyHostToDevice, cstream));
      } else {  // only this rank's tiles of the row cross the host link
        for (int j = 0; j <= i; ++j) {
          if (!mine(i, j)) continue;
          const int cw = std::min(lb, n - j * lb);
          SPH_CUDA(cudaMemcpy2DAsync(dst + static_cast<int64_t>(j) * lb, sizeof(double) * n,
                                     a + static_cast<int64_t>(i) * lb * lda + static_cast<int64_t>(j) * lb,
                                     sizeof(double) * lda, sizeof(double) * cw, rows(i), cudaMemcpyHostToDevice,
                                     cstream));
        }
      }
      SPH_CUDA(cudaEventRecord(ev_in_full[s], cstream));
      SPH_CUDA(cudaStreamWaitEvent(stream, ev_in_full[s], 0));
      k_load_dense<<<dim3(static_cast<unsigned>(i + 1), gy), 256, 0, stream>>>(
          store(), dst, n, sat.get(), static_cast<int64_t>(tix(i, 0)), i * lb, diag_shift);
      SPH_LAUNCH_CHECK();
      SPH_CUDA(cudaEventRecord(ev_in_free[s], stream));
      ++used;
    }
  }

  void begin_host_out(double* out, int64_t ldo) {
    ensure_io();
    if (oslab.n < static_cast<size_t>(n) * lb * col_group()) oslab.alloc(static_cast<size_t>(n) * lb * col_group());
    col_pending = -1;
    hout = out;
    hldo = ldo;
    packed_out = false;
    if (packed_io()) begin_packed_out();
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    static const int t_env = [] {
      const char* e = std::getenv("SPHEMU_ZERO_THREADS");
      return e ? std::atoi(e) : -1;
    }();
    const int T = t_env >= 0 ? t_env : static_cast<int>(std::min(8u, std::max(1u, hw / 2)));
    const int nn = n, l = lb;
    for (int t = 0; t < T; ++t)
      zeroers.emplace_back([=] {
        for (int64_t R = t; R < nn; R += T) {
          const int64_t c0 = (R / l + 1) * l;
          if (c0 < nn) zero_row(out + R * ldo + c0, nn - c0);
        }
        _mm_sfence();
      });
  }

  // Column k of the factor is final on stream s: convert and copy it out.
  // Column k of the factor is final on stream s. Columns leave in groups of
  // kColGroup (one conversion kernel + one 2-D copy with rows of
  // kColGroup * lb doubles: wide rows keep the D2H engine efficient).
  int col_group() const {
    static const int g = [] {
      const char* e = std::getenv("SPHEMU_COL_GROUP");
      return e ? std::max(1, std::atoi(e)) : 4;
    }();
    return g;
  }
  int col_pending = -1;  // first column of the open group
  void col_out(int k, cudaStream_t s, const TileStore* from = nullptr) {
    if (!hout) return;
    const int G = col_group();
    if (col_pending < 0) col_pending = k;
    if (k - col_pending + 1 < G && k + 1 < nt) return;
    const int k0 = col_pending;
    col_pending = -1;
    SPH_CUDA(cudaEventRecord(ev_col, s));
    SPH_CUDA(cudaStreamWaitEvent(dstream, ev_col, 0));
    const int h = n - k0 * lb;
    if (packed_out) {
      if (k0 % G) throw std::runtime_error("packed output expects column groups aligned to the group size");
      const int g = k0 / G;
      k_store_cols_packed<<<h, 256, 0, dstream>>>(from ? *from : store(), k0, k + 1,
                                                  d_grp_off.get() + static_cast<size_t>(g) * nt,
                                                  d_grp_rb.get() + static_cast<size_t>(g) * nt,
                                                  reinterpret_cast<char*>(oslab.get()));
      SPH_LAUNCH_CHECK();
      SPH_CUDA(cudaMemcpyAsync(pin_out.p + grp_base[g], oslab.get(), static_cast<size_t>(grp_base[g + 1] - grp_base[g]),
                               cudaMemcpyDeviceToHost, dstream));
      SPH_CUDA(cudaEventRecord(ev_grp[g], dstream));
      {
        std::lock_guard<std::mutex> lk(out_mu);
        groups_issued = g + 1;
      }
      out_cv.notify_all();
      return;
    }
    const int W = G * lb;
    k_store_cols<<<h, 256, 0, dstream>>>(from ? *from : store(), k0, k + 1, W, oslab.get());
    SPH_LAUNCH_CHECK();
    const int width = std::min(n, (k + 1) * lb) - k0 * lb;
    SPH_CUDA(cudaMemcpy2DAsync(hout + static_cast<int64_t>(k0) * lb * hldo + static_cast<int64_t>(k0) * lb,
                               sizeof(double) * hldo, oslab.get(), sizeof(double) * W, sizeof(double) * width, h,
                               cudaMemcpyDeviceToHost, dstream));
  }

  void end_host_out() {
    stop_expander();  // every group was issued by now, or the factorization failed
    for (auto& t : zeroers) t.join();
    zeroers.clear();
    packed_out = false;
    if (!hout) return;
    hout = nullptr;
    SPH_CUDA(cudaStreamSynchronize(dstream));
    if (out_err) {
      std::exception_ptr e = out_err;
      out_err = nullptr;
      std::rethrow_exception(e);
    }
  }

  int rows(int i) const { return std::min(lb, n - i * lb); }
  size_t tix(int i, int j) const { return static_cast<size_t>(i) * (i + 1) / 2 + j; }

  TileStore store() const {
    return TileStore{arena.get(), d_off.get(), d_prec.get(), n, b, nt, lb};
  }

  Chol(int n_, const sphemu_chol_config& c, int P_ = 1, int Q_ = 1, int rank_ = 0, ncclComm_t comm_ = nullptr,
       const uint8_t* map = nullptr)
      : n(n_), P(P_), Q(Q_), rank(rank_), comm(comm_), cfg(c) {
    validate_config(cfg);
    if (n < 1) throw std::invalid_argument("matrix is empty");
    lb = cfg.tile_size;
    if (lb > 1024) throw std::invalid_argument("tile_size above 1024 is not supported");
    // Storage pitch: the logical tile padded with zeros to the kernel granule
    // (64 for the FP64 kernels, 128 for the tcgen05 tiles).
    const int granule = cfg.compute == SPHEMU_COMPUTE_TENSOR ? 128 : 64;
    b = (lb + granule - 1) / granule * granule;
    nt = (n + lb - 1) / lb;
    pmap = assign_precisions(nt, cfg);
    if (map) {  // an explicit precision map (the tile-norm policy): the diagonal stays DP (POTRF is FP64)
      for (int i = 0; i < nt; ++i)
        for (int j = 0; j <= i; ++j) {
          const uint8_t p = map[tix(i, j)];
          if (p > SPHEMU_PREC_HP) throw std::invalid_argument("precision map entries must be 0, 1 or 2");
          if (i == j && p != SPHEMU_PREC_DP) throw std::invalid_argument("diagonal tiles must be double precision");
        }
      pmap.assign(map, map + pmap.size());
    }
    sprec.resize(pmap.size());
    for (size_t t = 0; t < pmap.size(); ++t)
      sprec[t] = static_cast<uint8_t>(pmap[t] == SPHEMU_PREC_DP
                                          ? kDP
                                          : (pmap[t] == SPHEMU_PREC_SP ? kSP
                                                                       : (cfg.hp_format == SPHEMU_HP_BF16 ? kBF : kHP)));
    BlockCyclic layout(nt, b, sprec, P, Q, rank);
    off = layout.off;
    const int64_t o = off.back();
    arena.alloc(static_cast<size_t>(std::max<int64_t>(o, static_cast<int64_t>(128) * b)));
    d_off.alloc(pmap.size());
    d_prec.alloc(pmap.size());
    SPH_CUDA(cudaMemcpy(d_off.get(), off.data(), pmap.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    SPH_CUDA(cudaMemcpy(d_prec.get(), sprec.data(), pmap.size(), cudaMemcpyHostToDevice));
    SPH_CUDA(cudaMemset(arena.get(), 0, static_cast<size_t>(o)));
    for (int p = 0; p < kSets; ++p) linv_[p].alloc(static_cast<size_t>(b) * b);
    dinv.alloc(static_cast<size_t>(b / PC_BLK + 1) * PC_BLK * PC_BLK);
    if (nt > 1)
      for (int p = 0; p < kSets; ++p) p64_[p].alloc(static_cast<size_t>(nt - 1) * b * b);
    fail.alloc(1);
    sat.alloc(1);
    sched_ctr.alloc(12);  // [stream: main, chain, bulk2][class 0..2, 3 = panel]
    pc_bar.alloc(1);
    SPH_CUDA(cudaMemset(pc_bar.get(), 0, sizeof(unsigned)));
    yield_flag.alloc(1);
    SPH_CUDA(cudaMemset(yield_flag.get(), 0, sizeof(int)));
    // Per-step output-tile lists by precision class.
    list_off.assign(static_cast<size_t>(nt) * kParts * 3 + 1, 0);
    list_cnt.assign(static_cast<size_t>(nt) * kParts * 3, 0);
    std::vector<int2> all;
    for (int k = 0; k < nt; ++k)
      for (int part = 0; part < kParts; ++part)
        for (int cls = 0; cls < 3; ++cls) {
          const size_t slot = (static_cast<size_t>(k) * kParts + part) * 3 + cls;
          list_off[slot] = static_cast<int64_t>(all.size());
          int j_lo = part == 1 ? k + 2 : k + 1, j_hi = part == 1 ? nt : std::min(k + 2, nt);
          if (part == 3) j_lo = k + 2, j_hi = std::min(k + 3, nt);
          if (part == 4) j_lo = k + 3, j_hi = std::min(k + 4, nt);
          if (part == 5) j_lo = k + 4, j_hi = nt;
          // wide bulk lists (parts 1 and 5) in blocks of JB columns, rows outer:
          // the items in flight together share B (column) and A (row) panel
          // operands in L2 (SPHEMU_LIST_JB, 1 = plain column-major order).
          // JB 1 / 2 / 4 / 8 / 12 / 16 / 32: C2 45.3 / 45.0 / 44.8 / 44.7 / 44.9 /
          // 44.9 / 45.4 ms, C3 792 / - / 755 / 749 / 748 / 761 / 768 ms.
          static const int jb_env = [] {
            const char* e = std::getenv("SPHEMU_LIST_JB");
            return e ? std::max(1, std::atoi(e)) : 8;
          }();
          const int JB = (part == 1 || part == 5) ? jb_env : 1;
          for (int j0 = j_lo; j0 < j_hi; j0 += JB)
            for (int i = j0; i < nt; ++i)
              for (int j = j0; j < std::min(j0 + JB, j_hi) && j <= i; ++j) {
                if (part == 0 && i != j) continue;
                if (part == 2 && i == j) continue;
                if (pmap[tix(i, j)] == cls && mine(i, j)) all.push_back(make_int2(i, j));
              }
          list_cnt[slot] = static_cast<int64_t>(all.size()) - list_off[slot];
        }
    if (!all.empty()) {
      lists.alloc(all.size());
      SPH_CUDA(cudaMemcpy(lists.get(), all.data(), all.size() * sizeof(int2), cudaMemcpyHostToDevice));
      // Per entry: the tile's first row in the arena viewed as rows of b
      // elements at the tile's storage width (the update kernels' C operand).
      std::vector<int> rowsv(all.size());
      for (size_t e = 0; e < all.size(); ++e) {
        const size_t t = tix(all[e].x, all[e].y);
        rowsv[e] = static_cast<int>(off[t] / (static_cast<int64_t>(prec_bytes(sprec[t])) * b));
      }
      lrows.alloc(rowsv.size());
      SPH_CUDA(cudaMemcpy(lrows.get(), rowsv.data(), rowsv.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    plist_off.assign(nt, 0);
    plist_dp.assign(nt, 0);
    plist_lo.assign(nt, 0);
    plist_bf.assign(nt, 0);
    // BF16-class panel tiles go through the bf16 x (hi + lo) panel kernel
    // (SPHEMU_PANEL_BF16=0: 3xTF32 like the SP class): listed last per step.
    static const bool panel_bf_env = [] {
      const char* e = std::getenv("SPHEMU_PANEL_BF16");
      return !(e && e[0] == '0');
    }();
    const bool bf_split = panel_bf_env && cfg.hp_format == SPHEMU_HP_BF16 && cfg.compute == SPHEMU_COMPUTE_TENSOR;
    std::vector<int2> pl;
    for (int k = 0; k < nt; ++k) {
      plist_off[k] = static_cast<int64_t>(pl.size());
      for (int i = k + 1; i < nt; ++i)
        if (fp64_class(pmap[tix(i, k)]) && mine(i, k)) pl.push_back(make_int2(i, k));
      plist_dp[k] = static_cast<int64_t>(pl.size()) - plist_off[k];
      for (int i = k + 1; i < nt; ++i) {
        const int c = pmap[tix(i, k)];
        if (!fp64_class(c) && mine(i, k) && !(bf_split && c == SPHEMU_PREC_HP)) pl.push_back(make_int2(i, k));
      }
      plist_lo[k] = static_cast<int64_t>(pl.size()) - plist_off[k] - plist_dp[k];
      if (bf_split)
        for (int i = k + 1; i < nt; ++i)
          if (pmap[tix(i, k)] == SPHEMU_PREC_HP && mine(i, k)) pl.push_back(make_int2(i, k));
      plist_bf[k] = static_cast<int64_t>(pl.size()) - plist_off[k] - plist_dp[k] - plist_lo[k];
    }
    panel_bf = bf_split;
    pl_i.resize(pl.size());
    for (size_t e = 0; e < pl.size(); ++e) pl_i[e] = pl[e].x;
    if (!pl.empty()) {
      plists.alloc(pl.size());
      SPH_CUDA(cudaMemcpy(plists.get(), pl.data(), pl.size() * sizeof(int2), cudaMemcpyHostToDevice));
    }
    if (dist()) {
      ilist_off.assign(nt, 0);
      ilist_cnt.assign(nt, 0);
      xsend_off.assign(nt, 0);
      xsend_cnt.assign(nt, 0);
      std::vector<int2> il, xs;
      std::vector<int64_t> io, xo;
      xsends = layout.sends;
      xrecvs = layout.recvs;
      xroots = layout.roots;
      const bool bc = xchg_bcast();
      const int64_t xmax = layout.xmax;
      for (int k = 0; k + 1 < nt; ++k) {
        ilist_off[k] = static_cast<int64_t>(il.size());
        xsend_off[k] = static_cast<int64_t>(xs.size());
        if (bc) {
          for (int i : layout.others[k]) {
            il.push_back(make_int2(i, k));
            io.push_back(layout.xpos[k][i - k - 1]);
          }
        } else {
          for (const Xfer& x : layout.recvs[k]) {
            il.push_back(make_int2(x.i, k));
            io.push_back(x.pos);
          }
        }
        for (int i = k + 1; i < nt; ++i)
          if (mine(i, k) && (bc || !layout.needers(i, k).empty())) {
            xs.push_back(make_int2(i, k));
            xo.push_back(layout.xpos[k][i - k - 1]);
          }
        ilist_cnt[k] = static_cast<int64_t>(il.size()) - ilist_off[k];
        xsend_cnt[k] = static_cast<int64_t>(xs.size()) - xsend_off[k];
      }
      auto upload = [](auto& dev, const auto& host) {
        if (host.empty()) return;
        dev.alloc(host.size());
        SPH_CUDA(cudaMemcpy(dev.get(), host.data(), host.size() * sizeof(host[0]), cudaMemcpyHostToDevice));
      };
      upload(ilists, il);
      upload(ioffs, io);
      il_i.resize(il.size());
      for (size_t e = 0; e < il.size(); ++e) il_i[e] = il[e].x;
      xs_i.resize(xs.size());
      for (size_t e = 0; e < xs.size(); ++e) xs_i[e] = xs[e].x;
      xpos_h = layout.xpos;
      // which operand mirrors this rank's updates read, per panel row block
      std::vector<uint8_t> need(nt, 0);
      for (int i = 1; i < nt; ++i)
        for (int j = 1; j <= i; ++j) {
          if (!mine(i, j)) continue;
          const int c = pmap[tix(i, j)];
          const uint8_t bit = (fp64_class(c) || cfg.compute != SPHEMU_COMPUTE_TENSOR) ? 1 : (c == SPHEMU_PREC_HP ? 2 : 4);
          need[i] |= bit;
          need[j] |= bit;
        }
      upload(d_import_need, need);
      upload(xsend, xs);
      upload(xsoffs, xo);
      static const int xmode_ipc = [] {
        const char* e = std::getenv("SPHEMU_XCHG");
        return !(e && (std::string(e) == "p2p" || std::string(e) == "nccl"));
      }();
      xipc = bc && xmode_ipc && xmax > 0;
      xhalf = (xmax + 255) / 256 * 256;
      if (xmax > 0) xbuf.alloc(static_cast<size_t>(xipc ? 2 * xhalf : xmax));
      if (xipc) ipc_setup();

    }
    rowexp.alloc(n);
    SPH_CUDA(cudaMemset(rowexp.get(), 0, n * sizeof(int)));
    if (cfg.compute == SPHEMU_COMPUTE_TENSOR && nt > 1)
      for (int p = 0; p < kSets; ++p) {
        panel_[p].alloc(nt, b, pmap, cfg.hp_format, cfg.sp_compute == SPHEMU_SP_F16X3, rowexp.get());
        panel_[p].set_arena(arena.get(), std::max<int64_t>(o, static_cast<int64_t>(128) * b), b);
        panel_[p].pair_dyn_sp = nt < 96;  // see tc_update
      }
    {
      bool any_dp_update = false;
      for (int i = 1; i < nt && !any_dp_update; ++i)
        for (int j = 1; j <= i; ++j)
          if (pmap[tix(i, j)] == SPHEMU_PREC_DP && mine(i, j)) {
            any_dp_update = true;
            break;
          }
      // Not for the exact modes: the pure-FP64 variant and sp_compute = fp64
      // keep every FP64-class update on DMMA.
      oz = dp_emu_env() && cfg.variant != SPHEMU_VARIANT_DP && cfg.sp_compute != SPHEMU_SP_FP64 &&
           cfg.compute == SPHEMU_COMPUTE_TENSOR && nt > 1 && b % 128 == 0 && any_dp_update;
      oz_need.assign(nt, 0);
      for (int i = 1; i < nt; ++i)
        for (int j = 1; j <= i; ++j)
          if (pmap[tix(i, j)] == SPHEMU_PREC_DP && mine(i, j)) oz_need[i] = oz_need[j] = 1;
      oz_tiles.clear();
      for (int q = 0; q < nt; ++q)
        if (oz_need[q]) oz_tiles.push_back(q);
      if (oz) {
        for (int p = 0; p < kSets; ++p) oz_[p].alloc(static_cast<int64_t>(nt - 1) * b, b);
        // one GPU: the panel epilogue writes the digits itself (no FP64 mirror
        // of the SP/HP panel rows, no separate digit cut); process grids cut
        // them from the imported rows
        // (decided per step in op_panel: early steps, where the chain has slack)
        d_oz_tiles.alloc(oz_tiles.size());
        SPH_CUDA(cudaMemcpy(d_oz_tiles.get(), oz_tiles.data(), oz_tiles.size() * sizeof(int), cudaMemcpyHostToDevice));
      }
      oz_rest.assign(nt, 0);
      oz_fused.assign(nt, 0);
    }
    int prio_lo = 0, prio_hi = 0;
    SPH_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    SPH_CUDA(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, prio_lo));
    SPH_CUDA(cudaStreamCreateWithPriority(&pstream, cudaStreamNonBlocking, prio_hi));
    {
      SPH_CUDA(cudaStreamCreateWithPriority(&bstream, cudaStreamNonBlocking, prio_lo));
      ev_p4.resize(nt);
      ev_p5.resize(nt);
      for (int k = 0; k < nt; ++k) {
        SPH_CUDA(cudaEventCreateWithFlags(&ev_p4[k], cudaEventDisableTiming));
        SPH_CUDA(cudaEventCreateWithFlags(&ev_p5[k], cudaEventDisableTiming));
      }
    }
    if (xipc) {
      SPH_CUDA(cudaStreamCreateWithPriority(&xstream, cudaStreamNonBlocking, prio_hi));
      SPH_CUDA(cudaEventCreateWithFlags(&ev_xdone, cudaEventDisableTiming));
      SPH_CUDA(cudaEventCreateWithFlags(&ev_trdone, cudaEventDisableTiming));
    }
    if (dist() && xchg_bcast() && !xipc) {
      static const int env_chunks = [] {
        const char* e = std::getenv("SPHEMU_XCHG_CHUNKS");
        return e ? std::max(1, std::atoi(e)) : 1;  // measured slower when chunked (C3 2x2: 1 / 2 / 4 / 8 -> 358 / 374 / 388 / 425 ms)
      }();
      xchunks = env_chunks;
      if (xchunks > 1) {
        SPH_NCCL(ncclCommSplit(comm, 0, rank, &comm2, nullptr));
        SPH_CUDA(cudaStreamCreateWithPriority(&xstream, cudaStreamNonBlocking, prio_hi));
        ev_tr.resize(xchunks);
        for (auto& e : ev_tr) SPH_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        SPH_CUDA(cudaEventCreateWithFlags(&ev_xdone, cudaEventDisableTiming));
      }
    }
    ev_panel.resize(nt);
    ev_bulk.resize(nt);
    ev_colrest.resize(nt);
    for (int k = 0; k < nt; ++k) SPH_CUDA(cudaEventCreateWithFlags(&ev_colrest[k], cudaEventDisableTiming));
    ev_bulkdp.resize(nt);
    for (int k = 0; k < nt; ++k) SPH_CUDA(cudaEventCreateWithFlags(&ev_bulkdp[k], cudaEventDisableTiming));
    for (int k = 0; k < nt; ++k) {
      SPH_CUDA(cudaEventCreateWithFlags(&ev_panel[k], cudaEventDisableTiming));
      SPH_CUDA(cudaEventCreateWithFlags(&ev_bulk[k], cudaEventDisableTiming));
    }
    SPH_CUDA(cudaEventCreateWithFlags(&ev_start_p, cudaEventDisableTiming));
    SPH_CUDA(cudaEventCreate(&ev0));
    SPH_CUDA(cudaEventCreate(&ev1));
  }

  ~Chol() {
    stop_expander();
    for (auto& t : zeroers) t.join();
    for (auto e : ev_grp) cudaEventDestroy(e);
    if (dstream) cudaStreamSynchronize(dstream);
    if (cstream) cudaStreamSynchronize(cstream);
    for (int s = 0; s < kSlabs; ++s) {
      if (ev_in_full[s]) cudaEventDestroy(ev_in_full[s]);
      if (ev_in_free[s]) cudaEventDestroy(ev_in_free[s]);
    }
    if (ev_col) cudaEventDestroy(ev_col);
    if (cstream) cudaStreamDestroy(cstream);
    if (dstream) cudaStreamDestroy(dstream);
    if (stream) cudaStreamSynchronize(stream);
    if (pstream) cudaStreamSynchronize(pstream);
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto e : ev_panel) cudaEventDestroy(e);
    for (auto e : ev_bulk) cudaEventDestroy(e);
    for (auto e : ev_colrest) cudaEventDestroy(e);
    for (auto e : ev_bulkdp) cudaEventDestroy(e);
    if (ev_start_p) cudaEventDestroy(ev_start_p);
    if (xstream) cudaStreamSynchronize(xstream);
    if (bstream) cudaStreamSynchronize(bstream);
    for (auto e : ev_p4) cudaEventDestroy(e);
    for (auto e : ev_p5) cudaEventDestroy(e);
    if (bstream) cudaStreamDestroy(bstream);
    if (ev_trdone) cudaEventDestroy(ev_trdone);
    for (auto e : ev_tr) cudaEventDestroy(e);
    if (ev_xdone) cudaEventDestroy(ev_xdone);
    if (xstream) cudaStreamDestroy(xstream);
    if (comm2) ncclCommDestroy(comm2);
    if (pstream) cudaStreamDestroy(pstream);
    if (comm) ncclCommDestroy(comm);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
  }

  void reset_flags() {
    SPH_CUDA(cudaMemsetAsync(fail.get(), 0xff, sizeof(int), stream));
    SPH_CUDA(cudaMemsetAsync(sat.get(), 0, sizeof(unsigned), stream));
  }

  dim3 tile_grid() const {
    return dim3(static_cast<unsigned>(pmap.size()), static_cast<unsigned>(std::max(1, b * b / (256 * 64))));
  }

  void load_dense(const double* a, int where, int64_t lda, double diag_shift = 0.0) {
    factored = false;
    reset_flags();
    const int pl = prof_begin(kLoad);
    if (where == SPHEMU_HOST) {
      load_host(a, lda, diag_shift);
    } else if (n % 8 == 0 && lb % 8 == 0 && lda % 2 == 0 && reinterpret_cast<uintptr_t>(a) % 16 == 0) {
      k_load_dense8<<<tile_grid(), 256, 0, stream>>>(store(), a, lda, sat.get(), diag_shift);
      SPH_LAUNCH_CHECK();
    } else {
      k_load_dense<<<tile_grid(), 256, 0, stream>>>(store(), a, lda, sat.get(), 0, 0, diag_shift);
      SPH_LAUNCH_CHECK();
    }
    k_rowexp<<<ceil_div(n, 256), 256, 0, stream>>>(store(), rowexp.get());
    SPH_LAUNCH_CHECK();
    if (dist()) SPH_NCCL(ncclAllReduce(rowexp.get(), rowexp.get(), n, ncclInt32, ncclMax, comm, stream));
    prof_end(pl);
    // device input: stream-ordered with the factorization, no host wait
    if (where == SPHEMU_HOST) SPH_CUDA(cudaStreamSynchronize(stream));
  }

  void generate_spd(uint64_t seed, double rho = 0.9);

  // The loaded tiles are a factor already (a stored model's V): usable by
  // trmm / emulate without factoring.
  void mark_factored() {
    SPH_CUDA(cudaEventRecord(ev0, stream));
    SPH_CUDA(cudaEventRecord(ev1, stream));
    launches = 0;
    factored = true;
  }

  // ---- the per-step operations, on a given stream and panel buffer set ----
  void op_potrf(int k, cudaStream_t s) {
    const int pe = prof_begin(kPotrf, s);
    launch_potrf(k, s);
    prof_end(pe, s);
  }

  // max_ctas caps the persistent tcgen05 grid. The chain's panel runs
  // uncapped: CTAs beyond the SMs the bulk leaves free start as soon as the
  // bulk's CTAs retire (measured faster than a capped panel: C2 62 vs 73 ms).
  void op_panel(int k, cudaStream_t s, int max_ctas = 0) {
    const int set = set_of(k);
    const int pp = prof_begin(kPanel, s);
    if (cfg.compute == SPHEMU_COMPUTE_TENSOR) {
      if (oz && !dist()) {
        oz_fused[k] = k < oz_fuse_frac() * nt;
        panel_[set].s8 = oz_fused[k] ? oz_[set].s8.get() : nullptr;
        panel_[set].no_p64 = true;
      }
      const int2* base = plists.get() + plist_off[k];
      tc_panel_trsm(store(), k, base, plist_dp[k], base + plist_dp[k], plist_lo[k], linv_[set].get(),
                    p64_[set].get(), panel_[set], fail.get(), sat.get(), s, max_ctas, ctr(s, 3),
                    base + plist_dp[k] + plist_lo[k], plist_bf[k]);
      if (!dist() && oz && !oz_fused[k]) oz_slice_next(k, s);
    } else {
      const int below = nt - k - 1;
      k_panel_trsm_fp64<<<dim3(below * (b / DG_BM), b / DG_BN), DG_THREADS, 0, s>>>(
          store(), k, linv_[set].get(), p64_[set].get(), fail.get(), sat.get());
      SPH_LAUNCH_CHECK();
      k_panel_scatter<<<dim3(std::max(1, b * b / (256 * 16)), below), 256, 0, s>>>(store(), k, p64_[set].get(),
                                                                                    fail.get());
      SPH_LAUNCH_CHECK();
    }
    prof_end(pp, s);
  }

  // The chain's single diagonal-tile SYRK is latency-bound: 64 x 64 CTAs
  // (36 active on a 512 tile) finish sooner than the 128 x 64 bulk kernel's 20.
  static bool chain_small_syrk() {
    static const bool on = [] {
      const char* e = std::getenv("SPHEMU_CHAIN_SYRK64");
      return !(e && e[0] == '0');
    }();
    return on;
  }

  // Classes whose panel TRSM and trailing updates run in FP64 (DMMA): the DP
  // class always; the SP class too under SPHEMU_SP_FP64 (exact-parity mode:
  // the tensor cores' truncating fp32 accumulation is what separates the
  // fp16x3 / 3xTF32 SP results from the FP64 oracle on ill-conditioned input).
  bool fp64_class(int cls) const {
    return cls == SPHEMU_PREC_DP || (cls == SPHEMU_PREC_SP && cfg.sp_compute == SPHEMU_SP_FP64);
  }

  // dp_done (optional): recorded on s once the DP-class launch of this part
  // is enqueued (before the SP / HP launches), so the chain can wait for the
  // DP diagonal tiles only.
  void op_update(int k, int part, cudaStream_t s, int max_ctas, const int* yield = nullptr, bool resume = false,
                 cudaEvent_t dp_done = nullptr) {
    const int set = set_of(k);
    const bool merged = part == 4 || part == 5;  // panels k and k+1 in one pass
    const int set2 = set_of(k + 1);
    for (int cls = 0; cls < 3; ++cls) {
      if (cls == 1 && dp_done) SPH_CUDA(cudaEventRecord(dp_done, s));
      const size_t slot = (static_cast<size_t>(k) * kParts + part) * 3 + cls;
      const int64_t cnt = list_cnt[slot];
      if (!cnt) continue;
      const int2* lst = lists.get() + list_off[slot];
      const bool tensor = !fp64_class(cls) && cfg.compute == SPHEMU_COMPUTE_TENSOR;
      if (resume && !tensor) continue;  // only the persistent tcgen05 launches yield
      static const bool log = [] {
        const char* e = std::getenv("SPHEMU_LAUNCH_LOG");  // profiling aid: which step / part each launch is
        return e && e[0] == '1';
      }();
      if (log)
        std::fprintf(stderr, "update k=%d part=%d cls=%d tiles=%lld merged=%d resume=%d\n", k, part, cls,
                     static_cast<long long>(cnt), merged ? 1 : 0, resume ? 1 : 0);
      const int pu = prof_begin(kUpdDp + cls, s);
      if (oz && cls == 0) {
        if (part != 0) {  // unless the panel epilogue wrote them
          if (!oz_fused[k]) oz_slice_rest(k, s);
          if (merged && !oz_fused[k + 1]) oz_slice_rest(k + 1, s);
        }
        oz_update(store(), k, lst, cnt, oz_[set], merged ? k + 1 : -1, merged ? &oz_[set2] : nullptr, rowexp.get(),
                  fail.get(), s, max_ctas, ctr(s, 0));
      } else if (tensor) {
        tc_update(store(), k, cls, cfg.hp_format, lst, lrows.get() + list_off[slot], cnt, p64_[set].get(),
                  panel_[set], fail.get(), sat.get(), s, max_ctas, ctr(s, cls), yield, resume, merged ? k + 1 : -1,
                  merged ? &panel_[set2] : nullptr);
      } else {
        if (b % D2_BM == 0 && !(part == 0 && chain_small_syrk())) {
          smem_optin(reinterpret_cast<const void*>(k_update_fp64_v2), (int)sizeof(D2Smem));
          const int per = (b / D2_BM) * (b / D2_BN);
          k_update_fp64_v2<<<static_cast<unsigned>(cnt * per), D2_THREADS, sizeof(D2Smem), s>>>(
              store(), k, lst, p64_[set].get(), fail.get(), sat.get(), merged ? k + 1 : -1,
              merged ? p64_[set2].get() : nullptr);
        } else {
          const int per = (b / DG_BM) * (b / DG_BN);
          k_update_fp64<<<static_cast<unsigned>(cnt * per), DG_THREADS, 0, s>>>(store(), k, lst, p64_[set].get(),
                                                                                 fail.get(), sat.get());
          if (merged) {  // the 64 x 64 kernel has no second K range: the second step as its own pass
            SPH_LAUNCH_CHECK();
            k_update_fp64<<<static_cast<unsigned>(cnt * per), DG_THREADS, 0, s>>>(store(), k + 1, lst,
                                                                                   p64_[set2].get(), fail.get(),
                                                                                   sat.get());
          }
        }
        SPH_LAUNCH_CHECK();
      }
      prof_end(pu, s);
    }
  }

  // tiled_cholesky (mpchol.cpp:351-410). Without lookahead every operation is
  // serialized on one stream. With lookahead the critical chain (update of
  // column k+1 -> POTRF(k+1) -> panel(k+1)) runs on a high-priority stream
  // while the bulk update of step k (columns >= k+2) runs on the main stream;
  // the two touch disjoint tiles, panel buffers alternate by step parity, and
  // every tile still receives its updates in k order (results are bitwise
  // identical with and without lookahead).
  void factor() {
    factored = false;
    if (xipc) xepoch += static_cast<uint32_t>(nt) + 2;
    xlate.assign(nt, 0);
    std::fill(oz_rest.begin(), oz_rest.end(), 0);
    launches_at_start = launch_count();
    t_start = std::chrono::steady_clock::now();
    SPH_CUDA(cudaEventRecord(ev0, stream));
    if (xipc) {
      // every rank's previous factorization (all streams) is done before any
      // owner refills an exchange half of this one: a device-side barrier
      SPH_CUDA(cudaEventRecord(ev_start_p, pstream));
      SPH_CUDA(cudaStreamWaitEvent(stream, ev_start_p, 0));
      if (xstream) {
        SPH_CUDA(cudaEventRecord(ev_xdone, xstream));
        SPH_CUDA(cudaStreamWaitEvent(stream, ev_xdone, 0));
      }
      SPH_NCCL(ncclAllReduce(xbar.get(), xbar.get(), 1, ncclInt32, ncclSum, comm, stream));
    }
    // SMs left to the chain while the bulk runs. Early steps, where the bulk
    // is the critical stream (its work shrinks quadratically, the chain's only
    // linearly), leave the chain 8 SMs; the last 32 steps leave it 32
    // (SPHEMU_RESERVE_EARLY / SPHEMU_RESERVE_TAIL). POTRF's cooperative grid
    // follows the reserve so its CTAs stay co-resident. Measured (1 GPU):
    // C2 58.2 -> 56.4 ms, C3 1 246 -> 1 136 ms against a fixed reserve of 32
    // (tools/reserve_sweep*.sh); with the INT8 DP class and the SP pairs
    // 8 stays best once short factorizations run their SP pairs dynamically
    // (yielding to the panel): C2 47.8 ms (16: 48.5); static pairs would want
    // 16 on C2 (48.8 vs 50.3) but 8 on C3 (905 vs 938) (tools/gpu_tasks.sh sweep).
    static const int r_early_env = [] {
      const char* e = std::getenv("SPHEMU_RESERVE_EARLY");
      return e ? std::max(8, std::min(kChainCtas, std::atoi(e))) : 0;
    }();
    const int r_early = r_early_env ? r_early_env : 8;
    static const int r_tail = [] {
      const char* e = std::getenv("SPHEMU_RESERVE_TAIL");
      return e ? std::atoi(e) : 32;
    }();
    auto reserve_at = [&](int k) { return (nt - 1 - k > r_tail) ? r_early : kChainCtas; };
    int reserve = kChainCtas;
    potrf_cap = kChainCtas;
    if (merge_on() && nt >= 3) {
      run_merged(reserve_at);
    } else if (dist()) {
      factor_dist();
    } else if (!cfg.lookahead || nt == 1) {
      for (int k = 0; k < nt; ++k) {
        op_potrf(k, stream);
        if (k + 1 >= nt) {
          col_out(k, stream);
          break;
        }
        op_panel(k, stream);
        col_out(k, stream);
        op_update(k, 0, stream, 0);
        op_update(k, 2, stream, 0);
        op_update(k, 1, stream, 0);
      }
    } else {
      SPH_CUDA(cudaEventRecord(ev_start_p, stream));
      SPH_CUDA(cudaStreamWaitEvent(pstream, ev_start_p, 0));
      op_potrf(0, pstream);
      op_panel(0, pstream);
      record_panel(0);
      col_out(0, pstream);
      for (int k = 0; k + 1 < nt; ++k) {
        // chain: SYRK of the next diagonal tile -> POTRF -> (column below ready) -> panel.
        // Tile (k+1, k+1) last changed in the DP-class launch of bulk(k-1):
        // the chain waits for that launch only, not for the SP / HP bulk
        // (panel(k+1) still waits for column k+1, after all of bulk(k-1)).
        if (k > 0) SPH_CUDA(cudaStreamWaitEvent(pstream, ev_bulkdp[k - 1], 0));
        reserve = reserve_at(k);
        potrf_cap = reserve;
        op_update(k, 0, pstream, 0);
        op_potrf(k + 1, pstream);
        // main stream: column k+1 below the diagonal first (the chain's panel
        // waits for it), then the bulk of step k on the SMs the chain leaves
        SPH_CUDA(cudaStreamWaitEvent(stream, ev_panel[k], 0));
        op_update(k, 2, stream, 0);
        SPH_CUDA(cudaEventRecord(ev_colrest[k], stream));
        const bool yield = yield_on() && k + 2 < nt;
        if (k + 2 < nt) {
          SPH_CUDA(cudaStreamWaitEvent(pstream, ev_colrest[k], 0));
          // the bulk of step k hands its SMs to panel(k+1) and resumes after it
          if (yield) SPH_CUDA(cudaMemsetAsync(yield_flag.get(), 1, sizeof(int), pstream));
          op_panel(k + 1, pstream);
          if (yield) SPH_CUDA(cudaMemsetAsync(yield_flag.get(), 0, sizeof(int), pstream));
        }
        record_panel(k + 1);
        col_out(k + 1, pstream);
        const int bulk_ctas = std::max(1, num_sms() - reserve);
        op_update(k, 1, stream, bulk_ctas, yield ? yield_flag.get() : nullptr, false, ev_bulkdp[k]);
        if (yield) {
          SPH_CUDA(cudaStreamWaitEvent(stream, ev_panel[k + 1], 0));
          op_update(k, 1, stream, bulk_ctas, nullptr, true);
        }
        SPH_CUDA(cudaEventRecord(ev_bulk[k], stream));
      }
      SPH_CUDA(cudaStreamWaitEvent(stream, ev_panel[nt - 1], 0));
    }
    SPH_CUDA(cudaEventRecord(ev1, stream));
    launches = launch_count() - launches_at_start;
    factored = true;
  }

  // Merged two-step schedule (default; SPHEMU_MERGE=0 restores one update
  // pass per step). Steps run in pairs (k, k+1): the chain factors both
  // diagonal tiles and solves both panels as before, the main stream updates
  // column k+2 with panel k alone (it feeds the chain's next step), and every
  // tile right of it receives both steps' updates in ONE pass
  // (C -= P_k Q_k^T + P_k+1 Q_k+1^T: one C round trip and one storage rounding
  // for the two steps — halving the trailing matrix's HBM traffic, which the
  // 16-bit update is bound by). Column k+3 goes first (it feeds the next
  // pair's chain), then the bulk. Same arithmetic with and without lookahead
  // and on any P x Q grid (the lists hold each rank's tiles).
  static bool merge_on() {
    static const bool on = [] {
      const char* e = std::getenv("SPHEMU_MERGE");
      return !(e && e[0] == '0');
    }();
    return on;
  }

  template <class ReserveFn>
  void run_merged(ReserveFn reserve_at) {
    const bool D = dist();
    auto potrf = [&](int k, cudaStream_t s) {
      if (D) op_potrf_dist(k, s);
      else op_potrf(k, s);
    };
    auto panel = [&](int k, cudaStream_t s) {
      if (D) op_panel_dist(k, s);
      else op_panel(k, s);
    };
    auto cols = [&](int k, cudaStream_t s) {
      if (!D) col_out(k, s);
    };
    // chain reserve: one GPU as reserve_at; the distributed chain also carries the exchange (factor_dist)
    const char* env_reserve = std::getenv("SPHEMU_DIST_RESERVE");
    // SMs left to the distributed chain. With the copy-engine exchange (no
    // NCCL kernels in the chain) and tile k+1 sent first, fewer is better:
    // C3 2x2 16 / 20 / 24 / 28 / 32 -> 293.5 / 294 / 298 / 300 / 304 ms, 2x1
    // 16 / 24 / 32 -> 478 / 491 / 510 ms (NCCL exchange, round 2 start: 32
    // best, 379 ms)
    const int dist_reserve = env_reserve ? std::atoi(env_reserve) : (xipc ? 16 : kChainCtas);
    // the last dist_tail steps (chain-bound: the bulk idles behind the panel
    // and exchange) leave the chain kChainCtas SMs, as on one GPU. C3 2x2:
    // 0 / 32 / 64 / 128 steps -> 283.6 / 278.6 / 278.0 / 278.7 ms; 2x1: 0 /
    // 64 -> 471.9 / 476.6 ms, so grids of 4+ ranks only.
    static const int dist_tail_env = [] {
      const char* e = std::getenv("SPHEMU_DIST_RESERVE_TAIL");
      return e ? std::atoi(e) : -1;
    }();
    const int dist_tail = dist_tail_env >= 0 ? dist_tail_env : (P * Q >= 4 ? 64 : 0);
    auto reserve_for = [&](int k) {
      return D ? (nt - 1 - k > dist_tail ? dist_reserve : std::max(dist_reserve, kChainCtas)) : reserve_at(k);
    };
    if (!cfg.lookahead) {
      potrf(0, stream);
      panel(0, stream);
      cols(0, stream);
      int k = 0;
      while (k + 1 < nt) {
        if (k + 2 < nt) {
          op_update(k, 0, stream, 0);
          op_update(k, 2, stream, 0);
          op_update(k, 3, stream, 0);
          potrf(k + 1, stream);
          panel(k + 1, stream);
          cols(k + 1, stream);
          op_update(k + 1, 0, stream, 0);
          op_update(k + 1, 2, stream, 0);
          op_update(k, 4, stream, 0);
          op_update(k, 5, stream, 0);
          potrf(k + 2, stream);
          if (k + 3 < nt) panel(k + 2, stream);
          cols(k + 2, stream);
          k += 2;
        } else {
          op_update(k, 0, stream, 0);
          potrf(k + 1, stream);
          cols(k + 1, stream);
          k += 1;
        }
      }
    } else {
      SPH_CUDA(cudaEventRecord(ev_start_p, stream));
      SPH_CUDA(cudaStreamWaitEvent(pstream, ev_start_p, 0));
      potrf(0, pstream);
      panel(0, pstream);
      record_panel(0);
      cols(0, pstream);
      cudaEvent_t diag_ready = nullptr;  // diagonal tile (k+1, k+1) has every update of steps < k
      auto yielding_panel = [&](int k, bool y) {
        if (y) SPH_CUDA(cudaMemsetAsync(yield_flag.get(), 1, sizeof(int), pstream));
        panel(k, pstream);
        if (y) SPH_CUDA(cudaMemsetAsync(yield_flag.get(), 0, sizeof(int), pstream));
      };
      int k = 0;
      static const int split5_env = [] {
        const char* e = std::getenv("SPHEMU_SPLIT5");  // SMs the main stream keeps while part 5 runs (0 = off)
        return e ? std::atoi(e) : -1;
      }();
      const bool split5 = bstream && (split5_env > 0 || (split5_env < 0 && D));
      const int split5_ctas = split5_env > 0 ? split5_env : 16;
      int last_p5 = -1;
      while (k + 1 < nt) {
        const int reserve = reserve_for(k);
        potrf_cap = std::min(kChainCtas, reserve);
        const int bulk_ctas = std::max(1, num_sms() - reserve);
        static const bool dist_yield = [] {
          const char* e = std::getenv("SPHEMU_DIST_YIELD");  // A/B: yielding bulk on process grids
          return e && e[0] == '1';
        }();
        const bool y = yield_on() && (!D || dist_yield);
        if (diag_ready) SPH_CUDA(cudaStreamWaitEvent(pstream, diag_ready, 0));
        op_update(k, 0, pstream, 0);
        potrf(k + 1, pstream);
        SPH_CUDA(cudaStreamWaitEvent(stream, ev_panel[k], 0));
        op_update(k, 2, stream, 0);
        SPH_CUDA(cudaEventRecord(ev_colrest[k], stream));
        if (k + 2 >= nt) {  // the last step: no panel below the last diagonal tile
          record_panel(k + 1);
          cols(k + 1, pstream);
          break;
        }
        // ---- step k: panel k+1 on the chain, column k+2 by panel k on the main stream
        SPH_CUDA(cudaStreamWaitEvent(pstream, ev_colrest[k], 0));
        yielding_panel(k + 1, y);
        record_panel(k + 1);
        cols(k + 1, pstream);
        // column k+2 last received the previous pair's merged update (part 5 of k-2)
        if (split5 && k >= 2) SPH_CUDA(cudaStreamWaitEvent(stream, ev_p5[k - 2], 0));
        op_update(k, 3, stream, bulk_ctas, y ? yield_flag.get() : nullptr);
        if (y) {
          SPH_CUDA(cudaStreamWaitEvent(stream, ev_panel[k + 1], 0));
          op_update(k, 3, stream, bulk_ctas, nullptr, true);
        }
        SPH_CUDA(cudaEventRecord(ev_bulkdp[k], stream));  // column k+2 done with panel k
        // ---- step k+1: its diagonal and column k+2, then both steps' updates right of it
        SPH_CUDA(cudaStreamWaitEvent(pstream, ev_bulkdp[k], 0));
        op_update(k + 1, 0, pstream, 0);
        potrf(k + 2, pstream);
        SPH_CUDA(cudaStreamWaitEvent(stream, ev_panel[k + 1], 0));
        op_update(k + 1, 2, stream, 0);
        SPH_CUDA(cudaEventRecord(ev_colrest[k + 1], stream));
        const bool more = k + 3 < nt;
        if (more) {
          SPH_CUDA(cudaStreamWaitEvent(pstream, ev_colrest[k + 1], 0));
          yielding_panel(k + 2, y);
        }
        record_panel(k + 2);
        cols(k + 2, pstream);
        op_update(k, 4, stream, 0);  // column k+3: feeds the next pair's chain
        SPH_CUDA(cudaEventRecord(ev_bulk[k + 1], stream));
        diag_ready = ev_bulk[k + 1];
        if (split5) {
          // the right of column k+3 on its own stream (leaving SMs to the next
          // pair's column updates on the main stream)
          SPH_CUDA(cudaEventRecord(ev_p4[k], stream));
          SPH_CUDA(cudaStreamWaitEvent(bstream, ev_p4[k], 0));
          op_update(k, 5, bstream, std::max(1, bulk_ctas - split5_ctas));
          SPH_CUDA(cudaEventRecord(ev_p5[k], bstream));
          last_p5 = k;
        } else {
          op_update(k, 5, stream, bulk_ctas, (y && more) ? yield_flag.get() : nullptr);
          if (y && more) {
            SPH_CUDA(cudaStreamWaitEvent(stream, ev_panel[k + 2], 0));
            op_update(k, 5, stream, bulk_ctas, nullptr, true);
          }
        }
        SPH_CUDA(cudaEventRecord(ev_bulk[k], stream));
        k += 2;
      }
      if (last_p5 >= 0) SPH_CUDA(cudaStreamWaitEvent(stream, ev_p5[last_p5], 0));
      SPH_CUDA(cudaStreamWaitEvent(stream, ev_panel[nt - 1], 0));
    }
    if (D && xstream) {  // the last exchange's acknowledgements are part of the factorization
      SPH_CUDA(cudaEventRecord(ev_xdone, xstream));
      SPH_CUDA(cudaStreamWaitEvent(stream, ev_xdone, 0));
    }
    if (D) SPH_NCCL(ncclAllReduce(sat.get(), sat.get(), 1, ncclUint32, ncclSum, comm, stream));
  }

  // 2D block-cyclic step sequence (PAPER.md:570 pattern): the owner of
  // (k,k) factors it and broadcasts L_kk^{-1} (and the failure flag); the
  // process column k mod Q computes its panel tiles; every panel tile is
  // broadcast at its storage precision (the minimal bytes, rounded at the
  // sender) and receivers rebuild the FP64 / tensor-core operand mirrors;
  // every rank updates the trailing tiles it owns.
  // POTRF(k) on the owner of (k,k), then the failure flag and L_kk^{-1}
  // broadcast from it.
  void op_potrf_dist(int k, cudaStream_t s) {
    const int ok = owner(k, k);
    if (rank == ok) op_potrf(k, s);
    SPH_NCCL(ncclBroadcast(fail.get(), fail.get(), 1, ncclInt32, ok, comm, s));
    if (k + 1 < nt) {
      const int set = set_of(k);
      SPH_NCCL(ncclBroadcast(linv_[set].get(), linv_[set].get(), static_cast<size_t>(b) * b, ncclFloat64, ok, comm, s));
    }
    note_launch(2);
  }

  // Panel TRSM on the owned panel tiles, then every panel tile broadcast at
  // its storage precision and imported into the operand mirrors elsewhere.
  void ipc_setup() {
    const int W = P * Q;
    xbar.alloc(1);
    SPH_CUDA(cudaMemset(xbar.get(), 0, sizeof(int)));
    xsync.alloc(2 + W);  // [0] published step, [1 + r] acks, [1 + W] tile k+1 published early
    SPH_CUDA(cudaMemset(xsync.get(), 0, (2 + W) * sizeof(uint32_t)));
    cudaIpcMemHandle_t mine[2];
    SPH_CUDA(cudaIpcGetMemHandle(&mine[0], xbuf.get()));
    SPH_CUDA(cudaIpcGetMemHandle(&mine[1], xsync.get()));
    DevBuf<uint8_t> all(sizeof(mine) * W);
    DevBuf<uint8_t> one(sizeof(mine));
    SPH_CUDA(cudaMemcpy(one.get(), mine, sizeof(mine), cudaMemcpyHostToDevice));
    SPH_NCCL(ncclAllGather(one.get(), all.get(), sizeof(mine), ncclUint8, comm, stream));
    SPH_CUDA(cudaStreamSynchronize(stream));
    std::vector<cudaIpcMemHandle_t> hs(2 * W);
    SPH_CUDA(cudaMemcpy(hs.data(), all.get(), sizeof(mine) * W, cudaMemcpyDeviceToHost));
    peer_xbuf.assign(W, nullptr);
    peer_sync.assign(W, nullptr);
    for (int r = 0; r < W; ++r) {
      if (r == rank) {
        peer_xbuf[r] = xbuf.get();
        peer_sync[r] = xsync.get();
        continue;
      }
      void* pb = nullptr;
      void* ps = nullptr;
      SPH_CUDA(cudaIpcOpenMemHandle(&pb, hs[2 * r], cudaIpcMemLazyEnablePeerAccess));
      SPH_CUDA(cudaIpcOpenMemHandle(&ps, hs[2 * r + 1], cudaIpcMemLazyEnablePeerAccess));
      peer_xbuf[r] = static_cast<uint8_t*>(pb);
      peer_sync[r] = static_cast<uint32_t*>(ps);
    }
  }
  // Stream memory operations through the runtime's driver entry points (the
  // library does not link libcuda: it must load on hosts without a driver).
  using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static StreamValueFn driver_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      throw Error(SPHEMU_ERR_CUDA, std::string(name) + " unavailable");
    return reinterpret_cast<StreamValueFn>(p);
  }
  static void stream_write(cudaStream_t s, uint32_t* addr, uint32_t v) {
    static const StreamValueFn fn = driver_fn("cuStreamWriteValue32");
    const CUresult r = fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                          CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) throw Error(SPHEMU_ERR_CUDA, "cuStreamWriteValue32 failed: " + std::to_string(r));
  }
  static void stream_wait_geq(cudaStream_t s, uint32_t* addr, uint32_t v) {
    static const StreamValueFn fn = driver_fn("cuStreamWaitValue32");
    const CUresult r = fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), v,
                          CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) throw Error(SPHEMU_ERR_CUDA, "cuStreamWaitValue32 failed: " + std::to_string(r));
  }

  // The copy-engine exchange of step k's panel (see xipc): owners pack and
  // publish, readers pull every other owner's block, import, acknowledge.
  void xchg_ipc(int k, cudaStream_t s) {
    const int W = P * Q;
    const uint32_t ep = xepoch + static_cast<uint32_t>(k) + 1;
    const int64_t par = (k & 1) * xhalf;
    uint8_t* own = xbuf.get() + par;
    const unsigned gx = static_cast<unsigned>(std::max(1, b * b / (256 * 16)));
    if (xsend_cnt[k]) {
      // the half this step packs into was last read by the readers at step k-2
      if (k >= 2)
        for (int q = 0; q < W; ++q)
          if (q != rank) stream_wait_geq(s, xsync.get() + 1 + q, ep - 2);
      k_panel_pack<<<dim3(gx, static_cast<unsigned>(xsend_cnt[k])), 256, 0, s>>>(
          store(), k, xsend.get() + xsend_off[k], xsoffs.get() + xsend_off[k], own, fail.get());
      SPH_LAUNCH_CHECK();
      stream_write(s, xsync.get(), ep);
    }
    for (const Xfer& x : xroots[k]) {
      if (x.peer == rank) continue;
      stream_wait_geq(s, peer_sync[x.peer], ep);
      SPH_CUDA(cudaMemcpyAsync(own + x.pos, peer_xbuf[x.peer] + par + x.pos, static_cast<size_t>(x.bytes),
                               cudaMemcpyDeviceToDevice, s));
    }
    note_launch();
  }

  // Chunked form of op_panel_dist (broadcast mode, tensor compute): the
  // column below the diagonal is cut into xchunks slices by tile row; slice c's
  // TRSM (this rank's tiles of it) runs on the chain stream s while slice c-1
  // is packed, broadcast per owner on comm2 and imported on xstream, so the
  // exchange hides behind the TRSM. Slices are a function of the tile index
  // only, so every rank issues the same collectives in the same order.
  void op_panel_dist_chunked(int k, cudaStream_t s, int max_ctas) {
    const int set = set_of(k);
    const int below = nt - k - 1;
    const int C = std::min(xchunks, below);
    auto chunk_of = [&](int i) { return static_cast<int>((static_cast<int64_t>(i - k - 1) * C) / below); };
    // sub-range [lo, hi) of a tile-row-sorted list segment holding chunk c
    auto sub = [&](const std::vector<int>& rows, int64_t off, int64_t cnt, int c, int64_t& lo, int64_t& hi) {
      lo = off;
      while (lo < off + cnt && chunk_of(rows[lo]) < c) ++lo;
      hi = lo;
      while (hi < off + cnt && chunk_of(rows[hi]) == c) ++hi;
    };
    PanelFormats& pf = panel_[set];
    const unsigned gx = static_cast<unsigned>(std::max(1, b * b / (256 * 16)));
    const int2* pbase = plists.get() + plist_off[k];
    const int64_t lo_off = plist_off[k] + plist_dp[k];
    const int pp = prof_begin(kPanel, s);
    for (int c = 0; c < C; ++c) {
      int64_t a, z;
      sub(pl_i, lo_off, plist_lo[k], c, a, z);
      if (c == 0 || z > a)
        tc_panel_trsm(store(), k, pbase, c == 0 ? plist_dp[k] : 0, plists.get() + a, z - a, linv_[set].get(),
                      p64_[set].get(), pf, fail.get(), sat.get(), s, max_ctas, ctr(s, 3));
      SPH_CUDA(cudaEventRecord(ev_tr[c], s));
    }
    prof_end(pp, s);
    const int px = prof_begin(kXchg, xstream);
    for (int c = 0; c < C; ++c) {
      SPH_CUDA(cudaStreamWaitEvent(xstream, ev_tr[c], 0));
      int64_t a, z;
      sub(xs_i, xsend_off[k], xsend_cnt[k], c, a, z);
      if (z > a) {
        k_panel_pack<<<dim3(gx, static_cast<unsigned>(z - a)), 256, 0, xstream>>>(
            store(), k, xsend.get() + a, xsoffs.get() + a, xbuf.get(), fail.get());
        SPH_LAUNCH_CHECK();
      }
      bool any = false;
      for (const Xfer& x : xroots[k]) {
        int64_t lo = -1, hi = -1;
        for (int i = k + 1; i < nt; ++i)
          if (owner(i, k) == x.peer && chunk_of(i) == c) {
            const int64_t p0 = xpos_h[k][i - k - 1];
            const int64_t p1 = p0 + static_cast<int64_t>(b) * b * prec_bytes(sprec[tix(i, k)]);
            lo = lo < 0 ? p0 : std::min(lo, p0);
            hi = std::max(hi, p1);
          }
        if (lo < 0) continue;
        if (!any) SPH_NCCL(ncclGroupStart());
        any = true;
        SPH_NCCL(ncclBroadcast(xbuf.get() + lo, xbuf.get() + lo, static_cast<size_t>(hi - lo), ncclUint8, x.peer,
                               comm2, xstream));
      }
      if (any) SPH_NCCL(ncclGroupEnd());
      note_launch();
      sub(il_i, ilist_off[k], ilist_cnt[k], c, a, z);
      if (z > a) {
        const bool tensor = cfg.compute == SPHEMU_COMPUTE_TENSOR;
        k_panel_import<<<dim3(gx, static_cast<unsigned>(z - a)), 256, 0, xstream>>>(
            store(), k, ilists.get() + a, ioffs.get() + a, xbuf.get(), p64_[set].get(), tensor ? pf.tf32_hi() : nullptr,
            tensor ? pf.tf32_lo() : nullptr, tensor ? pf.half16() : nullptr,
            (tensor && pf.f16x3) ? pf.h_hi.get() : nullptr, (tensor && pf.f16x3) ? pf.h_lo.get() : nullptr,
            rowexp.get(), cfg.hp_format, d_import_need.get(), fail.get());
        SPH_LAUNCH_CHECK();
      }
    }
    oz_slice_next(k, xstream);
    prof_end(px, xstream);
    SPH_CUDA(cudaEventRecord(ev_xdone, xstream));
    SPH_CUDA(cudaStreamWaitEvent(s, ev_xdone, 0));
  }

  // Copy-engine exchange with tile k+1 first (see xlate): on the chain stream
  // s, tile (k+1, k)'s TRSM, pack and early publish; its pull + import on the
  // next diagonal's owner (+ its digits); then the rest of this rank's TRSM,
  // pack and publish. The pulls of the other owners' blocks, the import and
  // the acknowledgements run on xstream, so the chain's next SYRK / POTRF
  // overlap them; ev_panel[k] is recorded on xstream (record_panel).
  void op_panel_dist_early(int k, cudaStream_t s, int max_ctas) {
    const int set = set_of(k);
    const int W = P * Q;
    const uint32_t ep = xepoch + static_cast<uint32_t>(k) + 1;
    const int64_t par = (k & 1) * xhalf;
    uint8_t* own = xbuf.get() + par;
    const unsigned gx = static_cast<unsigned>(std::max(1, b * b / (256 * 16)));
    PanelFormats& pf = panel_[set];
    const bool tensor = cfg.compute == SPHEMU_COMPUTE_TENSOR;
    const int i1 = k + 1;
    const int o1 = owner(i1, k), d1 = owner(i1, i1);
    // the per-class panel lists are sorted by tile row: i1 can only be a list's first entry
    const int64_t off = plist_off[k], ndp = plist_dp[k], nlo = plist_lo[k], nbf = plist_bf[k];
    const int2* L = plists.get();
    auto first_is = [&](int64_t o, int64_t n) { return n > 0 && pl_i[o] == i1; };
    const bool in_dp = first_is(off, ndp), in_lo = first_is(off + ndp, nlo), in_bf = first_is(off + ndp + nlo, nbf);
    const int pp = prof_begin(kPanel, s);
    if (k >= 2 && xsend_cnt[k])  // this parity half was last read at step k-2
      for (int q = 0; q < W; ++q)
        if (q != rank) stream_wait_geq(s, xsync.get() + 1 + q, ep - 2);
    const bool mine1 = in_dp || in_lo || in_bf;
    if (!tensor) op_panel(k, s, max_ctas);  // FP64 compute: the whole column first
    if (mine1) {
      if (tensor)
        tc_panel_trsm(store(), k, L + off, in_dp ? 1 : 0, L + off + ndp, in_lo ? 1 : 0, linv_[set].get(),
                      p64_[set].get(), pf, fail.get(), sat.get(), s, max_ctas, ctr(s, 3), L + off + ndp + nlo,
                      in_bf ? 1 : 0);
      // the early pack: xsend is sorted by tile row, i1 is its first entry
      k_panel_pack<<<dim3(gx, 1), 256, 0, s>>>(store(), k, xsend.get() + xsend_off[k], xsoffs.get() + xsend_off[k],
                                               own, fail.get());
      SPH_LAUNCH_CHECK();
      stream_write(s, xsync.get() + 1 + W, ep);
    }
    if (d1 == rank && o1 != rank) {  // the next diagonal's SYRK reads tile (k+1, k)'s rows
      const int64_t x1 = xpos_h[k][0];
      const int64_t by = static_cast<int64_t>(b) * b * prec_bytes(sprec[tix(i1, k)]);
      stream_wait_geq(s, peer_sync[o1] + 1 + W, ep);
      SPH_CUDA(cudaMemcpyAsync(own + x1, peer_xbuf[o1] + par + x1, static_cast<size_t>(by), cudaMemcpyDeviceToDevice, s));
      // ilist is sorted by tile row too: i1 is its first entry here
      k_panel_import<<<dim3(gx, 1), 256, 0, s>>>(
          store(), k, ilists.get() + ilist_off[k], ioffs.get() + ilist_off[k], own, p64_[set].get(),
          tensor ? pf.tf32_hi() : nullptr, tensor ? pf.tf32_lo() : nullptr, tensor ? pf.half16() : nullptr,
          (tensor && pf.f16x3) ? pf.h_hi.get() : nullptr, (tensor && pf.f16x3) ? pf.h_lo.get() : nullptr,
          rowexp.get(), cfg.hp_format, d_import_need.get(), fail.get());
      SPH_LAUNCH_CHECK();
    }
    if (d1 == rank) oz_slice_next(k, s);  // the chain's own diagonal SYRK (other readers: after the import)
    // the rest of this rank's column
    if (tensor)
      tc_panel_trsm(store(), k, L + off + (in_dp ? 1 : 0), ndp - (in_dp ? 1 : 0), L + off + ndp + (in_lo ? 1 : 0),
                    nlo - (in_lo ? 1 : 0), linv_[set].get(), p64_[set].get(), pf, fail.get(), sat.get(), s, max_ctas,
                    ctr(s, 3), L + off + ndp + nlo + (in_bf ? 1 : 0), nbf - (in_bf ? 1 : 0));
    if (xsend_cnt[k]) {
      const int64_t skip = mine1 ? 1 : 0;
      if (xsend_cnt[k] > skip) {
        k_panel_pack<<<dim3(gx, static_cast<unsigned>(xsend_cnt[k] - skip)), 256, 0, s>>>(
            store(), k, xsend.get() + xsend_off[k] + skip, xsoffs.get() + xsend_off[k] + skip, own, fail.get());
        SPH_LAUNCH_CHECK();
      }
      stream_write(s, xsync.get(), ep);
    }
    prof_end(pp, s);
    SPH_CUDA(cudaEventRecord(ev_trdone, s));
    // pulls, import and acknowledgements off the chain
    SPH_CUDA(cudaStreamWaitEvent(xstream, ev_trdone, 0));
    const int px = prof_begin(kXchg, xstream);
    for (const Xfer& x : xroots[k]) {
      if (x.peer == rank) continue;
      stream_wait_geq(xstream, peer_sync[x.peer], ep);
      SPH_CUDA(cudaMemcpyAsync(own + x.pos, peer_xbuf[x.peer] + par + x.pos, static_cast<size_t>(x.bytes),
                               cudaMemcpyDeviceToDevice, xstream));
    }
    note_launch();
    if (ilist_cnt[k]) {
      const int64_t skip = (d1 == rank && o1 != rank) ? 1 : 0;  // imported early already
      if (ilist_cnt[k] > skip) {
        k_panel_import<<<dim3(gx, static_cast<unsigned>(ilist_cnt[k] - skip)), 256, 0, xstream>>>(
            store(), k, ilists.get() + ilist_off[k] + skip, ioffs.get() + ilist_off[k] + skip, own, p64_[set].get(),
            tensor ? pf.tf32_hi() : nullptr, tensor ? pf.tf32_lo() : nullptr, tensor ? pf.half16() : nullptr,
            (tensor && pf.f16x3) ? pf.h_hi.get() : nullptr, (tensor && pf.f16x3) ? pf.h_lo.get() : nullptr,
            rowexp.get(), cfg.hp_format, d_import_need.get(), fail.get());
        SPH_LAUNCH_CHECK();
      }
    }
    if (d1 != rank) oz_slice_next(k, xstream);
    for (int q = 0; q < W; ++q)
      if (q != rank) stream_write(xstream, peer_sync[q] + 1 + rank, ep);
    prof_end(px, xstream);
    xlate[k] = 1;
    if (s != pstream) {  // no lookahead: the caller's stream sees the whole panel
      SPH_CUDA(cudaEventRecord(ev_xdone, xstream));
      SPH_CUDA(cudaStreamWaitEvent(s, ev_xdone, 0));
      xlate[k] = 0;
    }
  }

  void op_panel_dist(int k, cudaStream_t s, int max_ctas = 0) {
    const int set = set_of(k);
    static const bool early = [] {
      const char* e = std::getenv("SPHEMU_XCHG_EARLY");
      return !(e && e[0] == '0');
    }();
    if (xipc && early && xstream) {
      op_panel_dist_early(k, s, max_ctas);
      return;
    }
    if (xchunks > 1 && xstream && cfg.compute == SPHEMU_COMPUTE_TENSOR && !panel_bf) {
      op_panel_dist_chunked(k, s, max_ctas);
      return;
    }
    op_panel(k, s, max_ctas);
    const int px = prof_begin(kXchg, s);
    const unsigned gx = static_cast<unsigned>(std::max(1, b * b / (256 * 16)));
    if (xipc) {
      xchg_ipc(k, s);
    } else {
    if (xsend_cnt[k]) {
      k_panel_pack<<<dim3(gx, static_cast<unsigned>(xsend_cnt[k])), 256, 0, s>>>(
          store(), k, xsend.get() + xsend_off[k], xsoffs.get() + xsend_off[k], xbuf.get(), fail.get());
      SPH_LAUNCH_CHECK();
    }
    SPH_NCCL(ncclGroupStart());
    if (xchg_bcast()) {
      for (const Xfer& x : xroots[k])
        SPH_NCCL(ncclBroadcast(xbuf.get() + x.pos, xbuf.get() + x.pos, static_cast<size_t>(x.bytes), ncclUint8, x.peer,
                               comm, s));
    } else {
      for (const Xfer& x : xsends[k])
        SPH_NCCL(ncclSend(xbuf.get() + x.pos, static_cast<size_t>(x.bytes), ncclUint8, x.peer, comm, s));
      for (const Xfer& x : xrecvs[k])
        SPH_NCCL(ncclRecv(xbuf.get() + x.pos, static_cast<size_t>(x.bytes), ncclUint8, x.peer, comm, s));
    }
    SPH_NCCL(ncclGroupEnd());
    note_launch();
    }
    const uint8_t* xsrc = xbuf.get() + (xipc ? (k & 1) * xhalf : 0);
    if (ilist_cnt[k]) {
      PanelFormats& pf = panel_[set];
      const bool tensor = cfg.compute == SPHEMU_COMPUTE_TENSOR;
      k_panel_import<<<dim3(gx, static_cast<unsigned>(ilist_cnt[k])), 256, 0, s>>>(
          store(), k, ilists.get() + ilist_off[k], ioffs.get() + ilist_off[k], xsrc, p64_[set].get(), tensor ? pf.tf32_hi() : nullptr,
          tensor ? pf.tf32_lo() : nullptr, tensor ? pf.half16() : nullptr,
          (tensor && pf.f16x3) ? pf.h_hi.get() : nullptr, (tensor && pf.f16x3) ? pf.h_lo.get() : nullptr,
          rowexp.get(), cfg.hp_format, d_import_need.get(), fail.get());
      SPH_LAUNCH_CHECK();
    }
    if (xipc)  // the pulled blocks are consumed: every owner may refill this parity at step k+2
      for (int q = 0; q < P * Q; ++q)
        if (q != rank) stream_write(s, peer_sync[q] + 1 + rank, xepoch + static_cast<uint32_t>(k) + 1);
    // tile k+1's digits (the chain's diagonal SYRK of the next step), once
    // its panel rows are here
    oz_slice_next(k, s);
    prof_end(px, s);
  }

  // 2D block-cyclic step sequence (PAPER.md:570 pattern): the owner of
  // (k,k) factors it and broadcasts L_kk^{-1} (and the failure flag); the
  // process column k mod Q computes its panel tiles; every panel tile is
  // broadcast at its storage precision (the minimal bytes, rounded at the
  // sender) and receivers rebuild the FP64 / tensor-core operand mirrors;
  // every rank updates the trailing tiles it owns. With lookahead the whole
  // chain (column k+1 update, POTRF, broadcasts, panel, exchange, import)
  // runs on the high-priority stream, all collectives in step order, while
  // the bulk update of step k runs on the main stream.
  void factor_dist() {
    if (!cfg.lookahead || nt == 1) {
      for (int k = 0; k < nt; ++k) {
        op_potrf_dist(k, stream);
        if (k + 1 >= nt) break;
        op_panel_dist(k, stream);
        op_update(k, 0, stream, 0);
        op_update(k, 2, stream, 0);
        op_update(k, 1, stream, 0);
      }
    } else {
      // SMs left free for the chain while the bulk runs: the distributed chain
      // also carries the panel exchange and import, and each rank's bulk
      // shrinks with the grid (SPHEMU_DIST_RESERVE overrides).
      // measured C3: 2x1 grid 32 -> 749 ms, 48 -> 816; 2x2 grid 32 -> 501, 48 -> 488, 64 -> 515
      const char* env_reserve = std::getenv("SPHEMU_DIST_RESERVE");
      const int reserve_late = env_reserve ? std::atoi(env_reserve) : (P * Q >= 4 ? 48 : kChainCtas);
      // early steps may leave the chain fewer SMs, as on one GPU
      const char* env_early = std::getenv("SPHEMU_DIST_RESERVE_EARLY");
      const char* env_tail = std::getenv("SPHEMU_DIST_RESERVE_TAIL");
      const int reserve_early = env_early ? std::max(8, std::atoi(env_early)) : reserve_late;
      const int tail = env_tail ? std::atoi(env_tail) : 32;
      int reserve = reserve_late;
      SPH_CUDA(cudaEventRecord(ev_start_p, stream));
      SPH_CUDA(cudaStreamWaitEvent(pstream, ev_start_p, 0));
      op_potrf_dist(0, pstream);
      op_panel_dist(0, pstream);
      record_panel(0);
      for (int k = 0; k + 1 < nt; ++k) {
        if (k > 0) SPH_CUDA(cudaStreamWaitEvent(pstream, ev_bulk[k - 1], 0));
        reserve = (nt - 1 - k > tail) ? reserve_early : reserve_late;
        potrf_cap = std::min(kChainCtas, reserve);
        op_update(k, 0, pstream, 0);
        op_potrf_dist(k + 1, pstream);
        SPH_CUDA(cudaStreamWaitEvent(stream, ev_panel[k], 0));
        op_update(k, 2, stream, 0);  // no collectives on the main stream
        SPH_CUDA(cudaEventRecord(ev_colrest[k], stream));
        if (k + 2 < nt) {
          SPH_CUDA(cudaStreamWaitEvent(pstream, ev_colrest[k], 0));
          op_panel_dist(k + 1, pstream);
        }
        record_panel(k + 1);
        op_update(k, 1, stream, std::max(1, num_sms() - reserve));
        SPH_CUDA(cudaEventRecord(ev_bulk[k], stream));
      }
      SPH_CUDA(cudaStreamWaitEvent(stream, ev_panel[nt - 1], 0));
    }
    if (xstream) {  // the last exchange's acknowledgements are part of the factorization
      SPH_CUDA(cudaEventRecord(ev_xdone, xstream));
      SPH_CUDA(cudaStreamWaitEvent(stream, ev_xdone, 0));
    }
    SPH_NCCL(ncclAllReduce(sat.get(), sat.get(), 1, ncclUint32, ncclSum, comm, stream));
  }

  // Diagonal tile factor + inverse on a cooperative grid (potrf_coop.cuh).
  void launch_potrf(int k, cudaStream_t s) {
    const size_t smem = potrf_coop_smem();
    smem_optin(reinterpret_cast<const void*>(k_potrf_coop), (int)smem);
    const int nblk = (rows(k) + PC_BLK - 1) / PC_BLK;
    const int G = std::max(1, std::min(potrf_cap, nblk * (nblk + 1) / 2));
    double* dkk = reinterpret_cast<double*>(arena.get() + off[tix(k, k)]);
    int bk = rows(k), kk = k, bb = b;
    double* lp = linv_[set_of(k)].get();
    double* dp = dinv.get();
    int* fp = fail.get();
    unsigned* bp = pc_bar.get();
    void* args[] = {&dkk, &bb, &bk, &lp, &dp, &fp, &kk, &bp};
    SPH_CUDA(cudaLaunchCooperativeKernel((void*)k_potrf_coop, dim3(G), dim3(DG_THREADS), args, smem, s));
    note_launch();
  }

  // Reads the failure flag; fills stats (mpchol.cpp:376-409).
  int wait(sphemu_chol_stats* st) {
    SPH_CUDA(cudaStreamSynchronize(pstream));
    SPH_CUDA(cudaStreamSynchronize(stream));
    int f = -1;
    unsigned s = 0;
    SPH_CUDA(cudaMemcpy(&f, fail.get(), sizeof(int), cudaMemcpyDeviceToHost));
    SPH_CUDA(cudaMemcpy(&s, sat.get(), sizeof(unsigned), cudaMemcpyDeviceToHost));
    prof_fold();
    if (st) fill_stats(st, s);
    return f;
  }

  // ---- emulation: Xi = H L^T over the stored tiles (trmm.cu) ----------------
  // Host plan per class, built on first use: DP tiles by band offset, SP / HP
  // tiles as CSR rows (j, first row of the tile in the class's A tensor map).
  struct TrmmPlan {
    bool built = false;
    std::vector<std::vector<int2>> dp_by_offset;
    std::vector<DevBuf<int2>> d_dp;
    std::vector<int> row_ptr[2];  // [0] SP, [1] HP
    std::vector<int2> ent[2];
    DevBuf<int> d_row_ptr[2];
    DevBuf<int2> d_ent[2];
    std::vector<int2> sp_tiles;
    DevBuf<int2> d_sp_tiles;
    DevBuf<uint16_t> sp_hi, sp_lo;  // fp16 split of the SP tiles (row-scaled), refreshed per call
    CUtensorMap m_arena16{}, m_sp_hi{}, m_sp_lo{};
    DevBuf<double> hp;
    DevBuf<uint16_t> h16[2][2];  // [fmt fp16 / bf16][hi / lo]
    int64_t h_cols = 0;
  } tp;

  void trmm_build() {
    if (tp.built) return;
    int max_off = 0;
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j <= i; ++j)
        if (pmap[tix(i, j)] == SPHEMU_PREC_DP && mine(i, j)) max_off = std::max(max_off, i - j);
    tp.dp_by_offset.assign(max_off + 1, {});
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j <= i; ++j)
        if (pmap[tix(i, j)] == SPHEMU_PREC_DP && mine(i, j)) tp.dp_by_offset[i - j].push_back(make_int2(i, j));
    tp.d_dp.resize(tp.dp_by_offset.size());
    for (size_t q = 0; q < tp.dp_by_offset.size(); ++q) {
      const auto& v = tp.dp_by_offset[q];
      if (v.empty()) continue;
      tp.d_dp[q].alloc(v.size());
      SPH_CUDA(cudaMemcpy(tp.d_dp[q].get(), v.data(), v.size() * sizeof(int2), cudaMemcpyHostToDevice));
    }
    for (int c = 0; c < 2; ++c) {
      const int cls = c == 0 ? SPHEMU_PREC_SP : SPHEMU_PREC_HP;
      tp.row_ptr[c].assign(nt + 1, 0);
      tp.ent[c].clear();
      for (int i = 0; i < nt; ++i) {
        tp.row_ptr[c][i] = static_cast<int>(tp.ent[c].size());
        for (int j = 0; j < i; ++j) {
          if (pmap[tix(i, j)] != cls || !mine(i, j)) continue;
          int arow;
          if (c == 0) {
            arow = static_cast<int>(tp.sp_tiles.size()) * b;
            tp.sp_tiles.push_back(make_int2(i, j));
          } else {
            arow = static_cast<int>(off[tix(i, j)] / (2 * static_cast<int64_t>(b)));
          }
          tp.ent[c].push_back(make_int2(j, arow));
        }
      }
      tp.row_ptr[c][nt] = static_cast<int>(tp.ent[c].size());
      tp.d_row_ptr[c].alloc(nt + 1);
      SPH_CUDA(cudaMemcpy(tp.d_row_ptr[c].get(), tp.row_ptr[c].data(), (nt + 1) * sizeof(int),
                          cudaMemcpyHostToDevice));
      if (!tp.ent[c].empty()) {
        tp.d_ent[c].alloc(tp.ent[c].size());
        SPH_CUDA(cudaMemcpy(tp.d_ent[c].get(), tp.ent[c].data(), tp.ent[c].size() * sizeof(int2),
                            cudaMemcpyHostToDevice));
      }
    }
    if (!tp.sp_tiles.empty()) {
      tp.d_sp_tiles.alloc(tp.sp_tiles.size());
      SPH_CUDA(cudaMemcpy(tp.d_sp_tiles.get(), tp.sp_tiles.data(), tp.sp_tiles.size() * sizeof(int2),
                          cudaMemcpyHostToDevice));
      const size_t el = tp.sp_tiles.size() * static_cast<size_t>(b) * b;
      tp.sp_hi.alloc(el);
      tp.sp_lo.alloc(el);
      const int64_t rows = static_cast<int64_t>(tp.sp_tiles.size()) * b;
      tp.m_sp_hi = make_map_strided(tp.sp_hi.get(), rows, b, 2 * static_cast<int64_t>(b), 2, 128);
      tp.m_sp_lo = make_map_strided(tp.sp_lo.get(), rows, b, 2 * static_cast<int64_t>(b), 2, 128);
    }
    tp.m_arena16 = make_map_strided(arena.get(), static_cast<int64_t>(arena.n) / (2 * b), b,
                                    2 * static_cast<int64_t>(b), 2, 128);
    tp.built = true;
  }

  // Xi (S x n, row-major FP64) = H (S x n) L^T on stream s, over the tiles
  // this rank stores (the caller reduces across ranks). The factorization
  // must have been enqueued (and waited for) before.
  void trmm(const double* eta, int64_t S, double* xi, cudaStream_t s) {
    if (!factored) throw std::invalid_argument("the handle holds no factor: call factor() and wait() first");
    trmm_build();
    SPH_CUDA(cudaStreamWaitEvent(s, ev1, 0));
    const int64_t ldh = static_cast<int64_t>(nt) * b;
    const bool fp16_hp = cfg.hp_format != SPHEMU_HP_BF16;
    const bool need_bf = !fp16_hp && !tp.ent[1].empty();
    if (tp.h_cols < S) {
      tp.hp.alloc(static_cast<size_t>(S) * ldh);
      for (int f = 0; f < 2; ++f)
        for (int h = 0; h < 2; ++h) tp.h16[f][h].release();
      tp.h_cols = S;
    }
    for (int f = 0; f < (need_bf ? 2 : 1); ++f)
      if (!tp.h16[f][0].get())
        for (int h = 0; h < 2; ++h) tp.h16[f][h].alloc(static_cast<size_t>(tp.h_cols) * ldh);
    // eta -> padded FP64 (the DP operand) + its fp16 (and bf16) hi/lo splits
    trmm_prep_eta(eta, S, n, lb, b, nt, tp.hp.get(), tp.h16[0][0].get(), tp.h16[0][1].get(), 0, s);
    if (need_bf) trmm_prep_eta(eta, S, n, lb, b, nt, tp.hp.get(), tp.h16[1][0].get(), tp.h16[1][1].get(), 1, s);
    SPH_CUDA(cudaMemsetAsync(xi, 0, static_cast<size_t>(S) * n * sizeof(double), s));
    // DP tiles, one band offset per launch (deterministic FP64 order)
    for (size_t q = 0; q < tp.dp_by_offset.size(); ++q)
      if (!tp.dp_by_offset[q].empty())
        trmm_dp_launch(store(), tp.d_dp[q].get(), static_cast<int64_t>(tp.dp_by_offset[q].size()), tp.hp.get(), ldh,
                       S, xi, s);
    static const int flush_env = [] {
      const char* e = std::getenv("SPHEMU_TRMM_FLUSH_K");
      return e ? std::atoi(e) : 8192;
    }();
    // fp32 TMEM partial sums over at most max(b, 8192) of K before the FP64
    // add: the tensor cores' truncating fp32 accumulation error grows with
    // the length (measured max rel. error 1.1e-6 at 512, 4.5e-6 at 2048,
    // 8.9e-6 at 8192) while every flush is an FP64 read-modify-write of the
    // 128 x 256 output block (at K = 512 those dominated the traffic).
    const int flush = std::max(1, flush_env / b);
    for (int c = 0; c < 2; ++c) {
      if (tp.ent[c].empty()) continue;
      if (c == 0)
        trmm_prep_sp(store(), tp.d_sp_tiles.get(), static_cast<int64_t>(tp.sp_tiles.size()), rowexp.get(),
                     tp.sp_hi.get(), tp.sp_lo.get(), s);
      // items: (tile row, 128-row block, 256-snapshot block), longest rows first
      std::vector<std::pair<int, int4>> its;
      const int mblk = (lb + 127) / 128;
      const int nblk = static_cast<int>((S + 255) / 256);
      for (int i = 0; i < nt; ++i) {
        const int cnt = tp.row_ptr[c][i + 1] - tp.row_ptr[c][i];
        if (!cnt) continue;
        for (int mb = 0; mb < mblk; ++mb) {
          if (mb * 128 >= rows(i)) continue;
          for (int nb = 0; nb < nblk; ++nb) its.push_back({cnt, make_int4(i, mb * 128, nb * 256, 0)});
        }
      }
      // snapshot-block-major (the eta block stays in L2), longest rows first within a block
      std::stable_sort(its.begin(), its.end(), [](const auto& x, const auto& y) {
        return x.second.z != y.second.z ? x.second.z < y.second.z : x.first > y.first;
      });
      std::vector<int4> items(its.size());
      for (size_t e = 0; e < its.size(); ++e) items[e] = its[e].second;
      DevBuf<int4> d_items(items.size());
      SPH_CUDA(cudaMemcpyAsync(d_items.get(), items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice, s));
      const int f = (c == 1 && !fp16_hp) ? 1 : 0;
      const CUtensorMap mh = make_map_strided(tp.h16[f][0].get(), S, ldh, 2 * ldh, 2, 256);
      const CUtensorMap ml = make_map_strided(tp.h16[f][1].get(), S, ldh, 2 * ldh, 2, 256);
      TrmmArgs a{tp.d_row_ptr[c].get(), tp.d_ent[c].get(), d_items.get(), static_cast<int64_t>(items.size()), b, lb,
                 n, S, xi, c == 0 ? rowexp.get() : nullptr, flush};
      const int opk = c == 0 ? TR_F16X3 : (fp16_hp ? TR_F16 : TR_BF16);
      trmm_tc_launch(opk, c == 0 ? tp.m_sp_hi : tp.m_arena16, c == 0 ? tp.m_sp_lo : tp.m_arena16, mh, ml, a, s);
      SPH_CUDA(cudaStreamSynchronize(s));  // d_items and the host vectors go out of scope
    }
  }

  void fill_stats(sphemu_chol_stats* st, unsigned saturations) const {
    std::memset(st, 0, sizeof *st);
    st->n = n;
    st->tile_size = b;
    st->n_tiles = nt;
    st->workers = cfg.workers;
    st->variant = cfg.variant;
    const int64_t N = nt;
    st->tasks_potrf = N;
    st->tasks_trsm = N * (N - 1) / 2;
    st->tasks_syrk = N * (N - 1) / 2;
    st->tasks_gemm = N * (N - 1) * (N - 2) / 6;
    for (int i = 0; i < nt; ++i)
      for (int j = 0; j <= i; ++j) {
        const int64_t e = static_cast<int64_t>(rows(i)) * rows(j);
        // writes: the input quantization, then TRSM + GEMM chain (off-diagonal)
        const int64_t writes = 1 + (i == j ? 0 : (1 + j));
        switch (pmap[tix(i, j)]) {
          case SPHEMU_PREC_DP: st->tiles_dp++; st->bytes_dp += 8 * e; break;
          case SPHEMU_PREC_SP: st->tiles_sp++; st->bytes_sp += 4 * e; st->demotions_sp += writes * e; break;
          default: st->tiles_hp++; st->bytes_hp += 2 * e; st->demotions_hp += writes * e; break;
        }
      }
    st->half_saturations = saturations;
    float ms = 0.f;
    if (factored && cudaEventElapsedTime(&ms, ev0, ev1) == cudaSuccess) st->device_ms = ms;
    st->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
    st->launches = launches;
  }

  void store_dense(double* out, int where, int64_t ldo) {
    double* dptr = out;
    int64_t ld = ldo;
    const int threads = 256;
    dim3 grid(std::max(1, std::min(ceil_div(n, threads), 64)), static_cast<unsigned>(std::min(n, 65535)));
    if (dist()) {
      // Gather every tile to rank 0 (collective: all ranks call store_dense).
      DevBuf<char> full;
      DevBuf<int64_t> goff;
      std::vector<int64_t> g(pmap.size());
      int64_t o = 0;
      for (size_t t = 0; t < pmap.size(); ++t) {
        g[t] = o;
        o += static_cast<int64_t>(b) * b * prec_bytes(sprec[t]);
        o = (o + 255) & ~int64_t{255};
      }
      if (rank == 0) {
        full.alloc(static_cast<size_t>(o));
        goff.alloc(pmap.size());
        SPH_CUDA(cudaMemcpy(goff.get(), g.data(), g.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
      }
      size_t t = 0;
      while (t < pmap.size()) {  // groups of up to 512 point-to-point transfers
        SPH_NCCL(ncclGroupStart());
        for (size_t e = 0; e < 512 && t < pmap.size(); ++t, ++e) {
          int x = 0;
          while ((x + 1) * (x + 2) / 2 <= static_cast<int64_t>(t)) ++x;
          const int ti = x, tj = static_cast<int>(t - static_cast<int64_t>(x) * (x + 1) / 2);
          const int o_r = owner(ti, tj);
          const size_t bytes = static_cast<size_t>(b) * b * prec_bytes(sprec[t]);
          if (o_r == 0) {
            if (rank == 0)
              SPH_CUDA(cudaMemcpyAsync(full.get() + g[t], arena.get() + off[t], bytes, cudaMemcpyDeviceToDevice,
                                       stream));
          } else if (rank == o_r) {
            SPH_NCCL(ncclSend(arena.get() + off[t], bytes, ncclUint8, 0, comm, stream));
          } else if (rank == 0) {
            SPH_NCCL(ncclRecv(full.get() + g[t], bytes, ncclUint8, o_r, comm, stream));
          }
        }
        SPH_NCCL(ncclGroupEnd());
      }
      if (rank == 0) {
        TileStore gs{full.get(), goff.get(), d_prec.get(), n, b, nt, lb};
        if (where == SPHEMU_HOST) {  // stream the gathered tiles out by columns (lower triangle only)
          begin_host_out(out, ldo);
          for (int k = 0; k < nt; ++k) col_out(k, stream, &gs);
          end_host_out();
          return;
        }
        k_store_dense<<<grid, threads, 0, stream>>>(gs, dptr, ld);
        SPH_LAUNCH_CHECK();
      }
      SPH_CUDA(cudaStreamSynchronize(stream));
      if (rank != 0) return;
    } else if (where == SPHEMU_HOST) {
      begin_host_out(out, ldo);
      for (int k = 0; k < nt; ++k) col_out(k, stream);
      end_host_out();
      return;
    } else {
      k_store_dense<<<grid, threads, 0, stream>>>(store(), dptr, ld);
      SPH_LAUNCH_CHECK();
    }
    SPH_CUDA(cudaStreamSynchronize(stream));
  }

  double residual(const double* a, int where, int64_t lda) {
    DevBuf<double> da, dl, sums(2);
    const double* ap = a;
    if (where == SPHEMU_HOST) {
      da.alloc(static_cast<size_t>(n) * n);
      SPH_CUDA(cudaMemcpy2D(da.get(), sizeof(double) * n, a, sizeof(double) * lda, sizeof(double) * n,
                            n, cudaMemcpyHostToDevice));
      ap = da.get();
      lda = n;
    }
    dl.alloc(static_cast<size_t>(n) * n);
    store_dense(dl.get(), SPHEMU_DEVICE, n);
    SPH_CUDA(cudaMemsetAsync(sums.get(), 0, 2 * sizeof(double), stream));
    dim3 grid(ceil_div(n, DG_BN), ceil_div(n, DG_BM));
    k_residual<<<grid, DG_THREADS, 0, stream>>>(ap, lda, dl.get(), n, n, sums.get());
    SPH_LAUNCH_CHECK();
    double h[2];
    SPH_CUDA(cudaMemcpyAsync(h, sums.get(), sizeof h, cudaMemcpyDeviceToHost, stream));
    SPH_CUDA(cudaStreamSynchronize(stream));
    return std::sqrt(h[0]) / std::sqrt(h[1]);
  }

  // ||(A - L L^T) x|| / ||A x|| over n_vec seeded vectors, A regenerated
  // from (d, pw) on the fly: a size-independent check at sizes the host
  // cannot hold.
  double residual_probe(uint64_t seed, int n_vec, double rho = 0.9) {
    std::vector<double> d(n), pw(n);
    host_spd_factors(n, seed, d.data(), pw.data(), rho);
    DevBuf<double> dd(n), dpw(n), x(n), y1(n), z(n), y2(n), sums(2);
    SPH_CUDA(cudaMemcpyAsync(dd.get(), d.data(), n * sizeof(double), cudaMemcpyHostToDevice, stream));
    SPH_CUDA(cudaMemcpyAsync(dpw.get(), pw.data(), n * sizeof(double), cudaMemcpyHostToDevice, stream));
    double worst = 0.0;
    for (int v = 0; v < n_vec; ++v) {
      k_probe_vec<<<ceil_div(n, 256), 256, 0, stream>>>(n, 0x9E3779B97F4A7C15ull * (v + 1) + seed, x.get());
      SPH_LAUNCH_CHECK();
      k_spd_matvec<<<ceil_div(n, 4), 128, 0, stream>>>(n, dd.get(), dpw.get(), x.get(), y1.get());
      SPH_LAUNCH_CHECK();
      SPH_CUDA(cudaMemsetAsync(z.get(), 0, n * sizeof(double), stream));
      SPH_CUDA(cudaMemsetAsync(y2.get(), 0, n * sizeof(double), stream));
      k_tile_matvec<<<static_cast<unsigned>(pmap.size()), 256, 0, stream>>>(store(), x.get(), z.get(), 1);
      SPH_LAUNCH_CHECK();
      if (dist()) SPH_NCCL(ncclAllReduce(z.get(), z.get(), n, ncclFloat64, ncclSum, comm, stream));
      k_tile_matvec<<<static_cast<unsigned>(pmap.size()), 256, 0, stream>>>(store(), z.get(), y2.get(), 0);
      SPH_LAUNCH_CHECK();
      if (dist()) SPH_NCCL(ncclAllReduce(y2.get(), y2.get(), n, ncclFloat64, ncclSum, comm, stream));
      SPH_CUDA(cudaMemsetAsync(sums.get(), 0, 2 * sizeof(double), stream));
      k_diff_norms<<<ceil_div(n, 256), 256, 0, stream>>>(n, y1.get(), y2.get(), sums.get());
      SPH_LAUNCH_CHECK();
      double h[2];
      SPH_CUDA(cudaMemcpyAsync(h, sums.get(), sizeof h, cudaMemcpyDeviceToHost, stream));
      SPH_CUDA(cudaStreamSynchronize(stream));
      worst = std::max(worst, std::sqrt(h[0]) / std::sqrt(h[1]));
    }
    return worst;
  }

  // Trailing-update flops by output class (the tcgen05/DMMA update kernels).
  void update_flops(double* f) const {
    f[0] = f[1] = f[2] = 0.0;
    for (int k = 0; k < nt; ++k)
      for (int j = k + 1; j < nt; ++j)
        for (int i = j; i < nt; ++i)
          if (mine(i, j)) f[pmap[tix(i, j)]] += (i == j ? 1.0 : 2.0) * rows(i) * rows(j) * rows(k);
  }

  void flops(double* f) const {
    f[0] = f[1] = f[2] = 0.0;
    auto cls = [&](int i, int j) { return static_cast<int>(pmap[tix(i, j)]); };
    for (int k = 0; k < nt; ++k) {
      const double bk = rows(k);
      f[cls(k, k)] += bk * bk * bk / 3.0;
      for (int i = k + 1; i < nt; ++i) {
        const double bi = rows(i);
        f[cls(i, k)] += bi * bk * bk;
        f[cls(i, i)] += bi * bi * bk;
        for (int j = k + 1; j < i; ++j) f[cls(i, j)] += 2.0 * bi * rows(j) * bk;
      }
    }
  }
};

// make_spd_test_matrix inputs computed on the host exactly as the reference
// does (GaussianRng uniform -> exp, std::pow(0.9, k)), matrix built on device.
void Chol::generate_spd(uint64_t seed, double rho) {
  factored = false;
  // d_i and rho^k (host mt19937_64 + exp / pow, as the reference) are
  // recomputed and uploaded only when (seed, rho) change; the generation
  // itself is stream-ordered with the factorization (no host wait)
  if (spd_d.n != static_cast<size_t>(n) || seed != spd_seed || rho != spd_rho) {
    std::vector<double> d(n), pw(n);
    host_spd_factors(n, seed, d.data(), pw.data(), rho);
    if (spd_d.n != static_cast<size_t>(n)) {
      spd_d.alloc(n);
      spd_pw.alloc(n);
    }
    SPH_CUDA(cudaMemcpyAsync(spd_d.get(), d.data(), n * sizeof(double), cudaMemcpyHostToDevice, stream));
    SPH_CUDA(cudaMemcpyAsync(spd_pw.get(), pw.data(), n * sizeof(double), cudaMemcpyHostToDevice, stream));
    SPH_CUDA(cudaStreamSynchronize(stream));  // the host vectors go out of scope
    spd_seed = seed;
    spd_rho = rho;
  }
  reset_flags();
  k_gen_spd<<<tile_grid(), 256, 0, stream>>>(store(), spd_d.get(), spd_pw.get(), sat.get());
  SPH_LAUNCH_CHECK();
  k_rowexp<<<ceil_div(n, 256), 256, 0, stream>>>(store(), rowexp.get());
  SPH_LAUNCH_CHECK();
  if (dist()) SPH_NCCL(ncclAllReduce(rowexp.get(), rowexp.get(), n, ncclInt32, ncclMax, comm, stream));
}

}  // namespace sphemu_gpu

using namespace sphemu_gpu;

struct sphemu_chol_s {
  Chol* c;
};

// One-shot calls reuse a cached handle (arena, lists, streams, slabs) while
// n, the configuration and the device are unchanged, so repeated
// tiled_cholesky_dense calls pay neither cudaMalloc nor cudaFree;
// sphemu_gpu_release_cache() frees it.
static std::mutex g_dense_mu;
static std::unique_ptr<Chol> g_dense;
static int g_dense_dev = -1;

static bool same_config(const sphemu_chol_config& x, const sphemu_chol_config& y) {
  return x.variant == y.variant && x.tile_size == y.tile_size && x.band_width_dp == y.band_width_dp &&
         x.sp_fraction == y.sp_fraction && x.workers == y.workers && x.hp_format == y.hp_format &&
         x.compute == y.compute && x.lookahead == y.lookahead && x.sp_compute == y.sp_compute;
}

static Chol& dense_handle(int n, const sphemu_chol_config& cfg) {
  int dev = 0;
  SPH_CUDA(cudaGetDevice(&dev));
  if (!g_dense || g_dense->n != n || g_dense_dev != dev || !same_config(g_dense->cfg, cfg)) {
    g_dense.reset();
    g_dense.reset(new Chol(n, cfg));
    g_dense_dev = dev;
  }
  return *g_dense;
}

extern "C" {

const char* sphemu_gpu_last_error(void) { return g_last_error.c_str(); }
const char* sphemu_gpu_version(void) { return "0.1.0"; }
int64_t sphemu_gpu_launch_count(void) { return launch_count(); }

int sphemu_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int sphemu_gpu_set_device(int device) {
  return guard([&] { SPH_CUDA(cudaSetDevice(device)); });
}

int sphemu_gpu_chol_config_validate(const sphemu_chol_config* cfg) {
  return guard([&] { validate_config(*cfg); });
}

int sphemu_gpu_assign_precisions(int n_tiles, const sphemu_chol_config* cfg, uint8_t* out) {
  return guard([&] {
    auto m = assign_precisions(n_tiles, *cfg);
    std::memcpy(out, m.data(), m.size());
  });
}

int sphemu_gpu_chol_create_map(int n, const sphemu_chol_config* cfg, const uint8_t* map, sphemu_chol_t* out) {
  return guard([&] {
    *out = nullptr;
    auto* h = new sphemu_chol_s{nullptr};
    try {
      h->c = new Chol(n, *cfg, 1, 1, 0, nullptr, map);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int sphemu_gpu_tile_norm_precisions(const double* a, int where, int64_t lda, int n, const sphemu_chol_config* cfg,
                                    double tolerance, uint8_t* map) {
  return guard([&] {
    validate_config(*cfg);
    if (n < 1) throw std::invalid_argument("matrix is empty");
    if (!(tolerance > 0.0)) throw std::invalid_argument("norm tolerance must be positive");
    const int b = cfg->tile_size, nt = (n + b - 1) / b;
    const size_t nel = static_cast<size_t>(n) * lda;
    DevBuf<double> da, sq(static_cast<size_t>(nt) * nt);
    const double* A = a;
    if (where == SPHEMU_HOST) {
      da.alloc(nel);
      SPH_CUDA(cudaMemcpy(da.get(), a, nel * sizeof(double), cudaMemcpyHostToDevice));
      A = da.get();
    }
    k_tile_sqnorms<<<dim3(nt, nt), 256>>>(A, lda, n, b, sq.get());
    SPH_LAUNCH_CHECK();
    std::vector<double> h(static_cast<size_t>(nt) * nt);
    SPH_CUDA(cudaMemcpy(h.data(), sq.get(), h.size() * sizeof(double), cudaMemcpyDeviceToHost));
    tile_norm_map(h, nt, *cfg, tolerance, map);
  });
}

int sphemu_gpu_chol_create(int n, const sphemu_chol_config* cfg, sphemu_chol_t* out) {
  return guard([&] {
    *out = nullptr;
    auto* h = new sphemu_chol_s{nullptr};
    try {
      h->c = new Chol(n, *cfg);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int sphemu_gpu_nccl_unique_id(void* out128) {
  return guard([&] {
    ncclUniqueId id;
    SPH_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int sphemu_gpu_chol_create_dist(int n, const sphemu_chol_config* cfg, int P, int Q, int rank, const void* uid128,
                                sphemu_chol_t* out) {
  return guard([&] {
    *out = nullptr;
    if (P < 1 || Q < 1 || rank < 0 || rank >= P * Q) throw std::invalid_argument("bad process grid");
    ncclUniqueId id;
    std::memcpy(&id, uid128, sizeof(id));
    ncclComm_t comm = nullptr;
    SPH_NCCL(ncclCommInitRank(&comm, P * Q, id, rank));
    auto* h = new sphemu_chol_s{nullptr};
    try {
      h->c = new Chol(n, *cfg, P, Q, rank, comm);
    } catch (...) {
      ncclCommDestroy(comm);
      delete h;
      throw;
    }
    *out = h;
  });
}

int sphemu_gpu_chol_destroy(sphemu_chol_t h) {
  return guard([&] {
    if (!h) return;
    delete h->c;
    delete h;
  });
}

int sphemu_gpu_chol_load_dense(sphemu_chol_t h, const double* a, int where, int64_t lda) {
  return guard([&] { h->c->load_dense(a, where, lda); });
}

int sphemu_gpu_chol_generate_spd(sphemu_chol_t h, uint64_t seed) {
  return guard([&] { h->c->generate_spd(seed); });
}

int sphemu_gpu_chol_factor(sphemu_chol_t h) {
  return guard([&] { h->c->factor(); });
}

int sphemu_gpu_chol_wait(sphemu_chol_t h, sphemu_chol_stats* st, int* failed_tile) {
  int rc = SPHEMU_OK;
  int g = guard([&] {
    const int f = h->c->wait(st);
    if (failed_tile) *failed_tile = f;
    if (f >= 0) {
      set_last_error("diagonal tile " + std::to_string(f) + " has a non-positive pivot");
      rc = SPHEMU_ERR_NOT_SPD;
    }
  });
  return g != SPHEMU_OK ? g : rc;
}

int sphemu_gpu_chol_store_dense(sphemu_chol_t h, double* factor, int where, int64_t ldf) {
  return guard([&] { h->c->store_dense(factor, where, ldf); });
}

int sphemu_gpu_chol_residual(sphemu_chol_t h, const double* a, int where, int64_t lda, double* out) {
  return guard([&] { *out = h->c->residual(a, where, lda); });
}

int sphemu_gpu_chol_flops(sphemu_chol_t h, double* f_dp, double* f_sp, double* f_hp) {
  return guard([&] {
    double f[3];
    h->c->flops(f);
    *f_dp = f[0];
    *f_sp = f[1];
    *f_hp = f[2];
  });
}

int sphemu_gpu_chol_generate_spd_decay(sphemu_chol_t h, uint64_t seed, double rho) {
  return guard([&] {
    if (!(rho > 0.0 && rho < 1.0)) throw std::invalid_argument("decay must lie in (0, 1)");
    h->c->generate_spd(seed, rho);
  });
}

int sphemu_gpu_chol_residual_probe_spd_decay(sphemu_chol_t h, uint64_t seed, double rho, int n_vec, double* out) {
  return guard([&] { *out = h->c->residual_probe(seed, n_vec, rho); });
}

int sphemu_gpu_chol_residual_probe_spd(sphemu_chol_t h, uint64_t seed, int n_vec, double* out) {
  return guard([&] { *out = h->c->residual_probe(seed, n_vec); });
}

int sphemu_gpu_chol_set_profiling(sphemu_chol_t h, int on) {
  return guard([&] {
    h->c->profiling = on != 0;
    h->c->prof_mask = (on & 0x100) ? static_cast<unsigned>(on & 0x7f) : 0x7fu;
  });
}

int sphemu_gpu_chol_phase_times(sphemu_chol_t h, double* ms, int64_t* counts, int reset) {
  return guard([&] {
    for (int p = 0; p < Chol::kNumPhases; ++p) {
      if (ms) ms[p] = h->c->phase_ms[p];
      if (counts) counts[p] = h->c->phase_n[p];
      if (reset) {
        h->c->phase_ms[p] = 0.0;
        h->c->phase_n[p] = 0;
      }
    }
  });
}

int sphemu_gpu_chol_timeline(sphemu_chol_t h, int* phase, int* stream, double* t0, double* t1, int cap,
                             int* count) {
  return guard([&] {
    const auto& tl = h->c->timeline;
    const int n = static_cast<int>(tl.size());
    for (int i = 0; i < n && i < cap; ++i) {
      phase[i] = tl[i].phase;
      stream[i] = tl[i].stream;
      t0[i] = tl[i].t0;
      t1[i] = tl[i].t1;
    }
    *count = n;
  });
}

int sphemu_gpu_chol_update_flops(sphemu_chol_t h, double* f_dp, double* f_sp, double* f_hp) {
  return guard([&] {
    double f[3];
    h->c->update_flops(f);
    *f_dp = f[0];
    *f_sp = f[1];
    *f_hp = f[2];
  });
}

void* sphemu_gpu_chol_stream(sphemu_chol_t h) { return h ? h->c->stream : nullptr; }

int sphemu_gpu_release_cache(void) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(g_dense_mu);
    g_dense.reset();
    g_dense_dev = -1;
    scratch_release_all();
  });
}

int sphemu_gpu_dist_layout(int n, const sphemu_chol_config* cfg, int P, int Q, int rank, int64_t* tiles_owned,
                           int64_t* arena_bytes, int64_t* xchg_bytes) {
  return guard([&] {
    validate_config(*cfg);
    if (n < 1 || P < 1 || Q < 1 || rank < 0 || rank >= P * Q) throw std::invalid_argument("bad process grid");
    const int lb = cfg->tile_size;
    const int granule = cfg->compute == SPHEMU_COMPUTE_TENSOR ? 128 : 64;
    const int b = (lb + granule - 1) / granule * granule;
    const int nt = (n + lb - 1) / lb;
    std::vector<uint8_t> pm = assign_precisions(nt, *cfg), sp(pm.size());
    for (size_t t = 0; t < pm.size(); ++t)
      sp[t] = static_cast<uint8_t>(pm[t] == SPHEMU_PREC_DP ? kDP
                                   : (pm[t] == SPHEMU_PREC_SP ? kSP : (cfg->hp_format == SPHEMU_HP_BF16 ? kBF : kHP)));
    BlockCyclic L(nt, b, sp, P, Q, rank);
    int64_t owned = 0;
    for (size_t t = 0; t + 1 < L.off.size(); ++t) owned += L.off[t] >= 0;
    if (tiles_owned) *tiles_owned = owned;
    if (arena_bytes) *arena_bytes = L.off.back();
    if (xchg_bytes) {
      std::fill(xchg_bytes, xchg_bytes + static_cast<size_t>(nt) * P * Q, int64_t{0});
      for (int k = 0; k < static_cast<int>(L.recv_bytes.size()); ++k)
        for (int r = 0; r < P * Q; ++r) xchg_bytes[static_cast<size_t>(k) * P * Q + r] = L.recv_bytes[k][r];
    }
  });
}

}  // extern "C"

namespace sphemu_gpu {
// estimate_innovation_covariance on the device; returns the factored handle
// of u_hat + nugget I (owned by the caller).
std::unique_ptr<Chol> innovation_factor(const double* resid, int where_resid, int64_t n_rows, int d, int r_len,
                                        int t_len, int order, const sphemu_chol_config* cfg, double* u_hat,
                                        int where_u, double* nugget_out, sphemu_chol_stats* stats) {
  if (n_rows < 2 || d < 1) throw std::invalid_argument("residual sample is too small");
  if (n_rows != static_cast<int64_t>(r_len) * (t_len - order))
    throw std::invalid_argument("residual row count does not match r_len*(t_len-order)");
  validate_config(*cfg);
  DevBuf<double> xi_dev, xt, u_dev;
  const double* xi = resid;
  if (where_resid == SPHEMU_HOST) {
    xi_dev.alloc(static_cast<size_t>(n_rows) * d);
    SPH_CUDA(cudaMemcpy(xi_dev.get(), resid, sizeof(double) * n_rows * d, cudaMemcpyHostToDevice));
    xi = xi_dev.get();
  }
  const int64_t ldt = (n_rows + 1) & ~int64_t{1};  // even stride: 16-byte rows for the DMMA loader
  xt.alloc(static_cast<size_t>(d) * ldt);
  k_transpose_pad<<<dim3(static_cast<unsigned>((ldt + 31) / 32), static_cast<unsigned>((d + 31) / 32)), dim3(32, 8)>>>(
      xi, n_rows, d, xt.get(), ldt);
  SPH_LAUNCH_CHECK();
  double* U = (where_u == SPHEMU_DEVICE && u_hat) ? u_hat : nullptr;
  if (!U) {
    u_dev.alloc(static_cast<size_t>(d) * d);
    U = u_dev.get();
  }
  smem_optin(reinterpret_cast<const void*>(k_cov_syrk), (int)sizeof(D2Smem));
  k_cov_syrk<<<dim3(static_cast<unsigned>((d + D2_BN - 1) / D2_BN), static_cast<unsigned>((d + D2_BM - 1) / D2_BM)),
               D2_THREADS, sizeof(D2Smem)>>>(xt.get(), ldt, n_rows, d, 1.0 / static_cast<double>(n_rows), U);
  SPH_LAUNCH_CHECK();
  std::vector<double> diag(d);
  SPH_CUDA(cudaMemcpy2D(diag.data(), sizeof(double), U, sizeof(double) * (d + 1), sizeof(double), d,
                        cudaMemcpyDeviceToHost));
  double sum = 0.0;
  for (double x : diag) sum += x;
  const double mean_diag = sum / d;
  if (!(mean_diag > 0.0)) throw std::runtime_error("innovation covariance has a non-positive mean diagonal");
  xt.release();
  xi_dev.release();
  double nugget = (n_rows < d) ? 1e-8 * mean_diag : 0.0;
  const double cap = 1e-2 * mean_diag;
  std::unique_ptr<Chol> c(new Chol(d, *cfg));
  while (true) {
    c->load_dense(U, SPHEMU_DEVICE, d, nugget);
    c->factor();
    if (c->wait(stats) < 0) break;
    const double next = (nugget == 0.0) ? 1e-8 * mean_diag : 10.0 * nugget;
    if (next > cap)
      throw std::runtime_error(
          "innovation covariance is not positive definite even with the largest allowed diagonal inflation");
    nugget = next;
  }
  if (nugget_out) *nugget_out = nugget;
  if (u_hat && where_u == SPHEMU_HOST)
    SPH_CUDA(cudaMemcpy(u_hat, U, sizeof(double) * d * d, cudaMemcpyDeviceToHost));
  return c;
}
}  // namespace sphemu_gpu

extern "C" {

// estimate_innovation_covariance (stochastic.cpp:109-172) with the sample
// covariance and every nugget retry on the device: U = Xi^T Xi / n by DMMA
// (cov_kernels.cuh), then tiled factorizations of U + nugget I read straight
// from U in HBM, the nugget escalated tenfold from 0 (or 1e-8 mean diag when
// n < d) until the factor succeeds, giving up past 1e-2 mean diag.
int sphemu_gpu_estimate_innovation_covariance(const double* resid, int where_resid, int64_t n_rows, int d,
                                              int r_len, int t_len, int order, const sphemu_chol_config* cfg,
                                              double* u_hat, int where_u, double* v, int where_v,
                                              double* nugget_out, sphemu_chol_stats* stats) {
  return guard([&] {
    auto c = innovation_factor(resid, where_resid, n_rows, d, r_len, t_len, order, cfg, u_hat, where_u, nugget_out,
                               stats);
    if (v) c->store_dense(v, where_v, d);
  });
}

int sphemu_gpu_innovation_factor(const double* resid, int where_resid, int64_t n_rows, int d, int r_len,
                                 int t_len, int order, const sphemu_chol_config* cfg, double* u_hat, int where_u,
                                 double* nugget_out, sphemu_chol_stats* stats, sphemu_chol_t* out) {
  return guard([&] {
    *out = nullptr;
    auto c = innovation_factor(resid, where_resid, n_rows, d, r_len, t_len, order, cfg, u_hat, where_u, nugget_out,
                               stats);
    *out = new sphemu_chol_s{c.release()};
  });
}

int sphemu_gpu_chol_load_factor(sphemu_chol_t h, const double* l, int where, int64_t ldl) {
  return guard([&] {
    Chol& c = *h->c;
    c.load_dense(l, where, ldl);
    c.mark_factored();
  });
}

int sphemu_gpu_chol_trmm(sphemu_chol_t h, const double* eta, int where_in, int64_t S, double* xi, int where_out) {
  return guard([&] {
    if (!h) throw std::invalid_argument("null handle");
    if (S < 1) throw std::invalid_argument("need at least one column");
    Chol& c = *h->c;
    const size_t el = static_cast<size_t>(S) * c.n;
    DevBuf<double> de, dx;
    const double* e = eta;
    if (where_in == SPHEMU_HOST) {
      de.alloc(el);
      SPH_CUDA(cudaMemcpyAsync(de.get(), eta, el * sizeof(double), cudaMemcpyHostToDevice, c.stream));
      e = de.get();
    }
    double* x = xi;
    if (where_out == SPHEMU_HOST) {
      dx.alloc(el);
      x = dx.get();
    }
    c.trmm(e, S, x, c.stream);
    if (c.dist()) SPH_NCCL(ncclAllReduce(x, x, el, ncclFloat64, ncclSum, c.comm, c.stream));
    if (where_out == SPHEMU_HOST)
      SPH_CUDA(cudaMemcpyAsync(xi, x, el * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    SPH_CUDA(cudaStreamSynchronize(c.stream));
  });
}

static void emulate_chol_impl(sphemu_chol_t h, sphemu_sht_t plan, const double* phi, int order,
                              const double* means, const double* sigma, const double* v2, int t_out, uint64_t seed,
                              int r_begin, int r_count, int rng_mode, double* out, int where_out,
                              const TrendArgs* trend);

int sphemu_gpu_emulate_chol(sphemu_chol_t h, sphemu_sht_t plan, const double* phi, int order, const double* means,
                            const double* sigma, const double* v2, int t_out, uint64_t seed, int r_begin,
                            int r_count, int rng_mode, double* out, int where_out) {
  return guard([&] {
    emulate_chol_impl(h, plan, phi, order, means, sigma, v2, t_out, seed, r_begin, r_count, rng_mode, out, where_out,
                      nullptr);
  });
}

int sphemu_gpu_emulate_chol_trend(sphemu_chol_t h, sphemu_sht_t plan, const double* phi, int order,
                                  const double* records, int harmonics, int period, const double* forcing_x,
                                  int64_t n_x, const double* forcing_history, int64_t n_history, int64_t t_start,
                                  const double* v2, int t_out, uint64_t seed, int r_begin, int r_count,
                                  int rng_mode, double* out, int where_out) {
  return guard([&] {
    const TrendArgs ta{records, harmonics, period, forcing_x, n_x, forcing_history, n_history, t_start};
    emulate_chol_impl(h, plan, phi, order, nullptr, nullptr, v2, t_out, seed, r_begin, r_count, rng_mode, out,
                      where_out, &ta);
  });
}

static void emulate_chol_impl(sphemu_chol_t h, sphemu_sht_t plan, const double* phi, int order,
                              const double* means, const double* sigma, const double* v2, int t_out, uint64_t seed,
                              int r_begin, int r_count, int rng_mode, double* out, int where_out,
                              const TrendArgs* trend) {
  {
    if (!h || !plan) throw std::invalid_argument("null handle");
    Chol& c = *h->c;
    EmulArgs a{};
    a.plan = plan;
    sht_plan_dims(plan, &a.n_theta, &a.n_phi, &a.L);
    a.d = c.n;
    a.phi = phi;
    a.order = order;
    a.means = means;
    a.sigma = sigma;
    a.v2 = v2;
    a.t_out = t_out;
    a.seed = seed;
    a.r_begin = r_begin;
    a.r_len = r_count;
    a.rng_mode = rng_mode;
    a.out = out;
    a.where_out = where_out;
    a.trend = trend;
    a.world = c.P * c.Q;
    a.rank = c.rank;
    static const int64_t budget = [] {
      const char* e = std::getenv("SPHEMU_EMUL_CHUNK_MB");
      return e ? (int64_t)std::atoll(e) << 20 : int64_t{0};
    }();
    a.chunk_bytes = budget;
    DevBuf<double> part;
    emulate_core(a, [&](const double* dH, int64_t S_all, const std::vector<int64_t>& col_off, double* dXi,
                        cudaStream_t s) {
      if (!c.dist()) {
        c.trmm(dH, S_all, dXi, s);
        return;
      }
      // partial product over this rank's tiles for every rank's columns, then
      // each rank's column block summed onto it (reduce-scatter by replicates)
      const size_t el = static_cast<size_t>(S_all) * c.n;
      if (part.n < el) part.alloc(el);
      c.trmm(dH, S_all, part.get(), s);
      SPH_NCCL(ncclGroupStart());
      for (int q = 0; q < c.P * c.Q; ++q) {
        const size_t cnt = static_cast<size_t>(col_off[q + 1] - col_off[q]) * c.n;
        if (!cnt) continue;
        SPH_NCCL(ncclReduce(part.get() + col_off[q] * c.n, dXi, cnt, ncclFloat64, ncclSum, q, c.comm, s));
      }
      SPH_NCCL(ncclGroupEnd());
      note_launch();
    });
  }
}

int sphemu_gpu_tiled_cholesky_dense(const double* a, int where_a, int n, const sphemu_chol_config* cfg,
                                    double* factor, int where_factor, sphemu_chol_stats* stats,
                                    int* failed_tile) {
  int rc = SPHEMU_OK;
  int g = guard([&] {
    std::lock_guard<std::mutex> lk(g_dense_mu);
    Chol& c = dense_handle(n, *cfg);
    // The host zero-fill of the output's upper triangle starts first, so it
    // overlaps the input's H2D instead of competing with the factor's D2H.
    const bool stream_out = where_factor == SPHEMU_HOST;
    if (stream_out) c.begin_host_out(factor, n);
    struct Finish {  // joins the host zero-fill threads on every exit path
      Chol& c;
      ~Finish() {
        try {
          c.end_host_out();
        } catch (...) {
        }
      }
    } finish{c};
    c.load_dense(a, where_a, n);
    c.factor();
    const int f = c.wait(stats);
    if (failed_tile) *failed_tile = f;
    if (f >= 0) {
      set_last_error("diagonal tile " + std::to_string(f) + " has a non-positive pivot");
      rc = SPHEMU_ERR_NOT_SPD;
      return;
    }
    if (stream_out) c.end_host_out();
    else c.store_dense(factor, where_factor, n);
  });
  return g != SPHEMU_OK ? g : rc;
}

}  // extern "C"
