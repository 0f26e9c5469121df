// potrf_coop.cuh — factor + invert one diagonal tile with a cooperative grid
// of CTAs (mpchol.cpp:230-252 potrf_tile, plus the inverse that turns the
// panel TRSM into a GEMM). The tile is split into 64 x 64 blocks; every
// block-level operation is a 64x64x64 FP64 DMMA GEMM (dgemm_64x64) spread over
// the grid, with grid-wide barriers between the dependent phases:
//   for s:  [CTA 0] factor + invert block (s,s) in shared memory
//           [all]   TRSM  X_rs = A_rs D_s^{-T}            (r > s)
//           [all]   SYRK/GEMM  A_rc -= X_rs X_cs^T        (s < c <= r)
//   TRTRI right-looking by block rows: X_s = D_s^{-1} R_s, R_r -= L_rs X_s.
// Pivot failures (not > 0, or NaN) set *fail = k like NotPositiveDefiniteError.
#pragma once

#include <cooperative_groups.h>

#include "chol_kernels.cuh"
#include "dgemm2.cuh"

namespace sphemu_gpu {

constexpr int PC_BLK = 64;
// Row stride of the 64 x 64 operand blocks staged for the DMMA products: 68
// doubles keeps the m8n8k4 fragment loads conflict-free per half-warp.
constexpr int PG_LD = 68;

struct PcSmallSmem {
  double T[64][65];
  double Di[64][65];
  double M[32][33];
  double X[64][PG_LD];  // CTA 0: its phase-A TRSM result X_{s+1,s}, the lookahead SYRK's operand
  double col[17];  // base-case column broadcast
  int bad;
};

// 16 x 16 base case (warp 0; lanes 0..15 own the rows, 16..31 mirror them):
// right-looking Cholesky with one rsqrt per column. The column values move by
// shuffles, and the next pivot goes first: lane c+1 forms its updated
// diagonal from its own l_{c+1,c} and broadcasts it before the other rows'
// updates, so a column's critical path is rsqrt -> fma -> shuffle (the
// earlier shared-memory broadcast put a store, a warp barrier and a load in
// every step). Same arithmetic as the row updates: bitwise the same factor.
// Then the inverse by forward substitution (lane j owns column j, reading L
// from s.T). Small unrolled code: the cooperative kernel is sensitive to
// instruction-cache pressure.
__device__ __noinline__ void pc_base16(PcSmallSmem& s, int o, int w, int lane) {
  const int row = lane & 15;
  double a[16], rl[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) a[t] = s.T[o + row][o + t];
  bool ok = true;
  double piv = __shfl_sync(0xffffffffu, a[0], 0);
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    if (c < w && !(piv > 0.0)) ok = false;
    rl[c] = rsqrt(piv);
    const double lrc = (row == c) ? piv * rl[c] : a[c] * rl[c];
    a[c] = lrc;
    if (c + 1 < 16) piv = __shfl_sync(0xffffffffu, fma(-lrc, lrc, a[c + 1]), c + 1);
#pragma unroll
    for (int j = c + 1; j < 16; ++j) a[j] = fma(-lrc, __shfl_sync(0xffffffffu, lrc, j), a[j]);
  }
  if (!ok) {
    if (lane == 0) s.bad = 1;
    return;
  }
  if (lane < 16)
#pragma unroll
    for (int t = 0; t < 16; ++t) s.T[o + lane][o + t] = t <= lane ? a[t] : 0.0;
  __syncwarp();
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = (i == row) ? 1.0 : 0.0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    x[r] *= rl[r];
#pragma unroll
    for (int i = r + 1; i < 16; ++i) x[i] -= s.T[o + i][o + r] * x[r];
  }
  if (lane < 16)
#pragma unroll
    for (int r = 0; r < 16; ++r) s.Di[o + r][o + lane] = x[r];
}

// 32 x 32 base case on one warp (lane = row): the same right-looking,
// next-pivot-first shuffle scheme as pc_base16 over 32 columns, then the
// inverse by forward substitution (lane j owns column j, L read back from
// s.T with broadcast loads). Replaces the 16-wide recursion level (two 16 x 16
// bases + four 16-wide products, each behind a CTA barrier): one warp, no
// barriers, 32 rsqrt-bound column steps.
__device__ __noinline__ void pc_base32(PcSmallSmem& s, int o, int w, int lane) {
  double a[32], rl[32];
#pragma unroll
  for (int t = 0; t < 32; ++t) a[t] = s.T[o + lane][o + t];
  bool ok = true;
  double piv = __shfl_sync(0xffffffffu, a[0], 0);
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    if (c < w && !(piv > 0.0)) ok = false;
    rl[c] = rsqrt(piv);
    const double lrc = (lane == c) ? piv * rl[c] : a[c] * rl[c];
    a[c] = lrc;
    if (c + 1 < 32) piv = __shfl_sync(0xffffffffu, fma(-lrc, lrc, a[c + 1]), c + 1);
#pragma unroll
    for (int j = c + 1; j < 32; ++j) a[j] = fma(-lrc, __shfl_sync(0xffffffffu, lrc, j), a[j]);
  }
  if (!ok) {
    if (lane == 0) s.bad = 1;
    return;
  }
#pragma unroll
  for (int t = 0; t < 32; ++t) s.T[o + lane][o + t] = t <= lane ? a[t] : 0.0;
  __syncwarp();
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    x[r] *= rl[r];
#pragma unroll
    for (int i = r + 1; i < 32; ++i) x[i] -= s.T[o + i][o + r] * x[r];
  }
#pragma unroll
  for (int r = 0; r < 32; ++r) s.Di[o + r][o + lane] = x[r];
}

// out(r, c, sum_t a(r, t) b(t, c)) for an N x N product on the whole CTA
// (128 threads); each thread keeps one row of a in registers. All reads
// finish (barrier) before any write, so in-place updates are safe.
template <int N, class FA, class FB, class FO>
__device__ __forceinline__ void pc_mm(FA fa, FB fb, FO fo) {
  constexpr int OUT = N * N / 128, PER_ROW = N / OUT;
  const int r = threadIdx.x / PER_ROW, cb = (threadIdx.x % PER_ROW) * OUT;
  double row[N], acc[OUT];
#pragma unroll
  for (int t = 0; t < N; ++t) row[t] = fa(r, t);
#pragma unroll
  for (int u = 0; u < OUT; ++u) {
    double v = 0.0;
#pragma unroll
    for (int t = 0; t < N; ++t) v += row[t] * fb(t, cb + u);
    acc[u] = v;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < OUT; ++u) fo(r, cb + u, acc[u]);
  __syncthreads();
}

// The same product on the FP64 tensor pipe: m8n8k4 DMMA tiles, the four
// warps splitting the (N/8)^2 output tiles.
template <int N, class FA, class FB, class FO>
__device__ __forceinline__ void pc_mm_t(FA fa, FB fb, FO fo) {
  constexpr int TPW = (N / 8) * (N / 8) / 4;
  static_assert(TPW >= 1, "N >= 16");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int lr = lane >> 2, lk = lane & 3;
  double acc[TPW][2];
#pragma unroll
  for (int u = 0; u < TPW; ++u) acc[u][0] = acc[u][1] = 0.0;
#pragma unroll
  for (int k = 0; k < N; k += 4) {
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
      const int tile = warp * TPW + u;
      const int tr = (tile / (N / 8)) * 8, tc = (tile % (N / 8)) * 8;
      dmma_8x8x4(acc[u][0], acc[u][1], fa(tr + lr, k + lk), fb(k + lk, tc + lr));
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    const int tile = warp * TPW + u;
    const int tr = (tile / (N / 8)) * 8, tc = (tile % (N / 8)) * 8;
    fo(tr + lr, tc + 2 * lk, acc[u][0]);
    fo(tr + lr, tc + 2 * lk + 1, acc[u][1]);
  }
  __syncthreads();
}

// Cholesky + inverse of the H x H block at (o, o) of s.T into s.T / s.Di by
// 2 x 2 recursion: L11, inv11 | L21 = A21 inv11^T | A22 -= L21 L21^T |
// L22, inv22 | inv21 = -inv22 (L21 inv11).
// Not inlined: the two calls per level share one copy of the code (the
// cooperative kernel is large enough for instruction fetch to matter).
#ifndef PC_BASE32
#define PC_BASE32 0  // measured slower: chol_inv<32> 5.65 vs 5.0 us (the per-column shuffle chain is ~250 cycles either way)
#endif
template <int H>
__device__ __noinline__ void pc_chol_inv(PcSmallSmem& s, int o, int w) {
  if constexpr (H == 16) {
    if ((threadIdx.x >> 5) == 0) pc_base16(s, o, w, threadIdx.x & 31);
    __syncthreads();
  } else if constexpr (H == 32 && PC_BASE32) {
    if ((threadIdx.x >> 5) == 0) pc_base32(s, o, w, threadIdx.x & 31);
    __syncthreads();
  } else {
    constexpr int N = H / 2;
    pc_chol_inv<N>(s, o, min(w, N));
    if (s.bad) return;
    pc_mm_t<N>([&](int r, int t) { return s.T[o + N + r][o + t]; },
               [&](int t, int c) { return s.Di[o + c][o + t]; },
               [&](int r, int c, double v) { s.T[o + N + r][o + c] = v; });
    pc_mm_t<N>([&](int r, int t) { return s.T[o + N + r][o + t]; },
               [&](int t, int c) { return s.T[o + N + c][o + t]; },
               [&](int r, int c, double v) {
                 if (c <= r) s.T[o + N + r][o + N + c] -= v;
               });
    pc_chol_inv<N>(s, o + N, max(0, w - N));
    if (s.bad) return;
    // M = L21 inv11 (after the recursion above: s.M is shared scratch).
    pc_mm_t<N>([&](int r, int t) { return s.T[o + N + r][o + t]; },
               [&](int t, int c) { return s.Di[o + t][o + c]; },
               [&](int r, int c, double v) { s.M[r][c] = v; });
    pc_mm_t<N>([&](int r, int t) { return s.Di[o + N + r][o + N + t]; },
               [&](int t, int c) { return s.M[t][c]; },
               [&](int r, int c, double v) {
                 s.Di[o + N + r][o + c] = -v;
                 s.Di[o + r][o + N + c] = 0.0;
               });
  }
}

#ifdef SPHEMU_POTRF_TRACE
__device__ unsigned long long* g_potrf_trace;
#define PTRACE(slot)                                                                         \
  do {                                                                                       \
    if (threadIdx.x == 0 && g_potrf_trace) {                                                 \
      unsigned long long t__;                                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t__));                                \
      g_potrf_trace[blockIdx.x * 64 + (slot)] = t__;                                         \
    }                                                                                        \
  } while (0)
#else
#define PTRACE(slot) \
  do {               \
  } while (0)
#endif

// 64 x 64 x K (K <= 64) FP64 product with both operands staged whole in
// shared memory by cp.async (every load in flight at once: one memory round
// trip instead of one per K-chunk), then 16 DMMA k-steps. Same accumulator
// layout as dgemm_64x64 (dg_for_each).
struct PgSmem {
  double a[64 * PG_LD];
  double b[64 * PG_LD];
  double c[64 * PG_LD];  // read-modify-write target of pgemm_64_rmw
};

template <class Acc>
__device__ __forceinline__ void pg_stage(const Acc& X, int K, double* s) {
  // KContig: element (r, k) at base[r*ld + k] -> s[r][k]; else (c, k) at base[k*ld + c] -> s[k][c]
  for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
    const int row = e >> 5, col = (e & 31) * 2;  // row: r (KContig) or k; col: k (KContig) or c
    const int r_lim = Acc::kKContig ? X.rows : K, c_lim = Acc::kKContig ? K : X.rows;
    int bytes = 0;
    const double* src = X.base;
    if (row < r_lim && col < c_lim) {
      bytes = (c_lim - col >= 2) ? 16 : 8;
      src = X.base + (int64_t)row * X.ld + col;
    }
    cp_async16(s + row * PG_LD + col, src, bytes);
  }
}

// acc = X X^T for a 64 x K block X already in shared memory (row stride
// PG_LD, zero beyond K): the lookahead SYRK without a memory round trip.
__device__ __forceinline__ void pg_syrk_smem(const double* X, int K, double (&acc)[4][4][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  const int kq = lane & 3, rq = lane >> 2;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  for (int kk = 0; kk < K; kk += 4) {
    double a[4], b[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = X[(wm * 32 + mi * 8 + rq) * PG_LD + kk + kq];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = X[(wn * 32 + ni * 8 + rq) * PG_LD + kk + kq];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
  }
}

template <class AccA, class AccB>
__device__ __forceinline__ void pgemm_64(const AccA& A, const AccB& B, int K, PgSmem& sm, double (&acc)[4][4][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  pg_stage(A, K, sm.a);
  pg_stage(B, K, sm.b);
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int kq = lane & 3, rq = lane >> 2;
  for (int kk = 0; kk < K; kk += 4) {
    double a[4], b[4];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = sm.a[(wm * 32 + mi * 8 + rq) * PG_LD + kk + kq];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int cn = wn * 32 + ni * 8 + rq;
      b[ni] = AccB::kKContig ? sm.b[cn * PG_LD + kk + kq] : sm.b[(kk + kq) * PG_LD + cn];
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
  }
  __syncthreads();  // smem reusable by the caller
}

// out -= A B^T on the elements keep(i, j) selects: the 64 x 64 output block is
// staged by cp.async together with the operands, updated in shared memory and
// written back with coalesced 16-byte stores (the whole block: elements the
// mask skips are written back unchanged; every block has one owner per phase).
template <class AccA, class AccB, class Keep>
__device__ __forceinline__ void pgemm_64_rmw(const AccA& A, const AccB& B, int K, double* out, int64_t ld,
                                             PgSmem& sm, Keep keep) {
  for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
    const int row = e >> 5, col = (e & 31) * 2;
    cp_async16(sm.c + row * PG_LD + col, out + (int64_t)row * ld + col, 16);
  }
  double acc[4][4][2];
  pgemm_64(A, B, K, sm, acc);  // its cp.async wait covers the staging above
  dg_for_each(acc, [&](int i, int j, double v) {
    if (keep(i, j)) sm.c[i * PG_LD + j] -= v;
  });
  __syncthreads();
  for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
    const int row = e >> 5, col = (e & 31) * 2;
    *reinterpret_cast<double2*>(out + (int64_t)row * ld + col) =
        *reinterpret_cast<const double2*>(sm.c + row * PG_LD + col);
  }
  __syncthreads();
}

// Factor + invert the 64 x 64 block already staged in s.T (lower part, zero
// upper part, unit diagonal on padding rows) and write back the factor and
// the inverse. Returns false on a bad pivot (not > 0, or NaN) among the
// first w columns.
__device__ bool pc_small_finish(double* A, int b, int j0, int w, double* dinv_out, PcSmallSmem& s) {
  const int tid = threadIdx.x;
  if (tid == 0) s.bad = 0;
  __syncthreads();
  if (j0 == 64) PTRACE(40);
  pc_chol_inv<64>(s, 0, w);
  __syncthreads();
  if (j0 == 64) PTRACE(41);
  if (s.bad) return false;
#pragma unroll 4
  for (int e = tid; e < 64 * 32; e += blockDim.x) {
    const int rr = e >> 5, c = (e & 31) * 2;
    if (rr < w) {
      double* dst = A + (int64_t)(j0 + rr) * b + j0 + c;
      if (c + 1 <= rr) *reinterpret_cast<double2*>(dst) = make_double2(s.T[rr][c], s.T[rr][c + 1]);
      else if (c <= rr) dst[0] = s.T[rr][c];
    }
    *reinterpret_cast<double2*>(dinv_out + rr * 64 + c) = make_double2(s.Di[rr][c], s.Di[rr][c + 1]);
  }
  return true;
}

// Factor + invert the 64 x 64 diagonal block at (j0, j0) (w valid rows).
__device__ bool pc_small(double* A, int b, int j0, int w, double* dinv_out, PcSmallSmem& s) {
  const int tid = threadIdx.x;
#pragma unroll 4
  for (int e = tid; e < 64 * 32; e += blockDim.x) {  // double2 granules, all loads in flight together
    const int r = e >> 5, c = (e & 31) * 2;
    double2 v = make_double2(0.0, 0.0);
    if (r < w) v = __ldcg(reinterpret_cast<const double2*>(A + (int64_t)(j0 + r) * b + j0 + c));
    s.T[r][c] = (r < w && c <= r) ? v.x : (r == c ? 1.0 : 0.0);
    s.T[r][c + 1] = (r < w && c + 1 <= r) ? v.y : (r == c + 1 ? 1.0 : 0.0);
  }
  return pc_small_finish(A, b, j0, w, dinv_out, s);
}

__device__ __forceinline__ double* blk(double* A, int b, int r, int c) {
  return A + (int64_t)r * PC_BLK * b + (int64_t)c * PC_BLK;
}

// Pipelined schedule, two grid barriers per 64-row block step s:
//   phase A: TRSM X_rs = A_rs D_s^{-T} (r > s)   |  TRTRI  X_sc = D_s^{-1} R_sc (c <= s)
//   phase B: CTA 0 updates block (s+1, s+1) and factors/inverts it (lookahead)
//            | the rest: A_rc -= X_rs X_cs^T (s < c <= r, not (s+1,s+1))
//            | TRTRI R_rc -= L_rs X_sc (r > s, c <= s)
//
// Barrier A is split: CTA 0 arrives after its phase-A items and goes straight
// on to the lookahead (it reads nothing the other CTAs write in phase A), so
// its factor + invert of block (s+1, s+1), the chain's long pole, starts one
// barrier earlier; the other CTAs wait for every arrival before their
// trailing updates. *bar counts arrivals (G per step); CTA 0 zeroes it after
// the last grid.sync, when every CTA is past its last wait.
__global__ void __launch_bounds__(DG_THREADS) k_potrf_coop(double* __restrict__ A, int b, int bk,
                                                           double* __restrict__ Linv,
                                                           double* __restrict__ dinv_all, int* fail, int k,
                                                           unsigned* __restrict__ bar) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) uint8_t pc_smem[];
  PgSmem& sm = *reinterpret_cast<PgSmem*>(pc_smem);
  PcSmallSmem& ss = *reinterpret_cast<PcSmallSmem*>(pc_smem + sizeof(PgSmem));  // disjoint: staged during the SYRK
  // An earlier step's failure (written by an earlier kernel) is uniform across
  // the grid; this kernel's own CTA 0 may set fail = k in the prologue while a
  // late CTA reads it, so that value must not send a CTA home before the
  // first grid barrier (the others would wait there forever).
  {
    const int f = *(volatile int*)fail;
    if (f >= 0 && f != k) return;
  }
  const int nblk = (bk + PC_BLK - 1) / PC_BLK;
  const int G = gridDim.x, cta = blockIdx.x;
  auto rows_of = [&](int r) { return min(PC_BLK, bk - r * PC_BLK); };
  double acc[4][4][2];
  // Prologue: Linv <- I (all CTAs) while CTA 0 factors block 0.
  for (int64_t e = (int64_t)cta * blockDim.x + threadIdx.x; e < (int64_t)b * b; e += (int64_t)G * blockDim.x) {
    const int r = (int)(e / b), c = (int)(e % b);
    Linv[e] = (r == c && r < bk) ? 1.0 : 0.0;
  }
  PTRACE(0);
  if (cta == 0 && !pc_small(A, b, 0, rows_of(0), dinv_all, ss) && threadIdx.x == 0) atomicCAS(fail, -1, k);
  PTRACE(1);
  __threadfence();
  grid.sync();
  PTRACE(2);
  auto reset_bar = [&] {
    if (cta == 0 && threadIdx.x == 0) *bar = 0u;
  };
  for (int s = 0; s < nblk; ++s) {
    if (*(volatile int*)fail >= 0) {
      reset_bar();
      return;
    }
    const int w = rows_of(s);
    const double* dinv = dinv_all + (int64_t)s * PC_BLK * PC_BLK;
    // ---- phase A ----
    const int n_trsm = nblk - s - 1;
    if (cta == 0 && n_trsm > 0) {
      // CTA 0's lookahead operand A_{s+1,s+1} (lower part) streams into
      // shared memory under this phase's products (waited for in phase B).
      const int r = s + 1, rr = rows_of(r), j0 = r * PC_BLK;
      for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
        const int ri = e >> 6, ci = e & 63;
        const bool in = ri < rr && ci <= ri;
        cp_async8(&ss.T[ri][ci], in ? A + (int64_t)(j0 + ri) * b + j0 + ci : A, in ? 8 : 0);
      }
      cp_async_commit();
    }
    for (int item = cta; item < n_trsm + s + 1; item += G) {
      if (item < n_trsm) {  // TRSM, in place (one CTA owns each block)
        const int r = s + 1 + item;
        RowMajorK a{blk(A, b, r, s), b, rows_of(r), w};
        RowMajorK d{dinv, PC_BLK, PC_BLK, w};
        pgemm_64(a, d, w, sm, acc);
        double* out = blk(A, b, r, s);
        const int rr = rows_of(r);
        dg_for_each(acc, [&](int i, int j, double v) {
          if (i < rr && j < w) out[(int64_t)i * b + j] = v;
        });
        if (item == 0)  // CTA 0: X_{s+1,s} stays in shared memory for the lookahead SYRK
          dg_for_each(acc, [&](int i, int j, double v) { ss.X[i][j] = (i < rr && j < w) ? v : 0.0; });
      } else {  // TRTRI X_sc = Dinv_s R_sc, in place
        const int c = item - n_trsm;
        RowMajorK d{dinv, PC_BLK, w, w};
        KMajor rsc{blk(Linv, b, s, c), b, rows_of(c), w};
        pgemm_64(d, rsc, w, sm, acc);
        double* out = blk(Linv, b, s, c);
        const int cc = rows_of(c);
        dg_for_each(acc, [&](int i, int j, double v) {
          if (i < w && j < cc) out[(int64_t)i * b + j] = v;
        });
      }
      __syncthreads();
    }
    PTRACE(3 + 4 * s);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(bar, 1u);
      if (G == 1 || cta > 0) {
        const unsigned target = static_cast<unsigned>(G) * static_cast<unsigned>(s + 1);
        while (*(volatile unsigned*)bar < target) {
        }
        __threadfence();
      }
    }
    __syncthreads();
    PTRACE(4 + 4 * s);
    // ---- phase B ----
    if (cta == 0) {
      if (s + 1 < nblk) {
        // Lookahead block: A_rr -= X_rs X_rs^T with both operands already in
        // shared memory (X from this CTA's phase-A TRSM, A_rr prefetched at
        // the start of phase A), then factor+invert.
        const int r = s + 1, rr = rows_of(r), j0 = r * PC_BLK;
        cp_async_wait<0>();
        __syncthreads();
        pg_syrk_smem(&ss.X[0][0], w, acc);
        dg_for_each(acc, [&](int i, int j, double v) {
          if (i < rr && j <= i) ss.T[i][j] -= v;
        });
        if (threadIdx.x >= rr && threadIdx.x < 64) ss.T[threadIdx.x][threadIdx.x] = 1.0;
        __syncthreads();
        if (!pc_small_finish(A, b, j0, rr, dinv_all + (int64_t)r * PC_BLK * PC_BLK, ss) && threadIdx.x == 0)
          atomicCAS(fail, -1, k);
      }
    }
    const int m = nblk - s - 1;
    const int pairs = m * (m + 1) / 2;       // trailing blocks, index 0 is (s+1, s+1)
    const int tri = m * (s + 1);             // TRTRI-b blocks
    const int workers = G > 1 ? G - 1 : 1;
    const int me = G > 1 ? cta - 1 : 0;
    if (G == 1 || cta > 0) {
      for (int item = me; item < (pairs - 1) + tri; item += workers) {
        if (item < pairs - 1) {
          int ri, ci;
          pair_from_index(item + 1, ri, ci);
          const int r = s + 1 + ri, c = s + 1 + ci;
          RowMajorK x1{blk(A, b, r, s), b, rows_of(r), w};
          RowMajorK x2{blk(A, b, c, s), b, rows_of(c), w};
          const int rr = rows_of(r), cc = rows_of(c);
          pgemm_64_rmw(x1, x2, w, blk(A, b, r, c), b, sm,
                       [&](int i, int j) { return i < rr && j < cc && (r != c || j <= i); });
        } else {
          const int q = item - (pairs - 1);
          const int r = s + 1 + q / (s + 1), c = q % (s + 1);
          RowMajorK l{blk(A, b, r, s), b, rows_of(r), w};
          KMajor x{blk(Linv, b, s, c), b, rows_of(c), w};
          const int rr = rows_of(r), cc = rows_of(c);
          pgemm_64_rmw(l, x, w, blk(Linv, b, r, c), b, sm, [&](int i, int j) { return i < rr && j < cc; });
        }
        __syncthreads();
      }
    }
    PTRACE(5 + 4 * s);
    __threadfence();
    grid.sync();
    PTRACE(6 + 4 * s);
  }
  reset_bar();
  // Strict upper part to zero (potrf_tile's final loop).
  for (int64_t e = (int64_t)cta * blockDim.x + threadIdx.x; e < (int64_t)b * b; e += (int64_t)G * blockDim.x) {
    const int r = (int)(e / b), c = (int)(e % b);
    if (c > r) A[e] = 0.0;
  }
}

inline size_t potrf_coop_smem() { return sizeof(PgSmem) + sizeof(PcSmallSmem); }

}  // namespace sphemu_gpu
