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

namespace sphemu_gpu {

constexpr int PC_BLK = 64;

struct PcSmallSmem {
  double T[64][65];
  double Di[64][65];
  double M[32][33];
  int bad;
};

// Warp-level Cholesky-Crout of T[o:o+32, o:o+32] (lane = row) and inverse
// into Di[o:o+32, o:o+32] (lane = column). Returns false on a bad pivot.
__device__ bool pc_factor32(PcSmallSmem& s, int o, int w, int lane) {
  for (int c = 0; c < 32; ++c) {
    double v = s.T[o + lane][o + c];
    for (int t = 0; t < c; ++t) v -= s.T[o + lane][o + t] * s.T[o + c][o + t];
    const double piv = __shfl_sync(0xffffffffu, v, c);
    if (c < w && !(piv > 0.0)) return false;
    const double l = sqrt(piv);
    if (lane == c) s.T[o + c][o + c] = l;
    else if (lane > c) s.T[o + lane][o + c] = v / l;
    __syncwarp();
  }
  for (int r = 0; r < 32; ++r) {
    if (r == lane) {
      s.Di[o + r][o + lane] = 1.0 / s.T[o + r][o + r];
    } else if (r > lane) {
      double acc = 0.0;
      for (int t = lane; t < r; ++t) acc += s.T[o + r][o + t] * s.Di[o + t][o + lane];
      s.Di[o + r][o + lane] = -acc / s.T[o + r][o + r];
    } else {
      s.Di[o + r][o + lane] = 0.0;
    }
    __syncwarp();
  }
  return true;
}

// Factor + invert the 64 x 64 diagonal block at (j0, j0) (w valid rows).
__device__ bool pc_small(double* A, int b, int j0, int w, double* dinv_out, PcSmallSmem& s) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < 64 * 64; e += blockDim.x) {
    const int r = e >> 6, c = e & 63;
    s.T[r][c] = (r < w && c <= r) ? A[(int64_t)(j0 + r) * b + j0 + c] : (r == c ? 1.0 : 0.0);
  }
  if (tid == 0) s.bad = 0;
  __syncthreads();
  if (warp == 0 && !pc_factor32(s, 0, min(w, 32), lane)) s.bad = 1;
  __syncthreads();
  if (s.bad) return false;
  // L21 = A21 * Di11^T (registers first: in place)
  {
    const int r = tid >> 2, cb = (tid & 3) * 8;
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double acc = 0.0;
      for (int t = 0; t <= cb + u; ++t) acc += s.T[32 + r][t] * s.Di[cb + u][t];
      x[u] = acc;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 8; ++u) s.T[32 + r][cb + u] = x[u];
  }
  __syncthreads();
  // A22 -= L21 L21^T (lower)
  for (int e = tid; e < 32 * 32; e += blockDim.x) {
    const int r = e >> 5, c = e & 31;
    if (c > r) continue;
    double acc = 0.0;
    for (int t = 0; t < 32; ++t) acc += s.T[32 + r][t] * s.T[32 + c][t];
    s.T[32 + r][32 + c] -= acc;
  }
  __syncthreads();
  if (warp == 0 && !pc_factor32(s, 32, max(0, w - 32), lane)) s.bad = 1;
  __syncthreads();
  if (s.bad) return false;
  // Di21 = -Di22 (L21 Di11):  M = L21 Di11, then Di21 = -Di22 M
  for (int e = tid; e < 32 * 32; e += blockDim.x) {
    const int r = e >> 5, c = e & 31;
    double acc = 0.0;
    for (int t = c; t < 32; ++t) acc += s.T[32 + r][t] * s.Di[t][c];
    s.M[r][c] = acc;
  }
  __syncthreads();
  for (int e = tid; e < 32 * 32; e += blockDim.x) {
    const int r = e >> 5, c = e & 31;
    double acc = 0.0;
    for (int t = 0; t <= r; ++t) acc += s.Di[32 + r][32 + t] * s.M[t][c];
    s.Di[32 + r][c] = -acc;
    s.Di[r][32 + c] = 0.0;
  }
  __syncthreads();
  for (int e = tid; e < 64 * 64; e += blockDim.x) {
    const int r = e >> 6, c = e & 63;
    if (r < w && c <= r) A[(int64_t)(j0 + r) * b + j0 + c] = s.T[r][c];
    dinv_out[e] = s.Di[r][c];
  }
  return true;
}

__device__ __forceinline__ double* blk(double* A, int b, int r, int c) {
  return A + (int64_t)r * PC_BLK * b + (int64_t)c * PC_BLK;
}

// Pipelined schedule, two grid barriers per 64-row block step s:
//   phase A: TRSM X_rs = A_rs D_s^{-T} (r > s)   |  TRTRI  X_sc = D_s^{-1} R_sc (c <= s)
//   phase B: CTA 0 updates block (s+1, s+1) and factors/inverts it (lookahead)
//            | the rest: A_rc -= X_rs X_cs^T (s < c <= r, not (s+1,s+1))
//            | TRTRI R_rc -= L_rs X_sc (r > s, c <= s)
__global__ void __launch_bounds__(DG_THREADS) k_potrf_coop(double* __restrict__ A, int b, int bk,
                                                           double* __restrict__ Linv,
                                                           double* __restrict__ dinv_all, int* fail, int k) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) uint8_t pc_smem[];
  DgSmem& sm = *reinterpret_cast<DgSmem*>(pc_smem);
  PcSmallSmem& ss = *reinterpret_cast<PcSmallSmem*>(pc_smem);
  if (*(volatile int*)fail >= 0) return;  // uniform across the grid
  const int nblk = (bk + PC_BLK - 1) / PC_BLK;
  const int G = gridDim.x, cta = blockIdx.x;
  auto rows_of = [&](int r) { return min(PC_BLK, bk - r * PC_BLK); };
  double acc[4][4][2];
  // Prologue: Linv <- I (all CTAs) while CTA 0 factors block 0.
  for (int64_t e = (int64_t)cta * blockDim.x + threadIdx.x; e < (int64_t)b * b; e += (int64_t)G * blockDim.x) {
    const int r = (int)(e / b), c = (int)(e % b);
    Linv[e] = (r == c && r < bk) ? 1.0 : 0.0;
  }
  if (cta == 0 && !pc_small(A, b, 0, rows_of(0), dinv_all, ss) && threadIdx.x == 0) atomicCAS(fail, -1, k);
  __threadfence();
  grid.sync();
  for (int s = 0; s < nblk; ++s) {
    if (*(volatile int*)fail >= 0) return;
    const int w = rows_of(s);
    const double* dinv = dinv_all + (int64_t)s * PC_BLK * PC_BLK;
    // ---- phase A ----
    const int n_trsm = nblk - s - 1;
    for (int item = cta; item < n_trsm + s + 1; item += G) {
      if (item < n_trsm) {  // TRSM, in place (one CTA owns each block)
        const int r = s + 1 + item;
        RowMajorK a{blk(A, b, r, s), b, rows_of(r), w};
        RowMajorK d{dinv, PC_BLK, PC_BLK, w};
        dgemm_64x64(a, d, w, sm, acc);
        double* out = blk(A, b, r, s);
        const int rr = rows_of(r);
        dg_for_each(acc, [&](int i, int j, double v) {
          if (i < rr && j < w) out[(int64_t)i * b + j] = v;
        });
      } else {  // TRTRI X_sc = Dinv_s R_sc, in place
        const int c = item - n_trsm;
        RowMajorK d{dinv, PC_BLK, w, w};
        KMajor rsc{blk(Linv, b, s, c), b, rows_of(c), w};
        dgemm_64x64(d, rsc, w, sm, acc);
        double* out = blk(Linv, b, s, c);
        const int cc = rows_of(c);
        dg_for_each(acc, [&](int i, int j, double v) {
          if (i < w && j < cc) out[(int64_t)i * b + j] = v;
        });
      }
      __syncthreads();
    }
    __threadfence();
    grid.sync();
    // ---- phase B ----
    if (cta == 0) {
      if (s + 1 < nblk) {
        const int r = s + 1, rr = rows_of(r);
        RowMajorK x1{blk(A, b, r, s), b, rr, w};
        dgemm_64x64(x1, x1, w, sm, acc);
        double* out = blk(A, b, r, r);
        dg_for_each(acc, [&](int i, int j, double v) {
          if (i < rr && j <= i) out[(int64_t)i * b + j] -= v;
        });
        __syncthreads();
        if (!pc_small(A, b, r * PC_BLK, rr, dinv_all + (int64_t)r * PC_BLK * PC_BLK, ss) && threadIdx.x == 0)
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
          dgemm_64x64(x1, x2, w, sm, acc);
          double* out = blk(A, b, r, c);
          const int rr = rows_of(r), cc = rows_of(c);
          dg_for_each(acc, [&](int i, int j, double v) {
            if (i < rr && j < cc && (r != c || j <= i)) out[(int64_t)i * b + j] -= v;
          });
        } else {
          const int q = item - (pairs - 1);
          const int r = s + 1 + q / (s + 1), c = q % (s + 1);
          RowMajorK l{blk(A, b, r, s), b, rows_of(r), w};
          KMajor x{blk(Linv, b, s, c), b, rows_of(c), w};
          dgemm_64x64(l, x, w, sm, acc);
          double* out = blk(Linv, b, r, c);
          const int rr = rows_of(r), cc = rows_of(c);
          dg_for_each(acc, [&](int i, int j, double v) {
            if (i < rr && j < cc) out[(int64_t)i * b + j] -= v;
          });
        }
        __syncthreads();
      }
    }
    __threadfence();
    grid.sync();
  }
  // Strict upper part to zero (potrf_tile's final loop).
  for (int64_t e = (int64_t)cta * blockDim.x + threadIdx.x; e < (int64_t)b * b; e += (int64_t)G * blockDim.x) {
    const int r = (int)(e / b), c = (int)(e % b);
    if (c > r) A[e] = 0.0;
  }
}

inline size_t potrf_coop_smem() {
  return sizeof(PcSmallSmem) > sizeof(DgSmem) ? sizeof(PcSmallSmem) : sizeof(DgSmem);
}

}  // namespace sphemu_gpu
