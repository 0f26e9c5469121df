// chol_kernels.cuh — device kernels of the tiled mixed-precision Cholesky
// (proj/src/mpchol.cpp:207-316): tile generation / load / store, the FP64
// POTRF + TRTRI of the diagonal tile, the FP64 panel TRSM (as a GEMM with the
// inverted diagonal tile), the panel scatter, and the FP64 (DMMA) trailing
// update for DP-class output tiles.
#pragma once

#include "common.cuh"
#include "dgemm.cuh"
#include "dgemm2.cuh"

namespace sphemu_gpu {

// HBM layout of the lower-triangular tiled matrix: tile (i, j), j <= i, packed
// by i(i+1)/2 + j, each padded to b x b row-major at its storage precision.
struct TileStore {
  char* base;
  const int64_t* off;   // byte offset per packed tile
  const uint8_t* prec;  // StorePrec per packed tile
  int n, b, nt;         // b = storage pitch (tile size padded to the kernel granule)
  int lb;               // logical tile size (MpCholConfig::tile_size)
  __device__ __forceinline__ int64_t idx(int i, int j) const { return (int64_t)i * (i + 1) / 2 + j; }
  __device__ __forceinline__ void* tile(int i, int j) const { return base + off[idx(i, j)]; }
  __device__ __forceinline__ int tprec(int i, int j) const { return prec[idx(i, j)]; }
  __device__ __forceinline__ int rows(int i) const { return min(lb, n - i * lb); }
  __device__ __forceinline__ bool owned(int i, int j) const { return off[idx(i, j)] >= 0; }
};

__device__ __forceinline__ void pair_from_index(int64_t p, int& a, int& c) {
  // p -> (a, c) with a >= c >= 0, p = a(a+1)/2 + c
  int64_t x = (int64_t)((sqrt(8.0 * (double)p + 1.0) - 1.0) * 0.5);
  while (x * (x + 1) / 2 > p) --x;
  while ((x + 1) * (x + 2) / 2 <= p) ++x;
  a = (int)x;
  c = (int)(p - x * (x + 1) / 2);
}

__device__ __forceinline__ void flush_sat(unsigned local, unsigned* sat) {
  local = warp_sum_u32(local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(sat, local);
}

// make_spd_test_matrix (mpchol.cpp:419-435) written straight into the tiles:
// a_ii = d_i*d_i*1.25, a_ij = d_i*d_j*0.25*pw[i-j] with i the larger index,
// multiplied in the reference's left-to-right order (bitwise equal), then
// stored through the tile precision (mpchol.cpp:360-363).
static __global__ void k_gen_spd(TileStore ts, const double* __restrict__ d, const double* __restrict__ pw,
                          unsigned* sat) {
  const int64_t t = blockIdx.x;
  if (ts.off[t] < 0) return;  // tile owned by another rank
  int i, j;
  pair_from_index(t, i, j);
  void* tp = ts.tile(i, j);
  const int p = ts.tprec(i, j);
  const int b = ts.b;
  unsigned local = 0;
  auto value = [&](int r, int c) {
    const int R = i * ts.lb + r, Cc = j * ts.lb + c;
    double v = 0.0;
    if (r < ts.lb && c < ts.lb && R < ts.n && Cc < ts.n) {
      if (R == Cc) v = __dmul_rn(__dmul_rn(d[R], d[R]), 1.25);
      else if (R > Cc) v = __dmul_rn(__dmul_rn(__dmul_rn(d[R], d[Cc]), 0.25), pw[R - Cc]);
      else v = __dmul_rn(__dmul_rn(__dmul_rn(d[Cc], d[R]), 0.25), pw[Cc - R]);
    }
    return v;
  };
  if ((b & 7) == 0) {
    // 8 consecutive elements of a row per thread: one 16 / 32 / 64-byte store
    for (int64_t g = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; g < (int64_t)b * b / 8;
         g += (int64_t)gridDim.y * blockDim.x) {
      const int64_t e = g * 8;
      const int r = (int)(e / b), c = (int)(e % b);
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = value(r, c + u);
      if (p == kDP) {
        double2* q = reinterpret_cast<double2*>(static_cast<double*>(tp) + e);
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = make_double2(v[2 * u], v[2 * u + 1]);
      } else if (p == kSP) {
        float4* q = reinterpret_cast<float4*>(static_cast<float*>(tp) + e);
        q[0] = make_float4(__double2float_rn(v[0]), __double2float_rn(v[1]), __double2float_rn(v[2]), __double2float_rn(v[3]));
        q[1] = make_float4(__double2float_rn(v[4]), __double2float_rn(v[5]), __double2float_rn(v[6]), __double2float_rn(v[7]));
      } else {
        uint16_t h[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          h[u] = p == kHP ? __half_as_ushort(to_half_sat(v[u], local)) : __bfloat16_as_ushort(to_bf16_sat(v[u], local));
        *reinterpret_cast<uint4*>(static_cast<uint16_t*>(tp) + e) = *reinterpret_cast<const uint4*>(h);
      }
    }
  } else {
    for (int64_t e = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; e < (int64_t)b * b;
         e += (int64_t)gridDim.y * blockDim.x)
      store_elem(tp, p, e, value((int)(e / b), (int)(e % b)), local);
  }
  flush_sat(local, sat);
}

// TiledMatrix::from_dense (mpchol.cpp:124-138) + input quantization.
// t0 / row0: launch over a run of packed tiles starting at t0, reading a
// slab whose first row is global row row0 (the streamed host input).
// diag_shift: added to the diagonal before quantization (the nugget of
// stochastic.cpp:147-151, dense = u + nugget * I).
static __global__ void k_load_dense(TileStore ts, const double* __restrict__ a, int64_t lda, unsigned* sat,
                                    int64_t t0 = 0, int row0 = 0, double diag_shift = 0.0) {
  const int64_t t = t0 + blockIdx.x;
  if (ts.off[t] < 0) return;  // tile owned by another rank
  int i, j;
  pair_from_index(t, i, j);
  void* tp = ts.tile(i, j);
  const int p = ts.tprec(i, j);
  const int b = ts.b;
  unsigned local = 0;
  for (int64_t e = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; e < (int64_t)b * b;
       e += (int64_t)gridDim.y * blockDim.x) {
    const int r = (int)(e / b), c = (int)(e % b);
    const int R = i * ts.lb + r, Cc = j * ts.lb + c;
    double v = (r < ts.lb && c < ts.lb && R < ts.n && Cc < ts.n) ? a[(int64_t)(R - row0) * lda + Cc] : 0.0;
    if (R == Cc && R < ts.n) v += diag_shift;
    store_elem(tp, p, e, v, local);
  }
  flush_sat(local, sat);
}

// Vectorized form of k_load_dense (device input, n and the tile size
// multiples of 8, 16-byte aligned rows): 8 consecutive columns per thread and
// iteration, 4 x 16-byte loads in flight, one 16/32/64-byte store per group.
static __global__ void k_load_dense8(TileStore ts, const double* __restrict__ a, int64_t lda, unsigned* sat,
                                     double diag_shift) {
  const int64_t t = blockIdx.x;
  if (ts.off[t] < 0) return;
  int i, j;
  pair_from_index(t, i, j);
  void* tp = ts.tile(i, j);
  const int p = ts.tprec(i, j);
  const int b = ts.b;
  unsigned local = 0;
  for (int64_t g = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; g < (int64_t)b * b / 8;
       g += (int64_t)gridDim.y * blockDim.x) {
    const int64_t e = g * 8;
    const int r = (int)(e / b), c = (int)(e % b);
    const int R = i * ts.lb + r, Cc = j * ts.lb + c;
    double v[8];
    if (r < ts.lb && c < ts.lb && R < ts.n && Cc < ts.n) {
      const double2* q = reinterpret_cast<const double2*>(a + (int64_t)R * lda + Cc);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 x = __ldcs(q + u);
        v[2 * u] = x.x;
        v[2 * u + 1] = x.y;
      }
      if (R >= Cc && R < Cc + 8) v[R - Cc] += diag_shift;
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = 0.0;
    }
    if (p == kDP) {
      double2* q = reinterpret_cast<double2*>(static_cast<double*>(tp) + e);
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = make_double2(v[2 * u], v[2 * u + 1]);
    } else if (p == kSP) {
      float4* q = reinterpret_cast<float4*>(static_cast<float*>(tp) + e);
      q[0] = make_float4(__double2float_rn(v[0]), __double2float_rn(v[1]), __double2float_rn(v[2]), __double2float_rn(v[3]));
      q[1] = make_float4(__double2float_rn(v[4]), __double2float_rn(v[5]), __double2float_rn(v[6]), __double2float_rn(v[7]));
    } else {
      uint16_t h[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        h[u] = p == kHP ? __half_as_ushort(to_half_sat(v[u], local)) : __bfloat16_as_ushort(to_bf16_sat(v[u], local));
      *reinterpret_cast<uint4*>(static_cast<uint16_t*>(tp) + e) = *reinterpret_cast<const uint4*>(h);
    }
  }
  flush_sat(local, sat);
}

// Packed host I/O (single GPU, host buffers): a tile row crosses the host
// link at its storage width — DP tiles as fp64, every other class as fp32
// (the reference's quantize goes double -> float first, so the float is the
// exact value the device stores or rounds further to binary16 / bf16). Each
// tile's segment of a row is padded to 16 bytes.
__host__ __device__ __forceinline__ int64_t packed_seg_bytes(int cw, int prec) {
  return ((int64_t)cw * (prec == kDP ? 8 : 4) + 15) & ~(int64_t)15;
}

// Row block i (tiles j = 0..i) from a packed slab with rowbytes per row.
static __global__ void k_load_packed(TileStore ts, const char* __restrict__ blk, int64_t rowbytes, unsigned* sat,
                                     int i, double diag_shift) {
  const int j = blockIdx.x;
  int64_t seg = 0;
  for (int jj = 0; jj < j; ++jj) seg += packed_seg_bytes(min(ts.lb, ts.n - jj * ts.lb), ts.tprec(i, jj));
  void* tp = ts.tile(i, j);
  const int p = ts.tprec(i, j);
  const int b = ts.b;
  const int rows = min(ts.lb, ts.n - i * ts.lb), cw = min(ts.lb, ts.n - j * ts.lb);
  unsigned local = 0;
  for (int64_t e = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; e < (int64_t)b * b;
       e += (int64_t)gridDim.y * blockDim.x) {
    const int r = (int)(e / b), c = (int)(e % b);
    double v = 0.0;
    if (r < rows && c < cw) {
      const char* row = blk + (int64_t)r * rowbytes + seg;
      v = p == kDP ? reinterpret_cast<const double*>(row)[c] : (double)reinterpret_cast<const float*>(row)[c];
      if (i == j && r == c) v += diag_shift;
    }
    store_elem(tp, p, e, v, local);
  }
  flush_sat(local, sat);
}

// Tile columns [k0, k1) of the factor, packed: one CTA per output row R >=
// k0 lb; row-block byte offsets rb_off[i] (from k0's block) and row widths
// rb_bytes[i] come from the host. Zeros above the diagonal inside the
// diagonal tile, like k_store_cols.
static __global__ void k_store_cols_packed(TileStore ts, int k0, int k1, const int64_t* __restrict__ rb_off,
                                           const int64_t* __restrict__ rb_bytes, char* __restrict__ slab) {
  const int R = k0 * ts.lb + blockIdx.x;
  const int i = R / ts.lb;
  char* row = slab + rb_off[i] + (int64_t)(R - i * ts.lb) * rb_bytes[i];
  const int64_t rb = (int64_t)(R % ts.lb) * ts.b;
  for (int j = k0; j < k1 && j <= i; ++j) {
    const int p = ts.tprec(i, j);
    const int cw = min(ts.lb, ts.n - j * ts.lb);
    const void* tp = ts.tile(i, j);
    for (int c = threadIdx.x; c < cw; c += blockDim.x) {
      const int C = j * ts.lb + c;
      const double v = C <= R ? load_elem(tp, p, rb + c) : 0.0;
      if (p == kDP) reinterpret_cast<double*>(row)[c] = v;
      else reinterpret_cast<float*>(row)[c] = (float)v;  // exact: the stored value is a float or narrower
    }
    row += packed_seg_bytes(cw, p);
  }
}

// TiledMatrix::to_dense_lower (mpchol.cpp:140-154): lower part from the
// tiles, exact zeros above the diagonal. One thread per output element.
static __global__ void k_store_dense(TileStore ts, double* __restrict__ out, int64_t ldo) {
  for (int R = blockIdx.y; R < ts.n; R += gridDim.y)  // gridDim.y <= 65535
  for (int Cc = blockIdx.x * blockDim.x + threadIdx.x; Cc < ts.n; Cc += gridDim.x * blockDim.x) {
    double v = 0.0;
    if (Cc <= R) {
      const int i = R / ts.lb, j = Cc / ts.lb;
      v = load_elem(ts.tile(i, j), ts.tprec(i, j), (int64_t)(R % ts.lb) * ts.b + (Cc % ts.lb));
    }
    out[(int64_t)R * ldo + Cc] = v;
  }
}

// Tile column k of the factor as a dense (n - k lb) x lb slab (pitch lb):
// exact zeros above the diagonal, one CTA per output row.
static __global__ void k_store_col(TileStore ts, int k, double* __restrict__ slab) {
  const int R = k * ts.lb + blockIdx.x;
  const int w = min(ts.lb, ts.n - k * ts.lb);
  const int i = R / ts.lb;
  const void* tp = ts.tile(i, k);
  const int p = ts.tprec(i, k);
  const int64_t rb = (int64_t)(R % ts.lb) * ts.b;
  for (int c = threadIdx.x; c < w; c += blockDim.x)
    slab[(int64_t)blockIdx.x * ts.lb + c] = (k * ts.lb + c <= R) ? load_elem(tp, p, rb + c) : 0.0;
}

// Tile columns [k0, k1) of the factor as a dense (n - k0 lb) x (k1 - k0) lb
// slab (pitch W): exact zeros above the diagonal, one CTA per output row.
static __global__ void k_store_cols(TileStore ts, int k0, int k1, int W, double* __restrict__ slab) {
  const int R = k0 * ts.lb + blockIdx.x;
  const int w = min(W, ts.n - k0 * ts.lb);
  const int i = R / ts.lb;
  const int64_t rb = (int64_t)(R % ts.lb) * ts.b;
  for (int c = threadIdx.x; c < w; c += blockDim.x) {
    const int C = k0 * ts.lb + c;
    double v = 0.0;
    if (C <= R) {
      const int j = C / ts.lb;
      v = load_elem(ts.tile(i, j), ts.tprec(i, j), rb + C % ts.lb);
    }
    slab[(int64_t)blockIdx.x * W + c] = v;
  }
  (void)k1;
}

// ---------------------------------------------------------------------------
// Diagonal tile: blocked right-looking POTRF (inner block 32) followed by the
// explicit inverse of the factor (used to turn the panel TRSM into a GEMM).
// One CTA of 512 threads; the tile (<= 1024^2 doubles) stays in L2.
// potrf_tile semantics (mpchol.cpp:230-252): fails when a pivot is not > 0,
// reporting the diagonal tile index; the strict upper part is zeroed.
// ---------------------------------------------------------------------------
constexpr int PT_THREADS = 256;

static __global__ void __launch_bounds__(PT_THREADS) k_potrf_trtri(double* __restrict__ A, int b, int bk,
                                                           double* __restrict__ Linv,
                                                           double* __restrict__ dinv_all,
                                                           int* fail, int k) {
  __shared__ double D[32][33];
  __shared__ double Di[32][33];
  __shared__ int bad;
  if (*(volatile int*)fail >= 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) bad = 0;
  __syncthreads();
  const int nblk = (bk + 31) / 32;
  for (int jb = 0; jb < bk; jb += 32) {
    const int w = min(32, bk - jb);
    for (int e = tid; e < 32 * 32; e += PT_THREADS) {
      const int r = e >> 5, c = e & 31;
      D[r][c] = (r < w && c <= r) ? A[(int64_t)(jb + r) * b + jb + c] : (r == c ? 1.0 : 0.0);
      Di[r][c] = 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      for (int c = 0; c < w; ++c) {
        double s = D[lane][c];
        for (int t = 0; t < c; ++t) s -= D[lane][t] * D[c][t];
        const double piv = __shfl_sync(0xffffffffu, s, c);
        if (!(piv > 0.0)) {
          if (lane == 0) bad = 1;
          break;
        }
        const double l = sqrt(piv);
        if (lane == c) D[c][c] = l;
        else if (lane > c && lane < w) D[lane][c] = s / l;
        __syncwarp();
      }
      __syncwarp();
      if (!bad) {
        // Di = D^{-1}: lane j owns column j (forward substitution).
        const int jcol = lane;
        for (int r = 0; r < 32; ++r) {
          if (r == jcol) {
            Di[r][jcol] = 1.0 / D[r][r];
          } else if (r > jcol) {
            double s = 0.0;
            for (int t = jcol; t < r; ++t) s += D[r][t] * Di[t][jcol];
            Di[r][jcol] = -s / D[r][r];
          }
          __syncwarp();
        }
      }
    }
    __syncthreads();
    if (bad) {
      if (tid == 0) atomicCAS(fail, -1, k);
      return;
    }
    // Write the factored block back and keep its inverse for TRTRI.
    for (int e = tid; e < 32 * 32; e += PT_THREADS) {
      const int r = e >> 5, c = e & 31;
      if (r < w && c <= r) A[(int64_t)(jb + r) * b + jb + c] = D[r][c];
      dinv_all[(int64_t)(jb / 32) * 1024 + e] = Di[r][c];
    }
    // Panel below the block: P <- P * Di^T.
    for (int r = jb + w + tid; r < bk; r += PT_THREADS) {
      double a[32];
      double* row = A + (int64_t)r * b + jb;
#pragma unroll
      for (int t = 0; t < 32; ++t) a[t] = t < w ? row[t] : 0.0;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        double x = 0.0;
#pragma unroll
        for (int t = 0; t <= c; ++t) x += a[t] * Di[c][t];
        if (c < w) row[c] = x;
      }
    }
    __syncthreads();
    // Trailing SYRK on the lower triangle, 32 x 32 blocks per warp (DMMA).
    const int m = bk - jb - w;
    if (m > 0) {
      const int nb2 = (m + 31) / 32;
      const int pairs = nb2 * (nb2 + 1) / 2;
      for (int p = warp; p < pairs; p += PT_THREADS / 32) {
        int I, J;
        pair_from_index(p, I, J);
        const int R0 = jb + w + I * 32, C0 = jb + w + J * 32;
        double acc[4][4][2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        for (int kk = 0; kk < w; kk += 4) {
          const int kc = kk + (lane & 3);
          double av[4], bv[4];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            const int r = R0 + mi * 8 + (lane >> 2);
            av[mi] = (r < bk && kc < w) ? A[(int64_t)r * b + jb + kc] : 0.0;
          }
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            const int r = C0 + ni * 8 + (lane >> 2);
            bv[ni] = (r < bk && kc < w) ? A[(int64_t)r * b + jb + kc] : 0.0;
          }
#pragma unroll
          for (int mi = 0; mi < 4; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], av[mi], bv[ni]);
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int r = R0 + mi * 8 + (lane >> 2), c = C0 + ni * 8 + (lane & 3) * 2 + e;
              if (r < bk && c <= r) A[(int64_t)r * b + c] -= acc[mi][ni][e];
            }
      }
    }
    __syncthreads();
  }
  // Zero the strict upper part (potrf_tile's final loop).
  for (int64_t e = tid; e < (int64_t)b * b; e += PT_THREADS) {
    const int r = (int)(e / b), c = (int)(e % b);
    if (c > r) A[e] = 0.0;
  }
  // TRTRI: Linv = L^{-1} by right-looking block forward substitution.
  for (int64_t e = tid; e < (int64_t)b * b; e += PT_THREADS) {
    const int r = (int)(e / b), c = (int)(e % b);
    Linv[e] = (r == c && r < bk) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int s = 0; s < nblk; ++s) {
    const int w = min(32, bk - s * 32);
    const double* dinv = dinv_all + (int64_t)s * 1024;
    // X_s = Dinv_s * R_s over columns [0, (s+1)*32).
    for (int col = tid; col < (s + 1) * 32 && col < bk; col += PT_THREADS) {
      double x[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) x[t] = t < w ? Linv[(int64_t)(s * 32 + t) * b + col] : 0.0;
#pragma unroll
      for (int r = 31; r >= 0; --r) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t <= r; ++t) acc += dinv[r * 32 + t] * x[t];
        x[r] = acc;
      }
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (t < w) Linv[(int64_t)(s * 32 + t) * b + col] = x[t];
    }
    __syncthreads();
    // R_r -= L_rs X_s for r > s, column blocks c <= s.
    const int rows_after = nblk - s - 1;
    const int pairs = rows_after * (s + 1);
    for (int p = warp; p < pairs; p += PT_THREADS / 32) {
      const int rb = s + 1 + p / (s + 1), cb = p % (s + 1);
      double acc[4][4][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      for (int kk = 0; kk < w; kk += 4) {
        const int kc = kk + (lane & 3);
        double av[4], bv[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int r = rb * 32 + mi * 8 + (lane >> 2);
          av[mi] = (r < bk && kc < w) ? A[(int64_t)r * b + s * 32 + kc] : 0.0;
        }
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          const int c = cb * 32 + ni * 8 + (lane >> 2);
          bv[ni] = (kc < w) ? Linv[(int64_t)(s * 32 + kc) * b + c] : 0.0;
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], av[mi], bv[ni]);
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int r = rb * 32 + mi * 8 + (lane >> 2), c = cb * 32 + ni * 8 + (lane & 3) * 2 + e;
            if (r < bk && c < bk) Linv[(int64_t)r * b + c] -= acc[mi][ni][e];
          }
    }
    __syncthreads();
  }
}

// Tile operand at its storage precision, element (r, k) of rows [r0, r0+64).
struct TileRowAcc {
  static constexpr bool kKContig = true;
  const void* base;
  int prec, ld, r0, rows, cols;
  __device__ double operator()(int r, int k) const {
    const int rr = r0 + r;
    return (rr < rows && k < cols) ? load_elem(base, prec, (int64_t)rr * ld + k) : 0.0;
  }
};

// Panel TRSM as a GEMM (mpchol.cpp:293-299): X_i = B_i * Linv^T written to
// the FP64 panel mirror, rounded through p(i, k). grid = (tiles*b/64, b/64).
static __global__ void __launch_bounds__(DG_THREADS) k_panel_trsm_fp64(TileStore ts, int k,
                                                                 const double* __restrict__ Linv,
                                                                 double* __restrict__ P64,
                                                                 const int* fail, unsigned* sat) {
  __shared__ DgSmem sm;
  if (*(volatile const int*)fail >= 0) return;
  const int sub_per = ts.b / DG_BM;
  const int i = k + 1 + blockIdx.x / sub_per;
  const int r0 = (blockIdx.x % sub_per) * DG_BM, c0 = blockIdx.y * DG_BN;
  const int b = ts.b;
  TileRowAcc A{ts.tile(i, k), ts.tprec(i, k), b, r0, b, b};
  RowMajorK B{Linv + (int64_t)c0 * b, b, DG_BN, b};
  double acc[4][4][2];
  dgemm_64x64(A, B, b, sm, acc);
  const int p = ts.tprec(i, k);
  double* out = P64 + (int64_t)(i - k - 1) * b * b;
  unsigned local = 0;
  dg_for_each(acc, [&](int r, int c, double v) {
    out[(int64_t)(r0 + r) * b + c0 + c] = quantize_value(v, p, local);
  });
  flush_sat(local, sat);
}

// Panel scatter: the rounded FP64 panel mirror back into the tiles (exact,
// the values are already representable at the tile precision).
static __global__ void k_panel_scatter(TileStore ts, int k, const double* __restrict__ P64, const int* fail) {
  if (*(volatile const int*)fail >= 0) return;
  const int b = ts.b;
  const int i = k + 1 + blockIdx.y;
  void* tp = ts.tile(i, k);
  const int p = ts.tprec(i, k);
  const double* src = P64 + (int64_t)blockIdx.y * b * b;
  unsigned dummy = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)b * b;
       e += (int64_t)gridDim.x * blockDim.x)
    store_elem(tp, p, e, src[e], dummy);
}

// Trailing update C(i,j) <- round_p(C(i,j) - P_i P_j^T) in FP64 (DMMA) for a
// list of output tiles (mpchol.cpp:300-314). One CTA per 64x64 sub-tile;
// strictly upper sub-tiles of diagonal (SYRK) tiles are skipped, the values
// there are never read and POTRF zeroes them.
static __global__ void __launch_bounds__(DG_THREADS) k_update_fp64(TileStore ts, int k,
                                                             const int2* __restrict__ list,
                                                             const double* __restrict__ P64,
                                                             const int* fail, unsigned* sat) {
  __shared__ DgSmem sm;
  if (*(volatile const int*)fail >= 0) return;
  const int b = ts.b;
  const int sub_side = b / DG_BM, per = sub_side * sub_side;
  const int2 ij = list[blockIdx.x / per];
  const int sub = blockIdx.x % per;
  const int r0 = (sub / sub_side) * DG_BM, c0 = (sub % sub_side) * DG_BN;
  const int i = ij.x, j = ij.y;
  if (i == j && c0 > r0) return;
  const double* Pi = P64 + (int64_t)(i - k - 1) * b * b;
  const double* Pj = P64 + (int64_t)(j - k - 1) * b * b;
  RowMajorK A{Pi + (int64_t)r0 * b, b, DG_BM, b};
  RowMajorK B{Pj + (int64_t)c0 * b, b, DG_BN, b};
  double acc[4][4][2];
  dgemm_64x64(A, B, b, sm, acc);
  void* tp = ts.tile(i, j);
  const int p = ts.tprec(i, j);
  unsigned local = 0;
  dg_for_each(acc, [&](int r, int c, double v) {
    const int64_t e = (int64_t)(r0 + r) * b + c0 + c;
    const double cur = load_elem(tp, p, e);
    store_elem(tp, p, e, cur - v, local);
  });
  flush_sat(local, sat);
}

// Same update on 128 x 64 sub-tiles with the cp.async DGEMM (dgemm2.cuh);
// needs b % 128 == 0. Sub-tiles strictly above the diagonal of SYRK tiles are
// skipped.
// k2 >= 0: merged two-step update, C -= P_k Q_k^T + P_k2 Q_k2^T (P64b = step k2's mirror).
static __global__ void __launch_bounds__(D2_THREADS) k_update_fp64_v2(TileStore ts, int k,
                                                                      const int2* __restrict__ list,
                                                                      const double* __restrict__ P64,
                                                                      const int* fail, unsigned* sat, int k2 = -1,
                                                                      const double* __restrict__ P64b = nullptr) {
  extern __shared__ __align__(16) uint8_t d2_smem[];
  D2Smem& sm = *reinterpret_cast<D2Smem*>(d2_smem);
  if (*(volatile const int*)fail >= 0) return;
  const int b = ts.b;
  const int sm_n = b / D2_BN, per = (b / D2_BM) * sm_n;
  const int2 ij = list[blockIdx.x / per];
  const int sub = blockIdx.x % per;
  const int r0 = (sub / sm_n) * D2_BM, c0 = (sub % sm_n) * D2_BN;
  const int i = ij.x, j = ij.y;
  if (i == j && c0 >= r0 + D2_BM) return;
  const double* Pi = P64 + (int64_t)(i - k - 1) * b * b;
  const double* Pj = P64 + (int64_t)(j - k - 1) * b * b;
  D2Op A{Pi + (int64_t)r0 * b, b, D2_BM, b};
  D2Op B{Pj + (int64_t)c0 * b, b, D2_BN, b};
  double acc[4][4][2];
  dgemm2_128x64<D2B::kNT, true>(A, B, b, sm, acc);
  if (k2 >= 0) {
    const double* Pi2 = P64b + (int64_t)(i - k2 - 1) * b * b;
    const double* Pj2 = P64b + (int64_t)(j - k2 - 1) * b * b;
    D2Op A2{Pi2 + (int64_t)r0 * b, b, D2_BM, b};
    D2Op B2{Pj2 + (int64_t)c0 * b, b, D2_BN, b};
    dgemm2_128x64<D2B::kNT, true>(A2, B2, b, sm, acc, false);
  }
  void* tp = ts.tile(i, j);
  const int p = ts.tprec(i, j);
  unsigned local = 0;
  if (p == kDP) {
    double* C = static_cast<double*>(tp);
    d2_for_each(acc, [&](int r, int c, double v0, double v1) {
      double2* q = reinterpret_cast<double2*>(C + (int64_t)(r0 + r) * b + c0 + c);
      double2 cur = *q;
      cur.x -= v0;
      cur.y -= v1;
      *q = cur;
    });
  } else {
    d2_for_each(acc, [&](int r, int c, double v0, double v1) {
      const int64_t e = (int64_t)(r0 + r) * b + c0 + c;
      store_elem(tp, p, e, load_elem(tp, p, e) - v0, local);
      store_elem(tp, p, e + 1, load_elem(tp, p, e + 1) - v1, local);
    });
  }
  flush_sat(local, sat);
}

// ||A - L L^T||_F^2 and ||A||_F^2 accumulated over 64x64 blocks of a dense
// row-major A and dense lower L (tests/support/reference.cpp:32-44).
static __global__ void __launch_bounds__(DG_THREADS) k_residual(const double* __restrict__ A, int64_t lda,
                                                         const double* __restrict__ L, int64_t ldl,
                                                         int n, double* sums) {
  __shared__ DgSmem sm;
  __shared__ double red[2][DG_THREADS / 32];
  const int r0 = blockIdx.y * DG_BM, c0 = blockIdx.x * DG_BN;
  const int kmax = min(min(r0 + DG_BM, c0 + DG_BN), n);
  RowMajorK La{L + (int64_t)r0 * ldl, ldl, min(DG_BM, n - r0), kmax};
  RowMajorK Lb{L + (int64_t)c0 * ldl, ldl, min(DG_BN, n - c0), kmax};
  double acc[4][4][2];
  dgemm_64x64(La, Lb, kmax, sm, acc);
  double num = 0.0, den = 0.0;
  dg_for_each(acc, [&](int r, int c, double v) {
    if (r0 + r < n && c0 + c < n) {
      const double a = A[(int64_t)(r0 + r) * lda + c0 + c];
      num += (a - v) * (a - v);
      den += a * a;
    }
  });
  num = warp_sum(num);
  den = warp_sum(den);
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = num;
    red[1][threadIdx.x >> 5] = den;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, d = 0;
    for (int w = 0; w < DG_THREADS / 32; ++w) {
      a += red[0][w];
      d += red[1][w];
    }
    atomicAdd(&sums[0], a);
    atomicAdd(&sums[1], d);
  }
}

}  // namespace sphemu_gpu
