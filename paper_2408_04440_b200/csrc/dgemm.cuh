// dgemm.cuh — FP64 tile GEMM on the B200 FP64 tensor pipe (DMMA,
// mma.sync.m8n8k4.f64). tcgen05 has no f64 kind, so every FP64 contraction of
// the hot path (DP-class Cholesky tiles, SHT Legendre stages, plan build)
// goes through this 64x64-per-CTA building block: 128 threads = 2x2 warps of
// 32x32, K staged through double-buffered shared memory in chunks of 16.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sphemu_gpu {

constexpr int DG_BM = 64, DG_BN = 64, DG_BK = 16, DG_THREADS = 128, DG_PAD = 8;
constexpr int DG_LDS = DG_BM + DG_PAD;  // 72 doubles per k-row: conflict-free fragment loads

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Shared staging: [2 buffers][BK][LDS] for A and for B.
struct DgSmem {
  double a[2][DG_BK][DG_LDS];
  double b[2][DG_BK][DG_LDS];
};

// Operand accessors. A(r, k) for r in [0,64), B(c, k) for c in [0,64).
// kKContig selects the coalesced mapping: true when consecutive k are
// adjacent in memory (row-major A / "NT" B), false when consecutive r (or c)
// are adjacent (K x N row-major B of an "NN" product).
// Each accessor returns 0 outside its valid extent.
struct RowMajorK {  // element (r, k) at base[r * ld + k]
  static constexpr bool kKContig = true;
  const double* base;
  int64_t ld;
  int rows, cols;  // valid r < rows, k < cols
  __device__ double operator()(int r, int k) const {
    return (r < rows && k < cols) ? base[(int64_t)r * ld + k] : 0.0;
  }
};

struct KMajor {  // element (c, k) at base[k * ld + c]  (K x N row-major)
  static constexpr bool kKContig = false;
  const double* base;
  int64_t ld;
  int rows, cols;  // valid c < rows, k < cols
  __device__ double operator()(int c, int k) const {
    return (c < rows && k < cols) ? base[(int64_t)k * ld + c] : 0.0;
  }
};

template <class Acc>
__device__ __forceinline__ void dg_load_chunk(const Acc& acc, int k0, double (&reg)[8]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int idx = t + DG_THREADS * e;  // 0..1023 over a 64 x 16 chunk
    int r, k;
    if constexpr (Acc::kKContig) {
      r = idx >> 4;
      k = idx & 15;
    } else {
      r = idx & 63;
      k = idx >> 6;
    }
    reg[e] = acc(r, k0 + k);
  }
}

template <class Acc>
__device__ __forceinline__ void dg_store_chunk(double (&dst)[DG_BK][DG_LDS], const double (&reg)[8]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int idx = t + DG_THREADS * e;
    int r, k;
    if constexpr (Acc::kKContig) {
      r = idx >> 4;
      k = idx & 15;
    } else {
      r = idx & 63;
      k = idx >> 6;
    }
    dst[k][r] = reg[e];
  }
}

// acc[mi][ni][e] holds C(row, col) with
//   row = wm*32 + mi*8 + (lane >> 2), col = wn*32 + ni*8 + (lane & 3)*2 + e.
template <class AccA, class AccB>
__device__ void dgemm_64x64(const AccA& A, const AccB& B, int K, DgSmem& sm,
                            double (&acc)[4][4][2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  if (K <= 0) return;
  double ra[8], rb[8];
  const int nk = (K + DG_BK - 1) / DG_BK;
  dg_load_chunk(A, 0, ra);
  dg_load_chunk(B, 0, rb);
  dg_store_chunk<AccA>(sm.a[0], ra);
  dg_store_chunk<AccB>(sm.b[0], rb);
  __syncthreads();
  for (int kc = 0; kc < nk; ++kc) {
    const int cur = kc & 1;
    if (kc + 1 < nk) {
      dg_load_chunk(A, (kc + 1) * DG_BK, ra);
      dg_load_chunk(B, (kc + 1) * DG_BK, rb);
    }
#pragma unroll
    for (int kk = 0; kk < DG_BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = sm.a[cur][kk + (lane & 3)][wm * 32 + mi * 8 + (lane >> 2)];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = sm.b[cur][kk + (lane & 3)][wn * 32 + ni * 8 + (lane >> 2)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
    if (kc + 1 < nk) {
      dg_store_chunk<AccA>(sm.a[cur ^ 1], ra);
      dg_store_chunk<AccB>(sm.b[cur ^ 1], rb);
    }
    __syncthreads();
  }
}

// Visits every accumulator element: f(row, col, value).
template <class F>
__device__ __forceinline__ void dg_for_each(const double (&acc)[4][4][2], F&& f) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e)
        f(wm * 32 + mi * 8 + (lane >> 2), wn * 32 + ni * 8 + (lane & 3) * 2 + e, acc[mi][ni][e]);
}

}  // namespace sphemu_gpu
