// dgemm2.cuh — FP64 DMMA GEMM tile, 128 x 64 per CTA (256 threads = 4 x 2
// warps of 32 x 32), K staged by cp.async through a 3-stage shared-memory
// ring (16 doubles of K per stage). Out-of-range rows / K are zero-filled by
// the cp.async src-size operand, so no host-side padding is required, but
// every row start must be 16-byte aligned (ld and K offsets even).
//
//   A : M x K row-major (K contiguous)                       -> smem [m][k]
//   B : kNT  -> N x K row-major (K contiguous, C = A B^T)     -> smem [n][k]
//       kNN  -> K x N row-major (N contiguous, C = A B)       -> smem [k][n]
// Row strides in smem are padded (20 doubles for [x][k], 72 for [k][n]) so
// the m8n8k4 fragment loads hit two wavefronts (the minimum for 256 bytes).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "dgemm.cuh"

namespace sphemu_gpu {

constexpr int D2_BM = 128, D2_BN = 64, D2_BK = 16, D2_THREADS = 256, D2_STAGES = 3;
constexpr int D2_LDK = 20;  // [x][k] row stride (doubles)
constexpr int D2_LDN = 72;  // [k][n] row stride (doubles)

enum class D2B { kNT, kNN };

struct D2Smem {
  double a[D2_STAGES][D2_BM * D2_LDK];
  double b[D2_STAGES][D2_BK * D2_LDN > D2_BN * D2_LDK ? D2_BK * D2_LDN : D2_BN * D2_LDK];
};

__device__ __forceinline__ uint32_t smem_addr_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_addr_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_addr_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Operand view: base pointer, leading dimension, valid extents.
struct D2Op {
  const double* p;
  int64_t ld;
  int rows;  // valid rows (M or N for [x][k] views, K for the [k][n] view)
  int cols;  // valid cols (K for [x][k] views, N for the [k][n] view)
};

// Issue the cp.async copies of one K-chunk into stage buffers. V16: 16-byte
// copies (rows 16-byte aligned: ld and K offsets even); else 8-byte copies.
template <D2B BL, bool V16>
__device__ __forceinline__ void d2_load_stage(const D2Op& A, const D2Op& B, int k0, double* sa, double* sb) {
  constexpr int W = V16 ? 2 : 1;             // doubles per copy
  constexpr int KQ = D2_BK / W;              // copies per [x][k] row
  const int t = threadIdx.x;
#pragma unroll
  for (int e = 0; e < D2_BM * KQ / D2_THREADS; ++e) {
    const int idx = t + D2_THREADS * e;
    const int r = idx / KQ, kq = (idx % KQ) * W;
    const int k = k0 + kq;
    int bytes = 0;
    const double* src = A.p;
    if (r < A.rows && k < A.cols) {
      bytes = (A.cols - k >= W) ? 8 * W : 8;
      src = A.p + (int64_t)r * A.ld + k;
    }
    if constexpr (V16) cp_async16(sa + r * D2_LDK + kq, src, bytes);
    else cp_async8(sa + r * D2_LDK + kq, src, bytes);
  }
  if constexpr (BL == D2B::kNT) {
#pragma unroll
    for (int e = 0; e < D2_BN * KQ / D2_THREADS; ++e) {
      const int idx = t + D2_THREADS * e;
      const int r = idx / KQ, kq = (idx % KQ) * W;
      const int k = k0 + kq;
      int bytes = 0;
      const double* src = B.p;
      if (r < B.rows && k < B.cols) {
        bytes = (B.cols - k >= W) ? 8 * W : 8;
        src = B.p + (int64_t)r * B.ld + k;
      }
      if constexpr (V16) cp_async16(sb + r * D2_LDK + kq, src, bytes);
      else cp_async8(sb + r * D2_LDK + kq, src, bytes);
    }
  } else {
    constexpr int NQ = D2_BN / W;
#pragma unroll
    for (int e = 0; e < D2_BK * NQ / D2_THREADS; ++e) {
      const int idx = t + D2_THREADS * e;
      const int kr = idx / NQ, nq = (idx % NQ) * W;
      const int k = k0 + kr;
      int bytes = 0;
      const double* src = B.p;
      if (k < B.rows && nq < B.cols) {
        bytes = (B.cols - nq >= W) ? 8 * W : 8;
        src = B.p + (int64_t)k * B.ld + nq;
      }
      if constexpr (V16) cp_async16(sb + kr * D2_LDN + nq, src, bytes);
      else cp_async8(sb + kr * D2_LDN + nq, src, bytes);
    }
  }
}

// acc[mi][ni][e]: C(row, col), row = wm*32 + mi*8 + (lane>>2), col = wn*32 + ni*8 + (lane&3)*2 + e,
// wm = warp >> 1 (0..3), wn = warp & 1.
// zero = false: acc += A B (a second K range into the same accumulator).
template <D2B BL, bool V16>
__device__ void dgemm2_128x64(const D2Op& A, const D2Op& B, int K, D2Smem& sm, double (&acc)[4][4][2],
                              bool zero = true) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  if (zero) {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  }
  const int nk = (K + D2_BK - 1) / D2_BK;
  if (nk <= 0) return;
#pragma unroll
  for (int s = 0; s < D2_STAGES - 1; ++s) {
    if (s < nk) d2_load_stage<BL, V16>(A, B, s * D2_BK, sm.a[s], sm.b[s]);
    cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<D2_STAGES - 2>();
    __syncthreads();
    const int nxt = kc + D2_STAGES - 1;
    if (nxt < nk) d2_load_stage<BL, V16>(A, B, nxt * D2_BK, sm.a[nxt % D2_STAGES], sm.b[nxt % D2_STAGES]);
    cp_async_commit();
    const double* sa = sm.a[kc % D2_STAGES];
    const double* sb = sm.b[kc % D2_STAGES];
#pragma unroll
    for (int kk = 0; kk < D2_BK; kk += 4) {
      double a[4], b[4];
      const int kq = kk + (lane & 3);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = sa[(wm * 32 + mi * 8 + (lane >> 2)) * D2_LDK + kq];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int n = wn * 32 + ni * 8 + (lane >> 2);
        b[ni] = BL == D2B::kNT ? sb[n * D2_LDK + kq] : sb[kq * D2_LDN + n];
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
}

template <class F>
__device__ __forceinline__ void d2_for_each(const double (&acc)[4][4][2], F&& f) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp >> 1, wn = warp & 1;
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
      f(wm * 32 + mi * 8 + (lane >> 2), wn * 32 + ni * 8 + (lane & 3) * 2, acc[mi][ni][0], acc[mi][ni][1]);
}

}  // namespace sphemu_gpu
