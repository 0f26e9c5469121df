// cov_kernels.cuh — innovation covariance U = Xi^T Xi / n on the FP64 tensor
// pipe (stochastic.cpp:109-136): Xi (n x d, row-major) is transposed once to
// Xt (d x ldt, the sample index contiguous), then every lower 128 x 64 block
// of U is a DMMA GEMM with K = n (dgemm2 kNT, A = B = Xt) whose epilogue
// divides by n and writes both the block and its mirror, so U is exactly
// symmetric (the reference's (U + U^T) / 2 is then the identity).
#pragma once

#include "dgemm2.cuh"

namespace sphemu_gpu {

// Xt[c][r] = X[r][c]; columns r >= n of Xt (padding to an even stride) are 0.
static __global__ void k_transpose_pad(const double* __restrict__ X, int64_t n, int d, double* __restrict__ Xt,
                                       int64_t ldt) {
  __shared__ double t[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k;
    const int c = c0 + threadIdx.x;
    t[k][threadIdx.x] = (r < n && c < d) ? X[r * d + c] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k;
    const int64_t r = r0 + threadIdx.x;
    if (c < d && r < ldt) Xt[(int64_t)c * ldt + r] = t[threadIdx.x][k];
  }
}

// One lower block (rows i0.., cols j0..) of U per CTA; blocks strictly above
// the diagonal exit. blockIdx.x enumerates (row block, col block) pairs.
static __global__ void __launch_bounds__(D2_THREADS) k_cov_syrk(const double* __restrict__ Xt, int64_t ldt, int64_t n,
                                                                int d, double inv_n, double* __restrict__ U) {
  extern __shared__ __align__(16) uint8_t d2_smem[];
  D2Smem& sm = *reinterpret_cast<D2Smem*>(d2_smem);
  const int i0 = blockIdx.y * D2_BM, j0 = blockIdx.x * D2_BN;
  if (j0 >= i0 + D2_BM || i0 >= d || j0 >= d) return;
  D2Op A{Xt + (int64_t)i0 * ldt, ldt, min(D2_BM, d - i0), (int)n};
  D2Op B{Xt + (int64_t)j0 * ldt, ldt, min(D2_BN, d - j0), (int)n};
  double acc[4][4][2];
  dgemm2_128x64<D2B::kNT, true>(A, B, (int)n, sm, acc);
  d2_for_each(acc, [&](int r, int c, double v0, double v1) {
    const int gi = i0 + r;
    const double w[2] = {v0 / (double)n, v1 / (double)n};
    (void)inv_n;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int gj = j0 + c + e;
      if (gi < d && gj < d && gj <= gi) {
        U[(int64_t)gi * d + gj] = w[e];
        U[(int64_t)gj * d + gi] = w[e];
      }
    }
  });
}

}  // namespace sphemu_gpu
