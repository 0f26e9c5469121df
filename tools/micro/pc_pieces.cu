// Timing of the pc_small ingredients (development aid).
#include <cstdio>
#include "../../paper_2408_04440_b200/csrc/potrf_coop.cuh"
using namespace sphemu_gpu;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Candidate base case: lanes 0..15 own rows; the factored column is
// broadcast through shared memory instead of shuffles.
__device__ void base16_v2(PcSmallSmem& s, int o, int w, int lane, double* col) {
  const int row = lane & 15;
  double a[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) a[t] = s.T[o + row][o + t];
  bool ok = true;
  double rl[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    if (row == c) col[16] = a[c];
    __syncwarp();
    const double piv = col[16];
    if (c < w && !(piv > 0.0)) ok = false;
    rl[c] = rsqrt(piv);
    const double lrc = (row == c) ? piv * rl[c] : a[c] * rl[c];
    a[c] = lrc;
    if (lane < 16) col[row] = lrc;
    __syncwarp();
#pragma unroll
    for (int j = c + 1; j < 16; ++j) a[j] -= lrc * col[j];
    __syncwarp();
  }
  if (!ok) {
    if (lane == 0) s.bad = 1;
    return;
  }
  if (lane < 16)
#pragma unroll
    for (int t = 0; t < 16; ++t) s.T[o + lane][o + t] = t <= lane ? a[t] : 0.0;
  // inverse: lane j owns column j of X = L^{-1}; needs L[i][r] for all lanes -> via T in smem
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

template <int WHAT>
__global__ void k_piece(int iters, unsigned long long* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  PcSmallSmem& s = *reinterpret_cast<PcSmallSmem*>(sm);
  for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) {
    const int r = e >> 6, c = e & 63;
    s.T[r][c] = r == c ? 4.0 : (c < r ? 0.01 : 0.0);
    s.Di[r][c] = 0.0;
  }
  if (threadIdx.x == 0) s.bad = 0;
  __syncthreads();
  unsigned long long t0 = gtime();
  for (int i = 0; i < iters; ++i) {
    if (WHAT == 0) {
      if ((threadIdx.x >> 5) == 0) pc_base16(s, 0, 16, threadIdx.x & 31);
      __syncthreads();
    } else if (WHAT == 1) {
      pc_mm<16>([&](int r, int t) { return s.T[16 + r][t]; }, [&](int t, int c) { return s.Di[c][t]; },
                [&](int r, int c, double v) { s.M[r][c] = v; });
    } else if (WHAT == 6) {
      __shared__ double col[32];
      if ((threadIdx.x >> 5) == 0) base16_v2(s, 0, 16, threadIdx.x & 31, col);
      __syncthreads();
    } else if (WHAT == 5) {
      pc_mm_t<32>([&](int r, int t) { return s.T[32 + r][t]; }, [&](int t, int c) { return s.Di[c][t]; },
                  [&](int r, int c, double v) { s.M[r][c] = v; });
    } else if (WHAT == 2) {
      pc_mm<32>([&](int r, int t) { return s.T[32 + r][t]; }, [&](int t, int c) { return s.Di[c][t]; },
                [&](int r, int c, double v) { s.M[r][c] = v; });
    } else if (WHAT == 3) {
      pc_chol_inv<32>(s, 0, 32);
    } else {
      pc_chol_inv<64>(s, 0, 64);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[WHAT] = gtime() - t0;
}

int main() {
  unsigned long long* out;
  cudaMalloc(&out, 64);
  const int iters = 100;
  const char* names[] = {"base16", "pc_mm<16>", "pc_mm<32>", "chol_inv<32>", "chol_inv<64>", "pc_mm_t<32>", "base16_v2"};
  auto run = [&](auto kern, int w) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PcSmallSmem));
    kern<<<1, 128, sizeof(PcSmallSmem)>>>(iters, out);
    cudaDeviceSynchronize();
    unsigned long long h[7];
    cudaMemcpy(h, out, 56, cudaMemcpyDeviceToHost);
    printf("%-14s %8.3f us\n", names[w], h[w] / 1e3 / iters);
  };
  run(k_piece<0>, 0);
  run(k_piece<1>, 1);
  run(k_piece<2>, 2);
  run(k_piece<3>, 3);
  run(k_piece<4>, 4);
  run(k_piece<5>, 5);
  run(k_piece<6>, 6);
  return 0;
}
