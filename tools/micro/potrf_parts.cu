// Microbenchmark of the cooperative POTRF ingredients (development aid).
#include <cstdio>
#include "../../paper_2408_04440_b200/csrc/potrf_coop.cuh"
using namespace sphemu_gpu;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void k_sync_bench(int iters, unsigned long long* out) {
  namespace cg = cooperative_groups;
  cg::grid_group g = cg::this_grid();
  g.sync();
  unsigned long long t0 = gtime();
  for (int i = 0; i < iters; ++i) {
    __threadfence();
    g.sync();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = gtime() - t0;
}

__global__ void k_small_bench(double* A, int b, double* dinv, int iters, unsigned long long* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  PcSmallSmem& ss = *reinterpret_cast<PcSmallSmem*>(sm);
  unsigned long long t0 = gtime();
  for (int i = 0; i < iters; ++i) pc_small(A, b, 0, 64, dinv, ss);
  __syncthreads();
  if (threadIdx.x == 0) out[1] = gtime() - t0;
}

__global__ void k_gemm_bench(double* A, int b, int iters, unsigned long long* out) {
  __shared__ DgSmem sm;
  double acc[4][4][2];
  unsigned long long t0 = gtime();
  for (int i = 0; i < iters; ++i) {
    RowMajorK x1{A + 64 * b, b, 64, 64};
    RowMajorK x2{A + 128 * b, b, 64, 64};
    dgemm_64x64(x1, x2, 64, sm, acc);
    double* o = A + 192 * b + 64;
    dg_for_each(acc, [&](int r, int c, double v) { o[(int64_t)r * b + c] -= v * 1e-30; });
    __syncthreads();
  }
  if (threadIdx.x == 0) out[2] = gtime() - t0;
}

int main() {
  const int b = 512;
  double* A;
  cudaMalloc(&A, sizeof(double) * b * b);
  double* hA = new double[b * b];
  for (int i = 0; i < b * b; ++i) hA[i] = 0.0;
  for (int i = 0; i < b; ++i) hA[i * b + i] = 4.0;
  for (int i = 1; i < b; ++i) hA[i * b + i - 1] = 1.0;
  cudaMemcpy(A, hA, sizeof(double) * b * b, cudaMemcpyHostToDevice);
  double* dinv;
  cudaMalloc(&dinv, sizeof(double) * 64 * 64 * 16);
  unsigned long long* out;
  cudaMalloc(&out, 64);
  int iters = 200;
  for (int G : {8, 16, 32, 64}) {
    void* args[] = {&iters, &out};
    cudaLaunchCooperativeKernel((void*)k_sync_bench, G, 128, args, 0, 0);
    cudaDeviceSynchronize();
    unsigned long long h[3];
    cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
    printf("grid.sync G=%d: %.2f us per sync\n", G, h[0] / 1e3 / iters);
  }
  cudaFuncSetAttribute(k_small_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PcSmallSmem));
  iters = 50;
  k_small_bench<<<1, 128, sizeof(PcSmallSmem)>>>(A, b, dinv, iters, out);
  k_gemm_bench<<<1, 128>>>(A, b, iters, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[3];
  cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
  printf("pc_small: %.2f us each; dgemm 64^3 + RMW epilogue: %.2f us each (%s)\n", h[1] / 1e3 / iters,
         h[2] / 1e3 / iters, cudaGetErrorString(e));
  return 0;
}
