// pc_small in isolation (one CTA, fresh SPD input each iteration) for ncu.
#include <cmath>
#include <cstdio>
#include <vector>
#include "../../paper_2408_04440_b200/csrc/potrf_coop.cuh"
using namespace sphemu_gpu;

__global__ void k_small(const double* pristine, double* A, int b, double* dinv, int iters, unsigned long long* out) {
  extern __shared__ __align__(16) uint8_t sm[];
  PcSmallSmem& ss = *reinterpret_cast<PcSmallSmem*>(sm);
  unsigned long long tot = 0;
  for (int i = 0; i < iters; ++i) {
    for (int e = threadIdx.x; e < 64 * 64; e += blockDim.x) A[(e >> 6) * b + (e & 63)] = pristine[e];
    __syncthreads();
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    bool ok = pc_small(A, b, 0, 64, dinv, ss);
    __syncthreads();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    tot += t1 - t0;
    if (!ok && threadIdx.x == 0) out[1] = 1;
  }
  if (threadIdx.x == 0) out[0] = tot;
}

int main() {
  const int b = 512;
  std::vector<double> h(64 * 64, 0.0);
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) h[i * 64 + j] = (i == j) ? 2.0 : 0.5 * std::pow(0.9, std::abs(i - j));
  double *P, *A, *dinv;
  unsigned long long* out;
  cudaMalloc(&P, 8 * 64 * 64);
  cudaMalloc(&A, 8 * b * b);
  cudaMalloc(&dinv, 8 * 64 * 64);
  cudaMalloc(&out, 16);
  cudaMemset(out, 0, 16);
  cudaMemcpy(P, h.data(), 8 * 64 * 64, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(PcSmallSmem));
  const int iters = 20;
  k_small<<<1, 128, sizeof(PcSmallSmem)>>>(P, A, b, dinv, iters, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long r[2];
  cudaMemcpy(r, out, 16, cudaMemcpyDeviceToHost);
  printf("pc_small %.2f us (fail %llu, %s)\n", r[0] / 1e3 / iters, r[1], cudaGetErrorString(e));
  return 0;
}
