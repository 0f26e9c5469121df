// Timeline of one k_potrf_coop launch on a 512 x 512 tile (development aid).
#define SPHEMU_POTRF_TRACE 1
#include <cmath>
#include <cstdio>
#include <vector>
#include "../../paper_2408_04440_b200/csrc/potrf_coop.cuh"
using namespace sphemu_gpu;

int main() {
  const int b = 512;
  std::vector<double> h(b * b, 0.0);
  for (int i = 0; i < b; ++i)
    for (int j = 0; j <= i; ++j) h[i * b + j] = (i == j) ? 2.0 + i * 1e-3 : 0.5 * std::pow(0.9, i - j);
  double *A, *Linv, *dinv;
  int* fail;
  unsigned long long* tr;
  cudaMalloc(&A, 8 * b * b);
  cudaMalloc(&Linv, 8 * b * b);
  cudaMalloc(&dinv, 8 * 64 * 64 * 9);
  cudaMalloc(&fail, 4);
  unsigned* bar;
  cudaMalloc(&bar, 4);
  cudaMemset(bar, 0, 4);
  cudaMalloc(&tr, 8 * 64 * 64);
  cudaMemcpyToSymbol(g_potrf_trace, &tr, sizeof(tr));
  const size_t smem = potrf_coop_smem();
  cudaFuncSetAttribute(k_potrf_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(A, h.data(), 8 * b * b, cudaMemcpyHostToDevice);
    cudaMemset(fail, 0xff, 4);
    cudaMemset(tr, 0, 8 * 64 * 64);
    int bb = b, bk = b, k = 0;
    void* args[] = {&A, &bb, &bk, &Linv, &dinv, &fail, &k, &bar};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((void*)k_potrf_coop, 32, 128, args, smem, 0);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> t(64 * 64);
    cudaMemcpy(t.data(), tr, 8 * 64 * 64, cudaMemcpyDeviceToHost);
    int f;
    cudaMemcpy(&f, fail, 4, cudaMemcpyDeviceToHost);
    printf("rep %d: %.1f us (%s, fail %d)\n", rep, ms * 1e3, cudaGetErrorString(err), f);
    if (rep == 2) {
      unsigned long long t0 = ~0ull;
      for (int c = 0; c < 32; ++c)
        if (t[c * 64] && t[c * 64] < t0) t0 = t[c * 64];
      for (int slot = 0; slot < 48; ++slot) {
        unsigned long long mn = ~0ull, mx = 0, c0 = t[slot];
        for (int c = 0; c < 32; ++c) {
          unsigned long long v = t[c * 64 + slot];
          if (!v) continue;
          mn = v < mn ? v : mn;
          mx = v > mx ? v : mx;
        }
        if (mx) printf("slot %2d: cta0 %8.2f  min %8.2f  max %8.2f us\n", slot, (c0 - t0) / 1e3, (mn - t0) / 1e3,
                       (mx - t0) / 1e3);
      }
    }
  }
  return 0;
}
