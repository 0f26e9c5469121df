// FP64 pipe microbenchmarks on the B200: DFMA throughput/latency, DMMA
// throughput, FP32 FFMA throughput for comparison (development aid).
#include <cstdio>
__global__ void k_dfma_tp(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
    a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_ffma_tp(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float m = 0.999999f, c = 1e-7f;
  for (int i = 0; i < iters; ++i) {
    a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
    a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_dfma_lat(double* out, int iters, long long* cyc) {
  double a = threadIdx.x;
  const double m = 0.999999, c = 1e-7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, m, c);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void k_dmma_tp(double* out, int iters) {
  double d[8][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 - a;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(d[t][0]), "+d"(d[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += d[t][0] + d[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* d; float* f; long long* cyc;
  cudaMalloc(&d, 1 << 26); cudaMalloc(&f, 1 << 26); cudaMalloc(&cyc, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  const int grid = sms * 8, block = 256, iters = 4096;
  k_dfma_tp<<<grid, block>>>(d, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); k_dfma_tp<<<grid, block>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("DFMA  : %.2f TFLOP/s\n", 2.0 * 8 * iters * (double)grid * block / (ms * 1e-3) / 1e12);
  cudaEventRecord(e0); k_ffma_tp<<<grid, block>>>(f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("FFMA  : %.2f TFLOP/s\n", 2.0 * 8 * iters * (double)grid * block / (ms * 1e-3) / 1e12);
  cudaEventRecord(e0); k_dmma_tp<<<grid, block>>>(d, iters / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("DMMA  : %.2f TFLOP/s (m8n8k4, 8 independent accumulators per warp)\n",
         2.0 * 256 * 8 * (iters / 4) * (double)grid * (block / 32) / (ms * 1e-3) / 1e12);
  k_dfma_lat<<<1, 32>>>(d, iters, cyc); long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA latency: %.1f cycles\n", (double)c / iters);
  return 0;
}
