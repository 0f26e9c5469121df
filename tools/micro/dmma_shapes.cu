// DMMA shape throughput on the B200 (development aid): m8n8k4 vs the sm_90+
// m16n8k{4,8,16} f64 shapes, 8 independent accumulators per warp.
#include <cstdio>
template <int SHAPE>
__global__ void k_dmma(double* out, int iters) {
  double acc[8][4] = {};
  double a[8], b[4];
  for (int t = 0; t < 8; ++t) a[t] = (threadIdx.x + t) * 1e-3;
  for (int t = 0; t < 4; ++t) b[t] = 1.0 - t * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if constexpr (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(a[0]), "d"(b[0]));
      else if constexpr (SHAPE == 1)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      else if constexpr (SHAPE == 2)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(acc[t][0]), "+d"(acc[t][1]), "+d"(acc[t][2]), "+d"(acc[t][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int t = 0; t < 8; ++t) s += acc[t][0] + acc[t][1] + acc[t][2] + acc[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int SHAPE>
void run(const char* name, double flop_per, int sms, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int wpsm : {4, 8, 16}) {
    const int grid = sms, block = 32 * wpsm, iters = 2048;
    k_dmma<SHAPE><<<grid, block>>>(d, 8);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k_dmma<SHAPE><<<grid, block>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = double(grid) * wpsm * iters * 8 * flop_per;
    printf("%-10s warps/SM %2d: %.2f TFLOP/s\n", name, wpsm, fl / ms / 1e9);
  }
}
int main() {
  double* d;
  cudaMalloc(&d, 1 << 26);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("m8n8k4", 2.0 * 8 * 8 * 4, sms, d);
  run<1>("m16n8k4", 2.0 * 16 * 8 * 4, sms, d);
  run<2>("m16n8k8", 2.0 * 16 * 8 * 8, sms, d);
  run<3>("m16n8k16", 2.0 * 16 * 8 * 16, sms, d);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
