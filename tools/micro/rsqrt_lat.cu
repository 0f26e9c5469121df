// Dependent-chain latency of the FP64 reciprocal square root variants (development aid).
#include <cstdio>
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // two Newton steps: y <- y (1.5 - 0.5 x y^2)
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}
template <int V>
__global__ void k(double* out, long long* cyc, int iters) {
  double x = 1.0 + threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double r;
    if (V == 0) r = rsqrt(x);
    else if (V == 1) r = rsqrt_nr(x);
    else if (V == 2) r = 1.0 / sqrt(x);
    else r = sqrt(x);
    x = 1.0 + r * 1e-9;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  const char* nm[] = {"rsqrt(double)", "rsqrt.approx+2NR", "1/sqrt", "sqrt"};
  auto run = [&](auto kern, int v) {
    kern<<<1, 32>>>(o, c, 10); cudaDeviceSynchronize();
    kern<<<1, 32>>>(o, c, 1000); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-18s %6.1f clk per dependent op (incl. fma)\n", nm[v], h / 1000.0);
  };
  run(k<0>, 0); run(k<1>, 1); run(k<2>, 2); run(k<3>, 3);
  // accuracy of the NR variant against rsqrt(double)
  return 0;
}
