// Standalone timing of the INT8 (Ozaki) DP-class update kernel (development
// aid): synthetic digit planes, a list of FP64 tiles, K = 512 (one step) and
// K = 1024 (merged pair); prints us per launch and the digit-product rate.
// Build: see tools/micro/build_oz_bench.sh (links lib/libsphemu_gpu.so).
#include <cstdio>
#include <vector>

#include "ozaki.cuh"

using namespace sphemu_gpu;

int main(int argc, char** argv) {
  const int b = 512, nt = 34;
  const int ntiles = nt * (nt + 1) / 2;
  std::vector<int64_t> off(ntiles);
  std::vector<uint8_t> prec(ntiles, kDP);
  for (int t = 0; t < ntiles; ++t) off[t] = static_cast<int64_t>(t) * b * b * 8;
  DevBuf<char> arena(static_cast<size_t>(ntiles) * b * b * 8);
  cudaMemset(arena.get(), 0, arena.n);
  DevBuf<int64_t> d_off(ntiles);
  DevBuf<uint8_t> d_prec(ntiles);
  cudaMemcpy(d_off.get(), off.data(), ntiles * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_prec.get(), prec.data(), ntiles, cudaMemcpyHostToDevice);
  TileStore ts{arena.get(), d_off.get(), d_prec.get(), nt * b, b, nt, b};
  DevBuf<int> rowexp(nt * b), fail(1), counter(1);
  std::vector<int> re(nt * b, 14);
  cudaMemcpy(rowexp.get(), re.data(), re.size() * 4, cudaMemcpyHostToDevice);
  int m1 = -1;
  cudaMemcpy(fail.get(), &m1, 4, cudaMemcpyHostToDevice);
  OzSlices oz1, oz2;
  oz1.alloc(static_cast<int64_t>(nt - 1) * b, b);
  oz2.alloc(static_cast<int64_t>(nt - 1) * b, b);
  // random digits in [-127, 127]
  std::vector<uint8_t> h(oz1.s8.n);
  uint32_t x = 12345;
  for (auto& v : h) {
    x = x * 1664525u + 1013904223u;
    v = static_cast<uint8_t>(static_cast<int8_t>(static_cast<int>((x >> 24) % 255) - 127));
  }
  cudaMemcpy(oz1.s8.get(), h.data(), h.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(oz2.s8.get(), h.data(), h.size(), cudaMemcpyHostToDevice);
  // off-diagonal tiles (i, j), 2 <= j < i < nt: rows (i-k-1) b valid for k = 0, 1
  std::vector<int2> lst;
  for (int i = 3; i < nt && lst.size() < 96; ++i)
    for (int j = 2; j < i && lst.size() < 96; ++j) lst.push_back(make_int2(i, j));
  std::vector<int2> diag;
  for (int i = 2; i < nt; ++i) diag.push_back(make_int2(i, i));
  DevBuf<int2> d_lst(lst.size()), d_diag(diag.size());
  cudaMemcpy(d_lst.get(), lst.data(), lst.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d_diag.get(), diag.data(), diag.size() * 8, cudaMemcpyHostToDevice);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, const int2* l, int64_t cnt, int blocks_per_tile, bool merged) {
    for (int w = 0; w < 2; ++w)
      oz_update(ts, 0, l, cnt, oz1, merged ? 1 : -1, merged ? &oz2 : nullptr, rowexp.get(), fail.get(), s, 0,
                counter.get());
    cudaEventRecord(e0, s);
    const int reps = 5;
    for (int r = 0; r < reps; ++r)
      oz_update(ts, 0, l, cnt, oz1, merged ? 1 : -1, merged ? &oz2 : nullptr, rowexp.get(), fail.get(), s, 0,
                counter.get());
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    const double K = merged ? 2.0 * b : b;
    const double items = static_cast<double>(cnt) * blocks_per_tile;
    const double ops = items * 36 * 2.0 * 128 * 64 * K;  // int8 digit-product ops
    const double fp64 = items * 2.0 * 128 * 64 * K;      // FP64-equivalent flops
    printf("%-22s items %6.0f  %8.1f us  %6.1f us/item/CTA  %6.0f TOPS int8  %5.1f TFLOP/s fp64-eq\n", name, items, us,
           us * 148 / items, ops / us / 1e6, fp64 / us / 1e6);
  };
  run("offdiag K=512", d_lst.get(), lst.size(), 32, false);
  run("offdiag K=1024", d_lst.get(), lst.size(), 32, true);
  run("diag K=512", d_diag.get(), diag.size(), 20, false);
  run("diag K=1024", d_diag.get(), diag.size(), 20, true);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
