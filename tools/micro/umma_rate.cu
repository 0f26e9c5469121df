// Raw tcgen05.mma issue rate per SM (development aid): kind::f16 vs kind::i8
// at M = 128 and N = 64 / 128 / 256, operands resident in shared memory.
#include <cuda.h>
#include <cstdio>
#include <cuda_fp16.h>

#include "../../paper_2408_04440_b200/csrc/tcgen05.cuh"
using namespace sphemu_gpu;

__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int KIND, int N>
__global__ void __launch_bounds__(128, 1) k_rate(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t holder;
  for (int e = threadIdx.x; e < (128 + N) * 128 / 16; e += blockDim.x) reinterpret_cast<uint4*>(sm)[e] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc(&holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t t = holder;
  if (threadIdx.x == 0) {
    const uint64_t a = umma_desc_k<128>(sm), b = umma_desc_k<128>(sm + 128 * 128);
    // i8: c_format S32 (2), a/b signed (1); f16: c_format F32 (1), a/b F16 (0)
    constexpr uint32_t idesc = KIND == 1 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24))
                                         : umma_idesc(0, 128, N);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t koff = (kk * 32) >> 4;  // 32 bytes per MMA-K step (16 fp16 or 32 int8)
        const uint32_t d = t + ((i & 1) ? 256 : 0) % 512;
        if (KIND == 1) umma_i8(d, a + koff, b + koff, idesc, 1u);
        else umma_f16(d, a + koff, b + koff, idesc, 1u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(t, 512);
  if (threadIdx.x == 0 && iters < 0) *sink = 1;
}

template <int KIND, int N>
void run(int sms, int* sink) {
  auto k = k_rate<KIND, N>;
  const int smem = (128 + N) * 128 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  k<<<sms, 128, smem>>>(16, sink);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  k<<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double k_per_mma = KIND == 1 ? 32 : 16;
  const double ops = 2.0 * sms * iters * 4 * 128.0 * N * k_per_mma;
  printf("%s M=128 N=%3d: %.0f T(FL)OP/s  (%.1f clk/MMA at 1.965 GHz)\n", KIND == 1 ? "i8 " : "f16", N, ops / ms / 1e9,
         ms * 1e-3 * 1.965e9 / (iters * 4.0));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* sink;
  cudaMalloc(&sink, 4);
  run<0, 64>(sms, sink);
  run<0, 128>(sms, sink);
  run<0, 256>(sms, sink);
  run<1, 64>(sms, sink);
  run<1, 128>(sms, sink);
  run<1, 256>(sms, sink);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
