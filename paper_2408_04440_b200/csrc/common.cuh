// common.cuh — shared helpers for the sphemu B200 kernels: status/error
// plumbing for the C-ABI, launch accounting, and the storage-precision
// conversions of proj/include/sphemu/half.hpp:13-85 expressed with sm_100a
// conversion instructions.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/sphemu_gpu.h"

namespace sphemu_gpu {

// ---- errors ---------------------------------------------------------------
struct Error : std::runtime_error {
  int code;
  int tile = -1;
  Error(int c, const std::string& m, int t = -1) : std::runtime_error(m), code(c), tile(t) {}
};

void set_last_error(const std::string& msg);
void note_launch(int64_t n = 1);
int64_t launch_count();

#define SPH_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t err__ = (call);                                                           \
    if (err__ != cudaSuccess)                                                             \
      throw ::sphemu_gpu::Error(SPHEMU_ERR_CUDA, std::string(#call) + ": " +              \
                                                     cudaGetErrorString(err__));          \
  } while (0)

// SPHEMU_SYNC_CHECK=1 (debugging): every launch is followed by a device
// synchronize, so an asynchronous fault is reported at the kernel that raised it.
bool sync_check();
// Diagnostic modes (SPHEMU_TC_DBG / SPHEMU_OZ_DBG: skip the MMAs or the
// epilogue for timing experiments) exist only in a diagnostics build
// (make DIAG=1); production kernels compile them out.
#ifdef SPHEMU_DIAG
#define SPH_DBG(args) ((args).dbg)
#define SPH_DBG_ENV(name) ([] { const char* e__ = std::getenv(name); return e__ ? std::atoi(e__) : 0; }())
#else
#define SPH_DBG(args) 0
#define SPH_DBG_ENV(name) 0
#endif

#define SPH_LAUNCH_CHECK()                                                                 \
  do {                                                                                     \
    ::sphemu_gpu::note_launch();                                                           \
    cudaError_t err__ = cudaGetLastError();                                                \
    if (err__ == cudaSuccess && ::sphemu_gpu::sync_check()) err__ = cudaDeviceSynchronize(); \
    if (err__ != cudaSuccess)                                                              \
      throw ::sphemu_gpu::Error(SPHEMU_ERR_CUDA, std::string("kernel launch (") + __FILE__ + \
                                ":" + std::to_string(__LINE__) + "): " + cudaGetErrorString(err__)); \
  } while (0)

// Runs f and converts exceptions to C-ABI status codes.
template <class F>
int guard(F&& f) {
  try {
    f();
    return SPHEMU_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return SPHEMU_ERR_INVALID_ARG;
  } catch (const std::bad_alloc& e) {
    set_last_error("out of memory");
    return SPHEMU_ERR_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SPHEMU_ERR_RUNTIME;
  }
}

// ---- device memory RAII ----------------------------------------------------
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    if (count == 0) return;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      throw Error(SPHEMU_ERR_OOM, "cudaMalloc of " + std::to_string(count * sizeof(T)) +
                                      " bytes failed: " + cudaGetErrorString(e));
    }
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
};

// ---- storage precisions -----------------------------------------------------
// Storage classes of the tiles. kHalf is IEEE binary16 (reference); kBf16 is
// the bfloat16 extension that stands in for kHalf when hp_format == BF16.
enum StorePrec : int { kDP = 0, kSP = 1, kHP = 2, kBF = 3 };

__host__ __device__ inline int prec_bytes(int p) { return p == kDP ? 8 : (p == kSP ? 4 : 2); }

// half.hpp:80-82: double -> float (RNE) -> binary16 (RNE), values rounding
// past 65504 (and +-inf) saturate to +-65504 and are counted; NaN stays NaN.
__device__ __forceinline__ __half to_half_sat(double v, unsigned& sat) {
  float f = __double2float_rn(v);
  __half h = __float2half_rn(f);
  if (__hisinf(h)) {
    ++sat;
    h = __ushort_as_half(f < 0.f ? (unsigned short)0xfbffu : (unsigned short)0x7bffu);
  }
  return h;
}

__device__ __forceinline__ __nv_bfloat16 to_bf16_sat(double v, unsigned& sat) {
  float f = __double2float_rn(v);
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  if (__hisinf(h)) {
    ++sat;
    h = __ushort_as_bfloat16(f < 0.f ? (unsigned short)0xff7fu : (unsigned short)0x7f7fu);
  }
  return h;
}

// Loads one stored element as double.
__device__ __forceinline__ double load_elem(const void* base, int prec, size_t idx) {
  switch (prec) {
    case kDP: return static_cast<const double*>(base)[idx];
    case kSP: return (double)static_cast<const float*>(base)[idx];
    case kHP: return (double)__half2float(static_cast<const __half*>(base)[idx]);
    default: return (double)__bfloat162float(static_cast<const __nv_bfloat16*>(base)[idx]);
  }
}

// Stores v through the storage precision (quantize_tile, mpchol.cpp:207-225).
__device__ __forceinline__ void store_elem(void* base, int prec, size_t idx, double v,
                                           unsigned& sat) {
  switch (prec) {
    case kDP: static_cast<double*>(base)[idx] = v; break;
    case kSP: static_cast<float*>(base)[idx] = __double2float_rn(v); break;
    case kHP: static_cast<__half*>(base)[idx] = to_half_sat(v, sat); break;
    default: static_cast<__nv_bfloat16*>(base)[idx] = to_bf16_sat(v, sat); break;
  }
}

// The value the storage precision holds for v (for fp64-side mirrors).
__device__ __forceinline__ double quantize_value(double v, int prec, unsigned& sat) {
  switch (prec) {
    case kDP: return v;
    case kSP: return (double)__double2float_rn(v);
    case kHP: return (double)__half2float(to_half_sat(v, sat));
    default: return (double)__bfloat162float(to_bf16_sat(v, sat));
  }
}

__device__ __forceinline__ unsigned warp_sum_u32(unsigned v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

int num_sms();

// Grow-only device scratch reused across calls, one set of slots per (host
// thread, device) (the per-call buffers of the trend / fit_var entry points,
// which synchronize before returning). The buffers live in a process-wide,
// mutex-guarded registry so sphemu_gpu_release_cache() frees them (also those
// of threads that have exited); callers must not run entry points
// concurrently with that release.
void* scratch_bytes(int slot, size_t bytes);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the opt-in is per device context, so a process driving several GPUs needs it
// on each.
void smem_optin(const void* kernel, int bytes);
void scratch_release_all();
template <class T>
T* scratch(int slot, size_t count) {
  return static_cast<T*>(scratch_bytes(slot, count * sizeof(T)));
}

// TrendModel records + ForcingTrajectory for emulate's trend-model overload
// (trend.cu mean_table_device; trend.hpp:24-59).
struct TrendArgs {
  const double* records;
  int harmonics;
  int period;
  const double* fx;
  int64_t nx;
  const double* fh;
  int64_t nh;
  int64_t t_start;
};
void mean_table_device(const double* records, int64_t points, int harmonics, int period, const double* fx,
                       int64_t nx, const double* fh, int64_t nh, int t_len, int64_t t_start, double* d_table,
                       double* d_sigma, cudaStream_t stream, DevBuf<double>& d_rec, DevBuf<double>& d_rp);

}  // namespace sphemu_gpu
