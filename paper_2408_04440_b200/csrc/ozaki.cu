// ozaki.cu — DP-class trailing update on the INT8 tensor cores (see
// ozaki.cuh for the number format and the error bound).
//
// k_oz_slice: one warp per (panel row, 128 columns); each lane turns four
// FP64 values into 56-bit fixed point with integer shifts (no FP64 pipe
// work) and writes the eight digit bytes of each as 4-byte groups, so the
// warp's stores cover 1 KB contiguously.
//
// k_oz_update: persistent, warp-specialized like the tcgen05 updates of
// tc_gemm.cu — warp 0 claims 128 x 64 output blocks (atomic counter, 4-slot
// ring) and issues TMA (per 32-wide K chunk: digits 0-3 / 4-7 of the 128 A
// rows and of the 64 B rows, 48 KB per stage, 4 stages), warp 1 issues the
// 36 kind::i8 MMAs of each chunk into eight int32 accumulators C_0..C_7
// (64 TMEM columns each, all 512), warps 4-7 (one per TMEM lane quarter,
// a thread per output row) fold the eight diagonals into FP64 and subtract
// the scaled sum from the FP64 tile in place.
#include <algorithm>
#include <cstdlib>

#include "ozaki.cuh"  // chol_kernels.cuh -> common.cuh first
#include "tc_gemm.cuh"
#include "tcgen05.cuh"

namespace sphemu_gpu {

namespace {

constexpr int OZ_BM = 128, OZ_BN = 64;
constexpr int OZ_BOX_A = OZ_BM * 128;                   // 16 KB: 4 digits x 32 K of 128 rows
constexpr int OZ_BOX_B = OZ_BN * 128;                   // 8 KB
constexpr int OZ_STAGE = 2 * OZ_BOX_A + 2 * OZ_BOX_B;   // 48 KB
constexpr int OZ_STAGES = 4;
constexpr int OZ_SMEM = OZ_STAGES * OZ_STAGE + 1024 /*align*/ + 256 /*barriers, ring, TMEM holder*/;
#ifndef OZ_EPI_WARPS
#define OZ_EPI_WARPS 8
#endif
constexpr int OZ_EPI = OZ_EPI_WARPS;  // per TMEM lane quarter: 1 (64 columns) or 2 (32 columns each)
constexpr int OZ_THREADS = 32 * (4 + OZ_EPI);  // warp 0 TMA, 1 MMA, 2 TMEM owner, 3 idle, then the epilogue

// S32 accumulate, signed int8 A and B, K-major, M = 128, N = 64.
constexpr uint32_t kOzIdesc =
    (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(OZ_BN >> 3) << 17) | (static_cast<uint32_t>(OZ_BM >> 4) << 24);

// Executed by the whole (converged) MMA warp: one elected lane issues, so the
// operands stay warp-uniform and the compiler keeps them in uniform
// registers (issued from a lane == 0 branch, every MMA paid ~16 extra
// instructions of per-lane broadcast: N = 64 MMAs are short enough for that
// to throttle the tensor pipe).
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kOzIdesc), "r"(acc));
}
constexpr uint32_t kOzIdesc128 =
    (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(128 >> 3) << 17) | (static_cast<uint32_t>(OZ_BM >> 4) << 24);
__device__ __forceinline__ void umma_i8_n128(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kOzIdesc128), "r"(acc));
}
__device__ __forceinline__ void umma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ int oz_mu(const int* rowexp, int g) { return oz_mu_of(__ldg(rowexp + g)); }
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double(static_cast<long long>(1023 + e) << 52); }

// tiles != nullptr: rows [0, rows) index the panel rows of tiles[0..] (b
// each) instead of the contiguous range starting at row_begin.
__global__ void __launch_bounds__(256) k_oz_slice(TileStore ts, int k, const double* __restrict__ p64, int64_t row_begin,
                                                  int64_t rows, const int* __restrict__ tiles,
                                                  const int* __restrict__ rowexp, uint8_t* __restrict__ s8,
                                                  const int* fail) {
  if (*(volatile const int*)fail >= 0) return;
  const int b = ts.b;
  const int chunks = b / 128;
  const int64_t w = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int64_t v = w / chunks;
  if (v >= rows) return;
  const int64_t r = tiles ? static_cast<int64_t>(tiles[v / b] - k - 1) * b + v % b : row_begin + v;
  const int c0 = static_cast<int>(w % chunks) * 128 + 4 * lane;
  const int tile = k + 1 + static_cast<int>(r / b), rr = static_cast<int>(r % b);
  const int mu = oz_mu(rowexp, min(tile * ts.lb + rr, ts.n - 1));
  double xs[4];
  if (p64) {
    const double2 v01 = __ldcg(reinterpret_cast<const double2*>(p64 + r * b + c0));
    const double2 v23 = __ldcg(reinterpret_cast<const double2*>(p64 + r * b + c0 + 2));
    xs[0] = v01.x, xs[1] = v01.y, xs[2] = v23.x, xs[3] = v23.y;
  } else {
    // straight from the panel tile (i, k) at its storage precision: the
    // rounded panel value the FP64 mirror would hold, at 2-8 bytes instead of 8
    const int prec = ts.tprec(tile, k);
    const char* row = static_cast<const char*>(ts.tile(tile, k)) + static_cast<int64_t>(rr) * b * prec_bytes(prec);
    if (prec == kDP) {
      const double2 v01 = __ldcg(reinterpret_cast<const double2*>(row) + c0 / 2);
      const double2 v23 = __ldcg(reinterpret_cast<const double2*>(row) + c0 / 2 + 1);
      xs[0] = v01.x, xs[1] = v01.y, xs[2] = v23.x, xs[3] = v23.y;
    } else if (prec == kSP) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(row) + c0 / 4);
      xs[0] = v.x, xs[1] = v.y, xs[2] = v.z, xs[3] = v.w;
    } else {
      const uint2 v = __ldcg(reinterpret_cast<const uint2*>(row) + c0 / 4);
      const uint32_t w[2] = {v.x, v.y};
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (prec == kHP) {
          const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[u]));
          xs[2 * u] = f.x, xs[2 * u + 1] = f.y;
        } else {
          xs[2 * u] = __uint_as_float(w[u] << 16), xs[2 * u + 1] = __uint_as_float(w[u] & 0xffff0000u);
        }
      }
    }
  }
  uint32_t dig[OZ_DIGITS];
#pragma unroll
  for (int s = 0; s < OZ_DIGITS; ++s) dig[s] = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint64_t d = oz_digits(xs[u], mu);
#pragma unroll
    for (int s = 0; s < OZ_DIGITS; ++s) dig[s] |= static_cast<uint32_t>((d >> (8 * s)) & 0xff) << (8 * u);
  }
  uint8_t* rowp = s8 + r * (OZ_DIGITS * static_cast<int64_t>(b)) + (c0 >> 5) * 256 + (c0 & 31);
#pragma unroll
  for (int s = 0; s < OZ_DIGITS; ++s) *reinterpret_cast<uint32_t*>(rowp + s * 32) = dig[s];
}

struct OzArgs {
  TileStore ts;
  const int2* list;
  int64_t items;  // list entries x sub-blocks
  int per, subn;  // sub-blocks per tile, 64-wide column blocks per tile
  int k, k2;
  const int* rowexp;
  const int* fail;
  int* counter;   // dynamic claims (nullptr: static striding)
  int dbg;        // SPHEMU_OZ_DBG (timing experiments only): 1 = no epilogue math, 2 = no MMAs either
};

__global__ void __launch_bounds__(OZ_THREADS, 1)
    k_oz_update(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                const __grid_constant__ CUtensorMap mA2, const __grid_constant__ CUtensorMap mB2, const OzArgs args) {
  extern __shared__ __align__(1024) uint8_t oz_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(oz_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OZ_STAGES * OZ_STAGE);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* tfull = empty + OZ_STAGES;
  uint64_t* tempty = tfull + 1;  // [OZ_DIGITS]: accumulator C_d drained
  uint64_t* sfull = tempty + OZ_DIGITS;
  uint64_t* sempty = sfull + 4;
  int* sched = reinterpret_cast<int*>(sempty + 4);
  uint32_t* holder = reinterpret_cast<uint32_t*>(sched + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // An earlier POTRF failure: one read per CTA (a concurrent chain kernel may
  // set the flag between two threads' reads), so the whole CTA leaves together.
  __shared__ int s_fail;
  if (threadIdx.x == 0) s_fail = *(volatile const int*)args.fail;
  __syncthreads();
  if (s_fail >= 0) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    for (int d = 0; d < OZ_DIGITS; ++d) mbar_init(&tempty[d], OZ_EPI);
    for (int s = 0; s < 4; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 1 + OZ_EPI);  // the MMA warp + the epilogue warps
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mA);
    tma_prefetch(&mB);
    if (args.k2 >= 0) {
      tma_prefetch(&mA2);
      tma_prefetch(&mB2);
    }
  }
  if (warp == 2) tmem_alloc(holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  const int b = args.ts.b;
  const int kblocks = b / 32;
  const int halves = args.k2 >= 0 ? 2 : 1;

  auto decode = [&](int64_t w, int& i, int& j, int& r0, int& c0) {
    const int2 ij = args.list[w / args.per];
    const int sub = static_cast<int>(w % args.per);
    i = ij.x;
    j = ij.y;
    r0 = (sub / args.subn) * OZ_BM;
    c0 = (sub % args.subn) * OZ_BN;
  };
  auto ring_take = [&](int64_t n) -> int64_t {
    const int slot = static_cast<int>(n & 3);
    mbar_wait(&sfull[slot], static_cast<uint32_t>((n >> 2) & 1));
    return static_cast<int64_t>(*(volatile int*)&sched[slot]);
  };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t keep = l2_evict_last();  // the panel digits are re-read by every block of the step
      int stage = 0;
      uint32_t phase = 0;
      int64_t snext = blockIdx.x;  // static striding
      auto claim = [&]() -> int64_t {
        for (;;) {
          int64_t w;
          if (args.counter) {
            w = atomicAdd(args.counter, 1);
          } else {
            w = snext;
            snext += gridDim.x;
          }
          if (w >= args.items) return -1;
          int i, j, r0, c0;
          decode(w, i, j, r0, c0);
          if (!(i == j && c0 >= r0 + OZ_BM)) return w;  // blocks strictly above a diagonal tile's diagonal: skipped
        }
      };
      for (int64_t n = 0;; ++n) {
        const int64_t w = claim();
        const int slot = static_cast<int>(n & 3);
        mbar_wait(&sempty[slot], static_cast<uint32_t>(((n >> 2) & 1) ^ 1));
        sched[slot] = static_cast<int>(w);
        mbar_arrive(&sfull[slot]);
        if (w < 0) break;
        int i, j, r0, c0;
        decode(w, i, j, r0, c0);
        for (int kb2 = 0; kb2 < kblocks * halves; ++kb2) {
          const int hf = kb2 >= kblocks ? 1 : 0, kb = kb2 - hf * kblocks;
          const int kk = hf ? args.k2 : args.k;
          const CUtensorMap* ma = hf ? &mA2 : &mA;
          const CUtensorMap* mb = hf ? &mB2 : &mB;
          const int a_row = (i - kk - 1) * b + r0, b_row = (j - kk - 1) * b + c0;
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * OZ_STAGE;
          mbar_arrive_expect_tx(&full[stage], OZ_STAGE);
          const int x = kb * 128;  // 256 digit bytes per 32-wide K chunk, in 16-bit map units
          tma_load_2d_hint(ma, &full[stage], st, x, a_row, keep);
          tma_load_2d_hint(ma, &full[stage], st + OZ_BOX_A, x + 64, a_row, keep);
          tma_load_2d_hint(mb, &full[stage], st + 2 * OZ_BOX_A, x, b_row, keep);
          tma_load_2d_hint(mb, &full[stage], st + 2 * OZ_BOX_A + OZ_BOX_B, x + 64, b_row, keep);
          if (++stage == OZ_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int64_t n = 0;; ++n) {
      const int64_t w = ring_take(n);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[n & 3]);
      if (w < 0) break;
      for (int kb2 = 0; kb2 < kblocks * halves; ++kb2) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (SPH_DBG(args) == 2) {
          if (kb2 == 0)
            for (int d = 0; d < OZ_DIGITS; ++d) mbar_wait(&tempty[d], acc_phase ^ 1);
          umma_commit_elect(&empty[stage]);
        } else {
          uint8_t* st = smem + stage * OZ_STAGE;
          const uint64_t a0 = umma_desc_sw128(st), a1 = umma_desc_sw128(st + OZ_BOX_A);
          const uint64_t b0 = umma_desc_sw128(st + 2 * OZ_BOX_A), b1 = umma_desc_sw128(st + 2 * OZ_BOX_A + OZ_BOX_B);
          // Digit-major order (consecutive MMAs go to different accumulators:
          // N = 64 MMAs are too short to hide a same-accumulator dependency).
          // The first chunk of a block touches C_0, C_1, ..., C_7 first at
          // s = 0, the order the epilogue drains them: each waits for its
          // accumulator just before that MMA, so the previous block's
          // epilogue overlaps these MMAs.
#pragma unroll
          for (int s = 0; s < OZ_DIGITS; ++s) {
            const uint64_t ad = (s < 4 ? a0 : a1) + 2 * (s & 3);  // 32-byte K offset inside the swizzled row
#pragma unroll
            for (int t = 0; t + s < OZ_DIGITS; ++t) {
              if (kb2 == 0 && s == 0) {
                mbar_wait(&tempty[t], acc_phase ^ 1);
                tc_fence_after();
              }
              const uint64_t bd = (t < 4 ? b0 : b1) + 2 * (t & 3);
              umma_i8(tmem + (s + t) * OZ_BN, ad, bd, (kb2 > 0 || s > 0) ? 1u : 0u);
            }
          }
          umma_commit_elect(&empty[stage]);
        }
        if (++stage == OZ_STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      umma_commit_elect(tfull);
      acc_phase ^= 1;
    }
  } else if (warp >= 4) {
    constexpr int NH = 8 / OZ_EPI;      // 32-column halves per warp
    const int q = warp & 3;             // TMEM lane quarter (hardware: warp % 4)
    const int h0 = ((warp - 4) >> 2) * NH;
    const int row = q * 32 + lane;
    uint32_t acc_phase = 0;
    const TileStore& ts = args.ts;
    for (int64_t n = 0;; ++n) {
      int64_t w = -1;
      if (lane == 0) {
        w = ring_take(n);
        mbar_arrive(&sempty[n & 3]);
      }
      w = __shfl_sync(0xffffffffu, static_cast<int>(w), 0);
      if (w < 0) break;
      int i, j, r0, c0;
      decode(w, i, j, r0, c0);
      // the accumulators take a whole block of MMAs: wait politely, the MMA
      // and TMA warps share these warps' schedulers
      while (!mbar_try(tfull, acc_phase)) __nanosleep(128);
      tc_fence_after();
      double v[NH][32];
#pragma unroll
      for (int hh = 0; hh < NH; ++hh)
#pragma unroll
        for (int c = 0; c < 32; ++c) v[hh][c] = 0.0;
      // C_0 2^-14, ..., C_7 2^-63 (the MMA warp's first-touch order); each
      // drained accumulator goes straight back to the MMA warp
#pragma unroll 1
      for (int d = 0; d < OZ_DIGITS; ++d) {
        uint32_t x[NH][32];
        if (!SPH_DBG(args)) {
#pragma unroll
          for (int hh = 0; hh < NH; ++hh)
            tmem_ld32_nowait(tmem + (static_cast<uint32_t>(q * 32) << 16) + d * OZ_BN + (h0 + hh) * 32, x[hh]);
          tmem_wait_ld();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[d]);
        if (!SPH_DBG(args)) {
          const double wgt = pow2(-7 * (d + 2));
#pragma unroll
          for (int hh = 0; hh < NH; ++hh)
#pragma unroll
            for (int c = 0; c < 32; ++c) v[hh][c] = fma(static_cast<double>(static_cast<int>(x[hh][c])), wgt, v[hh][c]);
        }
      }
      if (!SPH_DBG(args)) {
        const double si = pow2(oz_mu(args.rowexp, min(i * ts.lb + r0 + row, ts.n - 1)));
#pragma unroll
        for (int hh = 0; hh < NH; ++hh) {
          const int cb = c0 + (h0 + hh) * 32;
          double2* cp = reinterpret_cast<double2*>(static_cast<double*>(ts.tile(i, j)) + static_cast<int64_t>(r0 + row) * b + cb);
#pragma unroll
          for (int c2 = 0; c2 < 16; ++c2) {
            const int cg = j * ts.lb + cb + 2 * c2;
            const double s0 = si * pow2(oz_mu(args.rowexp, min(cg, ts.n - 1)));
            const double s1 = si * pow2(oz_mu(args.rowexp, min(cg + 1, ts.n - 1)));
            double2 cur = cp[c2];
            cur.x -= v[hh][2 * c2] * s0;
            cur.y -= v[hh][2 * c2 + 1] * s1;
            cp[c2] = cur;
          }
        }
      }
      acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

// Wide form (SPHEMU_OZ_BN=128): 128 x 128 output blocks and N = 128 MMAs
// (4.58 TOPS against 3.05 at N = 64), the eight diagonals in two passes of
// four TMEM accumulators (128 columns each): pass 0 folds C_0..C_3 from
// digits 0-3 only (10 pairs, 32 KB stages), pass 1 C_4..C_7 from all digits
// (26 pairs, 64 KB stages); each pass's epilogue subtracts its partial sum
// from the FP64 tile (two read-modify-writes per block, both exact-order
// FP64). Each accumulator is released as soon as both 32-column halves of
// its rows are in registers.
constexpr int OZW_BN = 128;
constexpr int OZW_BOX = 128 * 128;  // 16 KB: 128 rows x 128 digit bytes
constexpr int OZW_STAGE = 4 * OZW_BOX;
constexpr int OZW_STAGES = 3;
constexpr int OZW_SMEM = OZW_STAGES * OZW_STAGE + 1024 + 256;

__global__ void __launch_bounds__(OZ_THREADS, 1)
    k_oz_update_w(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mA2, const OzArgs args) {
  extern __shared__ __align__(1024) uint8_t ozw_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ozw_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OZW_STAGES * OZW_STAGE);
  uint64_t* empty = full + OZW_STAGES;
  uint64_t* tfull = empty + OZW_STAGES;
  uint64_t* tempty = tfull + 1;  // [4] accumulator slot drained
  uint64_t* sfull = tempty + 4;
  uint64_t* sempty = sfull + 4;
  int* sched = reinterpret_cast<int*>(sempty + 4);
  uint32_t* holder = reinterpret_cast<uint32_t*>(sched + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ int s_fail;
  if (threadIdx.x == 0) s_fail = *(volatile const int*)args.fail;
  __syncthreads();
  if (s_fail >= 0) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZW_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    for (int x = 0; x < 4; ++x) mbar_init(&tempty[x], OZ_EPI);
    for (int s = 0; s < 4; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 1 + OZ_EPI);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mA);
    if (args.k2 >= 0) tma_prefetch(&mA2);
  }
  if (warp == 2) tmem_alloc(holder, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *holder;
  const int b = args.ts.b;
  const int kblocks = b / 32;
  const int halves = args.k2 >= 0 ? 2 : 1;
  auto decode = [&](int64_t w, int& i, int& j, int& r0, int& c0) {
    const int2 ij = args.list[w / args.per];
    const int sub = static_cast<int>(w % args.per);
    i = ij.x;
    j = ij.y;
    r0 = (sub / args.subn) * OZ_BM;
    c0 = (sub % args.subn) * OZW_BN;
  };
  auto ring_take = [&](int64_t n) -> int64_t {
    const int slot = static_cast<int>(n & 3);
    mbar_wait(&sfull[slot], static_cast<uint32_t>((n >> 2) & 1));
    return static_cast<int64_t>(*(volatile int*)&sched[slot]);
  };
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t keep = l2_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int64_t snext = blockIdx.x;
      auto claim = [&]() -> int64_t {
        for (;;) {
          int64_t w;
          if (args.counter) {
            w = atomicAdd(args.counter, 1);
          } else {
            w = snext;
            snext += gridDim.x;
          }
          if (w >= args.items) return -1;
          int i, j, r0, c0;
          decode(w, i, j, r0, c0);
          if (!(i == j && c0 >= r0 + OZ_BM)) return w;
        }
      };
      for (int64_t n = 0;; ++n) {
        const int64_t w = claim();
        const int slot = static_cast<int>(n & 3);
        mbar_wait(&sempty[slot], static_cast<uint32_t>(((n >> 2) & 1) ^ 1));
        sched[slot] = static_cast<int>(w);
        mbar_arrive(&sfull[slot]);
        if (w < 0) break;
        int i, j, r0, c0;
        decode(w, i, j, r0, c0);
        for (int pass = 0; pass < 2; ++pass)
          for (int kb2 = 0; kb2 < kblocks * halves; ++kb2) {
            const int hf = kb2 >= kblocks ? 1 : 0, kb = kb2 - hf * kblocks;
            const int kk = hf ? args.k2 : args.k;
            const CUtensorMap* ma = hf ? &mA2 : &mA;
            const int a_row = (i - kk - 1) * b + r0, b_row = (j - kk - 1) * b + c0;
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = smem + stage * OZW_STAGE;
            mbar_arrive_expect_tx(&full[stage], pass ? OZW_STAGE : 2 * OZW_BOX);
            const int x = kb * 128;
            // layout: A digits 0-3, B digits 0-3, A digits 4-7, B digits 4-7
            tma_load_2d_hint(ma, &full[stage], st, x, a_row, keep);
            tma_load_2d_hint(ma, &full[stage], st + OZW_BOX, x, b_row, keep);
            if (pass) {
              tma_load_2d_hint(ma, &full[stage], st + 2 * OZW_BOX, x + 64, a_row, keep);
              tma_load_2d_hint(ma, &full[stage], st + 3 * OZW_BOX, x + 64, b_row, keep);
            }
            if (++stage == OZW_STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
      }
    }
  } else if (warp == 1) {
    int stage = 0;
    uint32_t phase = 0, pass_phase = 0;
    for (int64_t n = 0;; ++n) {
      const int64_t w = ring_take(n);
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[n & 3]);
      if (w < 0) break;
      for (int pass = 0; pass < 2; ++pass) {
        for (int kb2 = 0; kb2 < kblocks * halves; ++kb2) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          uint8_t* st = smem + stage * OZW_STAGE;
          const uint64_t a0 = umma_desc_sw128(st), b0 = umma_desc_sw128(st + OZW_BOX);
          const uint64_t a1 = umma_desc_sw128(st + 2 * OZW_BOX), b1 = umma_desc_sw128(st + 3 * OZW_BOX);
#pragma unroll
          for (int s = 0; s < OZ_DIGITS; ++s) {
            const uint64_t ad = (s < 4 ? a0 : a1) + 2 * (s & 3);
#pragma unroll
            for (int t = 0; t + s < OZ_DIGITS; ++t) {
              const int d = s + t;
              if ((d >> 2) != pass) continue;
              if (kb2 == 0 && s == 0) {  // first touch of slot d & 3 in this pass
                mbar_wait(&tempty[d & 3], pass_phase ^ 1);
                tc_fence_after();
              }
              const uint64_t bd = (t < 4 ? b0 : b1) + 2 * (t & 3);
              umma_i8_n128(tmem + (d & 3) * OZW_BN, ad, bd, (kb2 > 0 || s > 0) ? 1u : 0u);
            }
          }
          umma_commit_elect(&empty[stage]);
          if (++stage == OZW_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_elect(tfull);
        pass_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // two warps per TMEM lane quarter, 64 columns each, in two 32-column halves
    const int q = warp & 3;
    const int cbase = ((warp - 4) >> 2) * 64;
    const int row = q * 32 + lane;
    uint32_t pass_phase = 0;
    const TileStore& ts = args.ts;
    for (int64_t n = 0;; ++n) {
      int64_t w = -1;
      if (lane == 0) {
        w = ring_take(n);
        mbar_arrive(&sempty[n & 3]);
      }
      w = __shfl_sync(0xffffffffu, static_cast<int>(w), 0);
      if (w < 0) break;
      int i, j, r0, c0;
      decode(w, i, j, r0, c0);
      const double si = pow2(oz_mu(args.rowexp, min(i * ts.lb + r0 + row, ts.n - 1)));
      for (int pass = 0; pass < 2; ++pass) {
        while (!mbar_try(tfull, pass_phase)) __nanosleep(128);
        tc_fence_after();
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          double v[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c] = 0.0;
#pragma unroll 1
          for (int x = 0; x < 4; ++x) {
            uint32_t xv[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + x * OZW_BN + cbase + h * 32, xv);
            if (h == 1) {  // both halves of slot x are read: back to the MMA warp
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty[x]);
            }
            const double wgt = pow2(-7 * (4 * pass + x + 2));
#pragma unroll
            for (int c = 0; c < 32; ++c) v[c] = fma(static_cast<double>(static_cast<int>(xv[c])), wgt, v[c]);
          }
          const int cb = c0 + cbase + h * 32;
          double2* cp = reinterpret_cast<double2*>(static_cast<double*>(ts.tile(i, j)) + static_cast<int64_t>(r0 + row) * b + cb);
#pragma unroll
          for (int c2 = 0; c2 < 16; ++c2) {
            const int cg = j * ts.lb + cb + 2 * c2;
            const double s0 = si * pow2(oz_mu(args.rowexp, min(cg, ts.n - 1)));
            const double s1 = si * pow2(oz_mu(args.rowexp, min(cg + 1, ts.n - 1)));
            double2 cur = cp[c2];
            cur.x -= v[2 * c2] * s0;
            cur.y -= v[2 * c2 + 1] * s1;
            cp[c2] = cur;
          }
        }
        pass_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, 512);
}

}  // namespace

void OzSlices::alloc(int64_t rows_, int b_) {
  rows = rows_;
  b = b_;
  s8.alloc(static_cast<size_t>(rows) * OZ_DIGITS * b);
  // int8 digits viewed as 16-bit map elements: 4 b per row, 128-byte boxes
  m_a = make_map_strided(s8.get(), rows, 4 * static_cast<int64_t>(b), OZ_DIGITS * static_cast<int64_t>(b), 2, OZ_BM);
  m_b = make_map_strided(s8.get(), rows, 4 * static_cast<int64_t>(b), OZ_DIGITS * static_cast<int64_t>(b), 2, OZ_BN);
}

void oz_slice(const TileStore& ts, int k, const double* p64, int64_t row_begin, int64_t row_end, const int* rowexp,
              OzSlices& oz, const int* fail, cudaStream_t s) {
  if (row_end <= row_begin) return;
  const int64_t warps = (row_end - row_begin) * (ts.b / 128);
  k_oz_slice<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, s>>>(ts, k, p64, row_begin, row_end - row_begin,
                                                                     nullptr, rowexp, oz.s8.get(), fail);
  SPH_LAUNCH_CHECK();
}

void oz_slice_tiles(const TileStore& ts, int k, const double* p64, const int* tiles, int64_t cnt, const int* rowexp,
                    OzSlices& oz, const int* fail, cudaStream_t s) {
  if (cnt <= 0) return;
  const int64_t rows = cnt * ts.b;
  const int64_t warps = rows * (ts.b / 128);
  k_oz_slice<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, s>>>(ts, k, p64, 0, rows, tiles, rowexp, oz.s8.get(),
                                                                     fail);
  SPH_LAUNCH_CHECK();
}

void oz_update(const TileStore& ts, int k, const int2* list, int64_t cnt, const OzSlices& oz, int k2,
               const OzSlices* oz2, const int* rowexp, const int* fail, cudaStream_t s, int max_ctas, int* counter) {
  if (cnt <= 0) return;
  OzArgs a{};
  a.ts = ts;
  a.list = list;
  a.subn = ts.b / OZ_BN;
  a.per = (ts.b / OZ_BM) * a.subn;
  a.items = cnt * a.per;
  a.k = k;
  a.k2 = (k2 >= 0 && oz2) ? k2 : -1;
  a.rowexp = rowexp;
  a.fail = fail;
  a.counter = counter;
  static const int dbg = SPH_DBG_ENV("SPHEMU_OZ_DBG");
  a.dbg = dbg;
  static const int bn = [] {
    const char* e = std::getenv("SPHEMU_OZ_BN");
    return e ? std::atoi(e) : 64;
  }();
  const bool wide = bn == 128 && ts.b % 128 == 0 && dbg == 0;
  if (wide) {
    a.subn = ts.b / 128;
    a.per = (ts.b / OZ_BM) * a.subn;
    a.items = cnt * a.per;
  }
  if (counter) SPH_CUDA(cudaMemsetAsync(counter, 0, sizeof(int), s));
  const int cap = max_ctas > 0 ? std::min(max_ctas, num_sms()) : num_sms();
  const int grid = static_cast<int>(std::min<int64_t>(a.items, std::max(1, cap)));
  const OzSlices& o2 = a.k2 >= 0 ? *oz2 : oz;
  if (wide) {
    smem_optin(reinterpret_cast<const void*>(k_oz_update_w), OZW_SMEM);
    k_oz_update_w<<<grid, OZ_THREADS, OZW_SMEM, s>>>(oz.m_a, o2.m_a, a);
  } else {
    smem_optin(reinterpret_cast<const void*>(k_oz_update), OZ_SMEM);
    k_oz_update<<<grid, OZ_THREADS, OZ_SMEM, s>>>(oz.m_a, oz.m_b, o2.m_a, o2.m_b, a);
  }
  SPH_LAUNCH_CHECK();
}

}  // namespace sphemu_gpu
