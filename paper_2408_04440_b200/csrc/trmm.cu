// trmm.cu — Xi += H L^T over the tiled factor (see trmm.cuh): the
// emulation generator's xi = V eta (stochastic.cpp:236-254) on B200 tensor
// cores, with V never leaving its tiles.
//
// Tensor-core kernel (SP / HP classes): persistent, warp-specialized like the
// Cholesky update (tc_gemm.cu): warp 0 issues TMA (A = 128 rows of tile (i, j),
// B = 256 snapshot rows of eta's split, 64 K per stage), warp 1 issues
// tcgen05.mma (one lane), warp 2 owns 512 TMEM columns (two 128 x 256 fp32
// accumulators), warps 4-11 drain an accumulator every `flush` tiles into the
// FP64 Xi (two warps per TMEM lane quarter, 128 columns each; for a fixed
// snapshot the 32 lanes of a warp touch 32 consecutive coefficients).
#include <algorithm>

#include "trmm.cuh"  // chol_kernels.cuh -> common.cuh (cuda_fp16 / cuda_bf16) first
#include "tcgen05.cuh"

namespace sphemu_gpu {

constexpr int TR_BM = 128, TR_BN = 256, TR_BK = 64;  // 64 16-bit K = one 128-byte swizzle row

template <int OPK>
struct TrLayout {
  static constexpr int kA = TR_BM * 128;  // one A box (16 KB)
  static constexpr int kB = TR_BN * 128;  // one eta box (32 KB)
  static constexpr int kNA = OPK == TR_F16X3 ? 2 : 1;
  static constexpr int kStage = kNA * kA + 2 * kB;
  static constexpr int kStages = (232448 - 2048) / kStage;
  static constexpr int kSmem = kStages * kStage + 1024 /*align*/ + 1024 /*barriers*/;
  static constexpr int kEpi = 8;
  static constexpr int kThreads = 32 * (4 + kEpi);
  static_assert(kStages >= 2, "two stages at least");
};

template <int OPK>
__global__ void __launch_bounds__(TrLayout<OPK>::kThreads, 1)
    k_tc_trmm(const __grid_constant__ CUtensorMap mA_hi, const __grid_constant__ CUtensorMap mA_lo,
              const __grid_constant__ CUtensorMap mH_hi, const __grid_constant__ CUtensorMap mH_lo,
              const TrmmArgs args) {
  using Lay = TrLayout<OPK>;
  constexpr int NS = Lay::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * Lay::kStage);
  uint64_t* empty = full + NS;
  uint64_t* tfull = empty + NS;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], Lay::kEpi);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch(&mA_hi);
    tma_prefetch(&mH_hi);
    tma_prefetch(&mH_lo);
    if (OPK == TR_F16X3) tma_prefetch(&mA_lo);
  }
  if (warp == 2) tmem_alloc(tmem_holder, 2 * TR_BN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int kblocks = args.b / TR_BK;
  auto item_at = [&](int64_t n) -> int64_t {
    const int64_t w = blockIdx.x + n * gridDim.x;
    return w < args.n_items ? w : -1;
  };

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // items run snapshot-block-major: the eta block (256 rows of the
      // splits) is re-read by every tile row and stays in L2; each factor
      // tile streams through once per snapshot block.
      const uint64_t keep = l2_evict_last(), stream = l2_evict_first();
      for (int64_t n = 0;; ++n) {
        const int64_t w = item_at(n);
        if (w < 0) break;
        const int4 it = args.items[w];
        const int e0 = args.row_ptr[it.x], e1 = args.row_ptr[it.x + 1];
        for (int e = e0; e < e1; ++e) {
          const int2 en = args.ent[e];
          const int arow = en.y + it.y, hcol = en.x * args.b;
          for (int kb = 0; kb < kblocks; ++kb) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = smem + stage * Lay::kStage;
            mbar_arrive_expect_tx(&full[stage], Lay::kStage);
            const int kx = kb * TR_BK;
            tma_load_2d_hint(&mA_hi, &full[stage], st, kx, arow, stream);
            if (OPK == TR_F16X3) tma_load_2d_hint(&mA_lo, &full[stage], st + Lay::kA, kx, arow, stream);
            tma_load_2d_hint(&mH_hi, &full[stage], st + Lay::kNA * Lay::kA, hcol + kx, it.z, keep);
            tma_load_2d_hint(&mH_lo, &full[stage], st + Lay::kNA * Lay::kA + Lay::kB, hcol + kx, it.z, keep);
            if (++stage == NS) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer =====
    constexpr uint32_t idesc = umma_idesc(OPK == TR_BF16 ? 1 : 0, TR_BM, TR_BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t n = 0;; ++n) {
      const int64_t w = item_at(n);
      if (w < 0) break;
      const int4 it = args.items[w];
      const int cnt = args.row_ptr[it.x + 1] - args.row_ptr[it.x];
      for (int t = 0; t < cnt; ++t) {
        const bool first = (t % args.flush) == 0;
        const bool last = (t % args.flush) == args.flush - 1 || t == cnt - 1;
        if (first) {
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          tc_fence_after();
        }
        const uint32_t d = tmem_base + acc * TR_BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            uint8_t* st = smem + stage * Lay::kStage;
            const uint64_t a_hi = umma_desc_sw128(st);
            const uint64_t h_hi = umma_desc_sw128(st + Lay::kNA * Lay::kA);
            const uint64_t h_lo = umma_desc_sw128(st + Lay::kNA * Lay::kA + Lay::kB);
#pragma unroll
            for (int kk = 0; kk < TR_BK / 16; ++kk) {
              const uint64_t koff = (kk * 16 * 2) >> 4;
              const uint32_t accum = (first && kb == 0 && kk == 0) ? 0u : 1u;
              if constexpr (OPK == TR_F16X3) {
                const uint64_t a_lo = umma_desc_sw128(st + Lay::kA);
                umma_f16(d, a_lo + koff, h_hi + koff, idesc, accum);
                umma_f16(d, a_hi + koff, h_lo + koff, idesc, 1u);
                umma_f16(d, a_hi + koff, h_hi + koff, idesc, 1u);
              } else {
                umma_f16(d, a_hi + koff, h_lo + koff, idesc, accum);
                umma_f16(d, a_hi + koff, h_hi + koff, idesc, 1u);
              }
            }
            umma_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == NS) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (last) {
          if (lane == 0) umma_commit(&tfull[acc]);
          __syncwarp();
          if (++acc == 2) {
            acc = 0;
            acc_phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ===== epilogue: TMEM partial sums -> FP64 Xi =====
    const int q = warp & 3, grp = (warp - 4) >> 2;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t n = 0;; ++n) {
      const int64_t w = item_at(n);
      if (w < 0) break;
      const int4 it = args.items[w];
      const int cnt = args.row_ptr[it.x + 1] - args.row_ptr[it.x];
      const int nfl = (cnt + args.flush - 1) / args.flush;
      const int r = it.y + q * 32 + lane;
      const int64_t g = static_cast<int64_t>(it.x) * args.lb + r;
      const bool valid = r < args.lb && g < args.n;
      double scale = 1.0;
      if (args.rowexp && valid) scale = ldexp(1.0, -args.rowexp[g]);
      for (int f = 0; f < nfl; ++f) {
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
#pragma unroll 1
        for (int c0 = 0; c0 < TR_BN / 2; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * TR_BN + grp * (TR_BN / 2) + c0, v);
          const int64_t col0 = static_cast<int64_t>(it.z) + grp * (TR_BN / 2) + c0;
          if (valid) {
            double old[32];
#pragma unroll
            for (int t = 0; t < 32; ++t)
              old[t] = (col0 + t < args.S) ? args.xi[(col0 + t) * args.n + g] : 0.0;
#pragma unroll
            for (int t = 0; t < 32; ++t)
              if (col0 + t < args.S)
                args.xi[(col0 + t) * args.n + g] = old[t] + scale * static_cast<double>(__uint_as_float(v[t]));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  }
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem_base, 2 * TR_BN);
}

template <int OPK>
static void launch_tr(const CUtensorMap& a_hi, const CUtensorMap& a_lo, const CUtensorMap& h_hi,
                      const CUtensorMap& h_lo, const TrmmArgs& args, cudaStream_t s) {
  using Lay = TrLayout<OPK>;
  auto kern = k_tc_trmm<OPK>;
  smem_optin(reinterpret_cast<const void*>(kern), Lay::kSmem);
  const int grid = static_cast<int>(std::min<int64_t>(args.n_items, num_sms()));
  kern<<<grid, Lay::kThreads, Lay::kSmem, s>>>(a_hi, a_lo, h_hi, h_lo, args);
  SPH_LAUNCH_CHECK();
}

void trmm_tc_launch(int opk, const CUtensorMap& a_hi, const CUtensorMap& a_lo, const CUtensorMap& h_hi,
                    const CUtensorMap& h_lo, const TrmmArgs& args, cudaStream_t s) {
  if (args.n_items <= 0) return;
  switch (opk) {
    case TR_F16: launch_tr<TR_F16>(a_hi, a_lo, h_hi, h_lo, args, s); break;
    case TR_BF16: launch_tr<TR_BF16>(a_hi, a_lo, h_hi, h_lo, args, s); break;
    default: launch_tr<TR_F16X3>(a_hi, a_lo, h_hi, h_lo, args, s); break;
  }
}

// ---- DP tiles: FP64 DMMA ---------------------------------------------------
// grid: x = row blocks of 64 over the tile, y = snapshot blocks of 128, z = tile.
__global__ void __launch_bounds__(D2_THREADS) k_trmm_dp(TileStore ts, const int2* __restrict__ tiles,
                                                         const double* __restrict__ hp, int64_t ldh, int64_t S,
                                                         double* __restrict__ xi) {
  extern __shared__ __align__(16) uint8_t d2_smem[];
  D2Smem& sm = *reinterpret_cast<D2Smem*>(d2_smem);
  const int2 t = tiles[blockIdx.z];
  const int i = t.x, j = t.y;
  const int r0 = blockIdx.x * D2_BN;
  const int64_t s0 = static_cast<int64_t>(blockIdx.y) * D2_BM;
  const int rows_i = ts.rows(i), kc = ts.rows(j);
  if (r0 >= rows_i) return;
  const double* L = static_cast<const double*>(ts.tile(i, j));
  D2Op A{hp + s0 * ldh + static_cast<int64_t>(j) * ts.b, ldh, static_cast<int>(S - s0 < D2_BM ? S - s0 : D2_BM), kc};
  D2Op B{L + static_cast<int64_t>(r0) * ts.b, ts.b, min(D2_BN, rows_i - r0), kc};
  double acc[4][4][2];
  dgemm2_128x64<D2B::kNT, true>(A, B, kc, sm, acc);
  const int64_t g0 = static_cast<int64_t>(i) * ts.lb + r0;
  d2_for_each(acc, [&](int s, int c, double v0, double v1) {
    if (s0 + s >= S) return;
    double* row = xi + (s0 + s) * ts.n + g0;
    if (r0 + c < rows_i) row[c] += v0;
    if (r0 + c + 1 < rows_i) row[c + 1] += v1;
  });
}

void trmm_dp_launch(const TileStore& ts, const int2* tiles, int64_t n_tiles, const double* hp, int64_t ldh,
                    int64_t S, double* xi, cudaStream_t s) {
  if (n_tiles <= 0 || S <= 0) return;
  smem_optin(reinterpret_cast<const void*>(&k_trmm_dp), static_cast<int>(sizeof(D2Smem)));
  for (int64_t t0 = 0; t0 < n_tiles; t0 += 65535) {
    const dim3 grid(ceil_div(ts.lb, D2_BN), ceil_div(S, D2_BM), static_cast<unsigned>(std::min<int64_t>(65535, n_tiles - t0)));
    k_trmm_dp<<<grid, D2_THREADS, sizeof(D2Smem), s>>>(ts, tiles + t0, hp, ldh, S, xi);
    SPH_LAUNCH_CHECK();
  }
}

// ---- operand preparation ----------------------------------------------------
__global__ void k_trmm_prep_eta(const double* __restrict__ eta, int64_t S, int n, int lb, int b, int nt,
                                double* __restrict__ hp, uint16_t* __restrict__ hhi, uint16_t* __restrict__ hlo,
                                int fmt) {
  const int64_t ldh = static_cast<int64_t>(nt) * b;
  const int64_t total = S * ldh;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = e / ldh;
    const int c = static_cast<int>(e - s * ldh);
    const int j = c / b, cc = c - j * b;
    const int64_t g = static_cast<int64_t>(j) * lb + cc;
    const double x = (cc < lb && g < n) ? eta[s * n + g] : 0.0;
    hp[e] = x;
    const float xf = __double2float_rn(x);
    uint16_t h, l;
    if (fmt == 0) {
      const __half hh = __float2half_rn(xf);
      h = __half_as_ushort(hh);
      l = __half_as_ushort(__float2half_rn(static_cast<float>(x - static_cast<double>(__half2float(hh)))));
    } else {
      const __nv_bfloat16 hh = __float2bfloat16_rn(xf);
      h = __bfloat16_as_ushort(hh);
      l = __bfloat16_as_ushort(
          __float2bfloat16_rn(static_cast<float>(x - static_cast<double>(__bfloat162float(hh)))));
    }
    hhi[e] = h;
    hlo[e] = l;
  }
}

void trmm_prep_eta(const double* eta, int64_t S, int n, int lb, int b, int nt, double* hp, uint16_t* h16_hi,
                   uint16_t* h16_lo, int fmt, cudaStream_t s) {
  k_trmm_prep_eta<<<8 * num_sms(), 256, 0, s>>>(eta, S, n, lb, b, nt, hp, h16_hi, h16_lo, fmt);
  SPH_LAUNCH_CHECK();
}

__global__ void k_trmm_prep_sp(TileStore ts, const int2* __restrict__ tiles, const int* __restrict__ rowexp,
                               uint16_t* __restrict__ hi, uint16_t* __restrict__ lo) {
  const int2 t = tiles[blockIdx.y];
  const float* x = static_cast<const float*>(ts.tile(t.x, t.y));
  const int64_t bb = static_cast<int64_t>(ts.b) * ts.b;
  uint16_t* oh = hi + blockIdx.y * bb;
  uint16_t* ol = lo + blockIdx.y * bb;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < bb;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / ts.b);
    const int R = min(t.x * ts.lb + r, ts.n - 1);
    f16_split(static_cast<double>(x[e]), rowexp[R], oh[e], ol[e]);
  }
}

void trmm_prep_sp(const TileStore& ts, const int2* tiles, int64_t n_tiles, const int* rowexp, uint16_t* hi,
                  uint16_t* lo, cudaStream_t s) {
  for (int64_t t0 = 0; t0 < n_tiles; t0 += 65535) {
    const dim3 grid(std::max(1, ts.b * ts.b / (256 * 16)), static_cast<unsigned>(std::min<int64_t>(65535, n_tiles - t0)));
    k_trmm_prep_sp<<<grid, 256, 0, s>>>(ts, tiles + t0, rowexp, hi + t0 * ts.b * ts.b, lo + t0 * ts.b * ts.b);
    SPH_LAUNCH_CHECK();
  }
}

}  // namespace sphemu_gpu
