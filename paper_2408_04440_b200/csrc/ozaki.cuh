// ozaki.cuh — the DP-class trailing update (mpchol.cpp:300-314 on FP64
// tiles, C -= P_i P_j^T) on the INT8 tensor cores: an Ozaki-scheme product
// with exact integer accumulation instead of FP64 DMMA.
//
// Every panel row g is written as a 56-bit fixed-point number relative to
// 2^mu_g, mu_g = E_g + 1 with sqrt(a_gg) < 2^E_g (|L_gk| <= sqrt(a_gg) for an
// SPD matrix, one bit of headroom), rounded to nearest, and split into eight
// signed base-128 digits s_0..s_7 (int8, sign-magnitude, |s| <= 127):
//     x = 2^mu sum_s s_s 2^{-7(s+1)}  (+ the rounding error, <= 2^{mu-57}).
// The product of rows i and j is then
//     sum_k x_ik y_jk = 2^{mu_i + mu_j} sum_{d} 2^{-7(d+2)} C_d,
//     C_d = sum_{s+t=d} S_s T_t^T  (int32, exact),
// keeping the 36 digit pairs with s + t <= 7: the dropped pairs and the
// rounding are below ~2^{mu_i+mu_j-53} per k, i.e. ~2^-51 sqrt(a_ii a_jj),
// against FP64's 2^-53 |L_i||L_j| (<= 2^-53 sqrt(a_ii a_jj)) for the same
// sum. An SP-class panel value (fp32, 24 bits) within 2^-31 of its row bound
// is represented exactly, so for the dpsp / dpsphp / dphp diagonal tiles
// every product is exact and the only roundings are the FP64 epilogue sum
// and the subtraction. The pure-FP64 variant "dp" keeps DMMA (its factor is
// meant to carry full double accuracy; measured backward error 1.6e-13 on
// INT8 against 7e-16 on DMMA at n = 4 096).
//
// Rate: kind::i8 M = 128, N = 64 runs at 3.05 POPS (tools/micro/umma_rate.cu;
// 4.58 at N >= 128): 36 digit products per FP64 product -> ~85 TFLOP/s
// FP64-equivalent against DMMA's 35.5 (cuBLAS DGEMM on this B200).
#pragma once

#include <cuda.h>

#include "chol_kernels.cuh"

namespace sphemu_gpu {

constexpr int OZ_DIGITS = 8;

// Digit planes of one panel set: per panel row 8 b bytes laid out
// [K/32 chunks][8 digits][32 K], so one 128-byte TMA box row holds digits
// 0-3 (or 4-7) of a 32-wide K chunk.
struct OzSlices {
  DevBuf<uint8_t> s8;
  CUtensorMap m_a{}, m_b{};  // 128-row (A role) and 64-row (B role) boxes
  int64_t rows = 0;
  int b = 0;
  void alloc(int64_t rows_, int b_);
};

// The eight signed base-128 digits of x relative to 2^mu (56-bit fixed
// point, round to nearest, saturated), digit s in byte s: integer shifts only.
__device__ __forceinline__ uint64_t oz_digits(double x, int mu) {
  const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
  const bool neg = bits >> 63;
  int e = static_cast<int>((bits >> 52) & 0x7ff);
  unsigned long long m = bits & ((1ull << 52) - 1);
  if (e) m |= 1ull << 52;
  else e = 1;
  const int sh = e - 1019 - mu;
  unsigned long long N;
  if (sh >= 0) N = (sh > 3 || ((m << sh) >> 56)) ? (1ull << 56) - 1 : (m << sh);
  else if (-sh >= 64) N = 0ull;
  else N = min((m >> -sh) + ((m >> (-sh - 1)) & 1ull), (1ull << 56) - 1);
  uint64_t out = 0;
#pragma unroll
  for (int s = 0; s < OZ_DIGITS; ++s) {
    int d = static_cast<int>((N >> (49 - 7 * s)) & 127);
    d = neg ? -d : d;
    out |= static_cast<uint64_t>(d & 0xff) << (8 * s);
  }
  return out;
}
// Writes the digits of 8 consecutive row elements x[0..8) at columns c0..c0+7
// (c0 % 8 == 0) into a digit row (8 b bytes, [c/32][digit][c%32] layout).
__device__ __forceinline__ void oz_store8(uint8_t* drow, int c0, const double (&x)[8], int mu) {
  uint64_t d[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) d[u] = oz_digits(x[u], mu);
  uint8_t* q = drow + (c0 >> 5) * 256 + (c0 & 31);
#pragma unroll
  for (int s = 0; s < OZ_DIGITS; ++s) {
    uint64_t v = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) v |= ((d[u] >> (8 * s)) & 0xffull) << (8 * u);
    *reinterpret_cast<uint64_t*>(q + s * 32) = v;
  }
}
// 2^mu_g bounds |panel row g| with one bit of headroom: rowexp = 14 - E with
// sqrt(a_gg) < 2^E (k_rowexp), so mu = E + 1.
__device__ __forceinline__ int oz_mu_of(int rowexp) { return 15 - rowexp; }

// Digits of panel rows [row_begin, row_end) of step k (panel row r belongs
// to tile k+1+r/b) from the FP64 mirror p64, or (p64 == nullptr) straight
// from the panel tiles at their storage precision.
void oz_slice(const TileStore& ts, int k, const double* p64, int64_t row_begin, int64_t row_end, const int* rowexp,
              OzSlices& oz, const int* fail, cudaStream_t s);

// Digits of the panel rows of tiles[0..cnt) (tile indices > k+1, device
// array) of step k.
void oz_slice_tiles(const TileStore& ts, int k, const double* p64, const int* tiles, int64_t cnt, const int* rowexp,
                    OzSlices& oz, const int* fail, cudaStream_t s);

// C_ij -= P_i P_j^T (+ P2_i P2_j^T for a merged pair: k2 >= 0, oz2 = step
// k2's digits) on the FP64 tiles of list[0..cnt). counter: dynamic item
// claims (zeroed here); max_ctas: grid cap (0 = all SMs).
void oz_update(const TileStore& ts, int k, const int2* list, int64_t cnt, const OzSlices& oz, int k2,
               const OzSlices* oz2, const int* rowexp, const int* fail, cudaStream_t s, int max_ctas, int* counter);

}  // namespace sphemu_gpu
