// trmm.cuh — the emulation generator's innovation product over the
// device-resident tiled factor: Xi (S x n, row-major FP64) += H L^T, i.e.
// xi_s = V eta_s for every snapshot column s (stochastic.cpp:236-254 with
// V = the tiled mixed-precision Cholesky factor, no dense V anywhere).
//
//   DP tiles : FP64 DMMA (dgemm2), one launch per band offset (deterministic).
//   SP tiles : tcgen05 kind::f16, the tile's fp16 hi/lo split (row-scaled by
//              2^rowexp like the update path) x eta's fp16 hi/lo, 3 MMAs.
//   HP tiles : tcgen05 kind::f16 straight from the stored fp16 / bf16 tile x
//              eta's hi/lo split in the same format, 2 MMAs.
// The tensor-core classes accumulate in TMEM (fp32) over at most `flush`
// tiles of K, then the epilogue adds the partial sum into Xi in FP64, so the
// fp32 accumulation length is bounded independently of n.
#pragma once

#include <cuda.h>

#include <vector>

#include "chol_kernels.cuh"

namespace sphemu_gpu {

enum : int { TR_F16 = 0, TR_BF16 = 1, TR_F16X3 = 2 };

struct TrmmArgs {
  const int* row_ptr;  // per tile row i: entries [row_ptr[i], row_ptr[i + 1])
  const int2* ent;     // (tile column j, first row of tile (i, j) in the A tensor map)
  const int4* items;   // (i, m0, n0, -): 128-row x 256-snapshot output blocks, longest rows first
  int64_t n_items;
  int b, lb, n;        // tile pitch, logical tile size, matrix order
  int64_t S;           // snapshot columns
  double* xi;          // S x n, accumulated in place
  const int* rowexp;   // SP class: per global row, the operand scale exponent (nullptr: unscaled)
  int flush;           // tiles per TMEM accumulation before the FP64 add
};

// One class launch (opk = TR_*): a_hi/a_lo = the A operand maps (tile rows,
// 128-row boxes), h_hi/h_lo = eta's hi/lo maps ([S][nt b] 16-bit, 256-row boxes).
void trmm_tc_launch(int opk, const CUtensorMap& a_hi, const CUtensorMap& a_lo, const CUtensorMap& h_hi,
                    const CUtensorMap& h_lo, const TrmmArgs& args, cudaStream_t s);

// DP tiles (i, j) of one band offset: Xi[s, i lb + r] += sum_c Hp[s, j b + c] L_ij[r, c]
// with Hp = eta in the padded FP64 layout [S][ldh].
void trmm_dp_launch(const TileStore& ts, const int2* tiles, int64_t n_tiles, const double* hp, int64_t ldh,
                    int64_t S, double* xi, cudaStream_t s);

// eta (S x n FP64, row-major) -> padded FP64 [S][nt b] and the hi/lo 16-bit
// splits in fp16 (fmt 0) or bf16 (fmt 1) of the same layout (zero padding).
void trmm_prep_eta(const double* eta, int64_t S, int n, int lb, int b, int nt, double* hp, uint16_t* h16_hi,
                   uint16_t* h16_lo, int fmt, cudaStream_t s);

// SP tiles -> fp16 hi/lo of x 2^rowexp[row] into a side arena (tile e at e b^2).
void trmm_prep_sp(const TileStore& ts, const int2* tiles, int64_t n_tiles, const int* rowexp, uint16_t* hi,
                  uint16_t* lo, cudaStream_t s);

}  // namespace sphemu_gpu
