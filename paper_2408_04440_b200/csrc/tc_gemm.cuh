// tc_gemm.cuh — tcgen05 (5th-gen tensor core) tile GEMMs of the Cholesky:
// the SP/HP-class trailing updates (mpchol.cpp:300-314) and the panel TRSM
// expressed as X = B * Linv^T (mpchol.cpp:293-299), with operands staged by
// TMA into 128B-swizzled shared memory and accumulators in TMEM.
//
//   HP class (fp16 / bf16 tiles): kind::f16 (or bf16) operands, FP32 accumulate.
//   SP class (fp32 tiles):        3xTF32 = hi*hi + hi*lo + lo*hi on kind::tf32,
//                                 FP32 accumulate (~2^-21 relative products).
// Operands are the per-step panel mirrors written once by the panel producer
// (sender-side conversion).
#pragma once

#include <cuda.h>

#include <vector>

#include "chol_kernels.cuh"

namespace sphemu_gpu {

// 2-D TMA map of a row-major array: rows x cols elements (2- or 4-byte), row
// pitch row_bytes, box = swizzle_bytes of K x box_rows rows (SWIZZLE_128B / 64B).
CUtensorMap make_map_strided(const void* base, int64_t rows, int64_t cols, int64_t row_bytes, int elem_bytes,
                             int box_rows, int swizzle_bytes = 128);

constexpr int TC_BM = 128;
constexpr int TC_EPI_WARPS = 8;                  // epilogue warps 4 .. 11
constexpr int TC_THREADS = 32 * (4 + TC_EPI_WARPS);

// Tensor-core operand mirrors of the current panel (rows (i-k-1)*b + r).
struct PanelFormats {
  int nt = 0, b = 0, hp_format = 0;
  DevBuf<float> p_hi, p_lo;       // tf32 split of the rounded panel
  DevBuf<uint16_t> p16;           // fp16/bf16 copy of the rounded panel
  DevBuf<float> in_hi, in_lo;     // tf32 split of the panel TRSM input B_i
  DevBuf<float> l_hi, l_lo;       // tf32 split of Linv (b x b)
  // TMA descriptors: A-role (128-row box) and B-role (BN-row box).
  CUtensorMap m_phi_a, m_plo_a, m_phi_b, m_plo_b, m_p16_a, m_p16_b;
  CUtensorMap m_inhi_a, m_inlo_a, m_lhi_b, m_llo_b;
  // FP16x3 panel TRSM operands: fp16 hi/lo of the scaled B_i and Linv, and
  // the per-Linv-row exponents g_j (see k_panel_prep16).
  DevBuf<uint16_t> in16_hi, in16_lo, l16_hi, l16_lo;
  DevBuf<int> lexp;
  CUtensorMap m_in16hi_a, m_in16lo_a, m_l16hi_b, m_l16lo_b;
  // FP16x3 path for the SP class: x * 2^e_row = hi + lo, both fp16.
  bool f16x3 = false;
  // Which mirrors have a consumer: the tf32 split only feeds the 3xTF32 SP
  // update, the 16-bit copy only the HP update; the panel skips the others.
  bool need_tf32 = true, need_p16 = true;
  float* tf32_hi() { return need_tf32 ? p_hi.get() : nullptr; }
  float* tf32_lo() { return need_tf32 ? p_lo.get() : nullptr; }
  uint16_t* half16() { return need_p16 ? p16.get() : nullptr; }
  const int* rowexp = nullptr;
  DevBuf<uint16_t> h_hi, h_lo;
  CUtensorMap m_hhi_a, m_hlo_a, m_hhi_b, m_hlo_b;
  CUtensorMap m_c16{}, m_c32{};  // C operand: the tile arena as 16-bit / fp32 rows (set_arena)
  void set_arena(const void* base, int64_t bytes, int b_);
  int bn = 256;
  bool pair_dyn_sp = false;  // SP-class CTA pairs claim items dynamically (and yield); see tc_update
  uint8_t* s8 = nullptr;     // INT8 DP digit planes of this set, written by the panel epilogue (one GPU)
  bool no_p64 = false;       // the SP/HP panel rows' FP64 mirror has no reader (one GPU, INT8 DP class)
  void alloc(int nt_, int b_, const std::vector<uint8_t>& pmap, int hp_format_, bool f16x3_,
             const int* rowexp_);
};

// Panel TRSM for all i > k: DP-class tiles through FP64 DMMA, SP/HP-class
// tiles (d_lo) through 3xTF32 tcgen05, BF16-class tiles (d_bf) through one
// bf16 operand x Linv's bf16 hi/lo split; writes the rounded P64 mirror, the
// tensor mirrors, and the tile storage.
void tc_panel_trsm(const TileStore& ts, int k, const int2* d_dp, int64_t n_dp, const int2* d_lo,
                   int64_t n_lo, const double* linv, double* p64, PanelFormats& pf, const int* fail,
                   unsigned* sat, cudaStream_t s, int max_ctas = 0, int* counter = nullptr,
                   const int2* d_bf = nullptr, int64_t n_bf = 0);

// Trailing update of the SP (cls 1) or HP (cls 2) output tiles of step k.
// yield (non-null, dynamically scheduled launches only): the CTAs stop
// claiming work items once *yield != 0 (the chain wants the SMs for the
// panel); resume = true continues such a launch from its counter (no reset).
// Statically scheduled launches (CTA pairs) never yield and skip the resume.
// k2 >= 0 (with pf2 = that step's operand mirrors): merged two-step update,
// C -= P_k Q_k^T + P_k2 Q_k2^T in one accumulator (one C round trip, one
// storage rounding for both steps).
void tc_update(const TileStore& ts, int k, int cls, int hp_format, const int2* list, const int* rows, int64_t cnt,
               const double* p64, PanelFormats& pf, const int* fail, unsigned* sat, cudaStream_t s,
               int max_ctas = 0, int* counter = nullptr, const int* yield = nullptr, bool resume = false,
               int k2 = -1, PanelFormats* pf2 = nullptr);

// Host-side inputs of make_spd_test_matrix: d_i = exp(0.6 u_i - 0.3) with the
// reference's GaussianRng uniform stream, pw[k] = std::pow(rho, k) (rho = 0.9:
// the reference generator; rho -> 1: the same D (I + K/4) D family with
// O(1) off-diagonal tiles, K the Kac-Murdock-Szego matrix).
void host_spd_factors(int n, uint64_t seed, double* d, double* pw, double rho = 0.9);

}  // namespace sphemu_gpu
