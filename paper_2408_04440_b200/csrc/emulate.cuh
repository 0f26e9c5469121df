// emulate.cuh — the emulation generator's driver (stochastic.cpp:217-277),
// shared by the dense-V entry points (emulate.cu) and the tiled-factor entry
// point (chol.cu, sphemu_gpu_emulate_chol): everything after the innovation
// product — RNG, AR(P), inverse SHT, retrend — is the same.
#pragma once

#include <functional>
#include <vector>

#include "common.cuh"

namespace sphemu_gpu {

// Innovation product of one replicate chunk on the given stream. dH holds
// the normals of every rank's chunk replicates (S_all x d, rank q's columns
// at [col_off[q], col_off[q + 1])); dXi receives this rank's columns of
// H V^T ((col_off[rank + 1] - col_off[rank]) x d). One GPU: col_off = {0, S_all}.
using XiFn = std::function<void(const double* dH, int64_t S_all, const std::vector<int64_t>& col_off, double* dXi,
                                cudaStream_t s)>;

struct EmulArgs {
  void* plan;  // sphemu_sht_t
  int n_theta, n_phi, L, d;
  const double* phi;  // order x d (host)
  int order;
  const double* means;  // t_out x points (host; unused with trend)
  const double* sigma;  // points (host; unused with trend)
  const double* v2;     // points (host)
  int t_out;
  uint64_t seed;
  int r_begin, r_len, rng_mode;
  double* out;  // (r_len, t_out, n_theta, n_phi)
  int where_out;
  const TrendArgs* trend;
  int64_t chunk_bytes;  // replicate-chunk buffer budget (0: 8 GiB)
  int world = 1, rank = 0;  // > 1: replicates split in `world` contiguous balanced blocks, this rank's in `out`
};

// Replicates [r_begin, r_begin + r_len) (this rank's block of them), in
// chunks that fit chunk_bytes; every rank runs the same number of chunks.
void emulate_core(const EmulArgs& a, const XiFn& xi);

// This rank's replicate block [lo, hi) of [r_begin, r_begin + r_len).
inline void emul_share(int r_begin, int r_len, int world, int rank, int& lo, int& hi) {
  lo = r_begin + static_cast<int>((static_cast<int64_t>(r_len) * rank) / world);
  hi = r_begin + static_cast<int>((static_cast<int64_t>(r_len) * (rank + 1)) / world);
}
void emulate_core(const EmulArgs& a, const XiFn& xi);

}  // namespace sphemu_gpu
