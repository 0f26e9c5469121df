// ref_mpchol_wrap.cpp — extern "C" entry points over the reference's OWN
// proj/src/mpchol.cpp (compiled in place by oracle/ref/build_ref.sh against
// oracle/ref/eigen_shim and the nlohmann json header shipped with
// cudnn_frontend). Test infrastructure: pins oracle/so_mpchol.c's scheduler,
// precision map, quantization and statistics to the reference's code.
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <string>

#include "sphemu/mpchol.hpp"

using namespace sphemu;

extern "C" {

// 0 ok, 1 not SPD (failed_tile set), -1 invalid config; stats JSON into json (cap bytes)
int ref_tiled_cholesky_dense(const double* a, int n, int variant, int tile, int workers, int band, double sp_frac,
                             double* factor, char* json, int cap, int* failed_tile) {
  try {
    MpCholConfig c;
    c.variant = static_cast<PrecisionVariant>(variant);
    c.tile_size = tile;
    c.workers = workers;
    c.band_width_dp = band;
    c.sp_fraction = sp_frac;
    DenseCholResult r = tiled_cholesky_dense(std::span<const double>(a, static_cast<size_t>(n) * n), n, c);
    std::memcpy(factor, r.factor.data(), r.factor.size() * sizeof(double));
    const std::string j = r.stats.to_json();
    std::strncpy(json, j.c_str(), static_cast<size_t>(cap - 1));
    json[cap - 1] = 0;
    return 0;
  } catch (const NotPositiveDefiniteError& e) {
    if (failed_tile) *failed_tile = e.tile_index();
    std::strncpy(json, e.what(), static_cast<size_t>(cap - 1));
    json[cap - 1] = 0;
    return 1;
  } catch (const std::exception& e) {
    std::strncpy(json, e.what(), static_cast<size_t>(cap - 1));
    json[cap - 1] = 0;
    return -1;
  }
}

int ref_assign_precisions(int nt, int variant, int band, double sp_frac, unsigned char* out) {
  MpCholConfig c;
  c.variant = static_cast<PrecisionVariant>(variant);
  c.band_width_dp = band;
  c.sp_fraction = sp_frac;
  PrecisionMap m = assign_precisions(nt, c);
  for (int i = 0; i < nt; ++i)
    for (int j = 0; j <= i; ++j) out[static_cast<size_t>(i) * (i + 1) / 2 + j] = static_cast<unsigned char>(m.at(i, j));
  return 0;
}

void ref_make_spd(int n, std::uint64_t seed, double* out) {
  auto a = make_spd_test_matrix(n, seed);
  std::memcpy(out, a.data(), a.size() * sizeof(double));
}

}  // extern "C"
