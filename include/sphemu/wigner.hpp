// sphemu/wigner.hpp — drop-in for proj/include/sphemu/wigner.hpp:13-49. The
// device plan (sphemu_gpu_sht_create) runs the Wigner recurrence itself, so
// this object carries the band limit and the memory cap the plan is built
// under (cap check and message as wigner.cpp:50-64); d_half_pi
// (wigner.cpp:136-150) reads the device-built tables through
// sphemu_gpu_wigner_d_half_pi, one table build per call (a lookup for tests
// and diagnostics, not a hot path).
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>

#include "detail_status.hpp"

namespace sphemu {

class WignerTables {
 public:
  int band_limit() const { return band_limit_; }
  double d_half_pi(int l, int m2, int m) const {
    if (l < 0 || l >= band_limit_) throw std::out_of_range("degree outside the table");
    double v = 0.0;
    detail::check(sphemu_gpu_wigner_d_half_pi(band_limit_, cap_, 1, &l, &m2, &m, &v, nullptr));
    return v;
  }
  int renorm_warnings() const {
    int r = 0, l = 0;
    double v = 0.0;
    detail::check(sphemu_gpu_wigner_d_half_pi(band_limit_, cap_, 1, &l, &l, &l, &v, &r));
    return r;
  }
  std::size_t memory_cap_bytes() const { return cap_; }
  // d chains + q rows + offsets, as wigner.cpp:54-60 sizes them.
  static std::size_t estimated_bytes(int band_limit) {
    const std::int64_t L = band_limit;
    std::int64_t d = 0;
    for (std::int64_t k = 0; k < L; ++k) d += (2 * k + 1) * (L - k);
    return static_cast<std::size_t>((d + L * L * (L + 1) / 2 + L * L + 1) * 8);
  }

 private:
  friend std::shared_ptr<const WignerTables> build_wigner_tables(int, std::size_t);
  int band_limit_ = 0;
  std::size_t cap_ = 0;
};

inline std::shared_ptr<const WignerTables> build_wigner_tables(int band_limit,
                                                               std::size_t memory_cap_bytes = std::size_t{2} << 30) {
  if (band_limit < 1) throw std::invalid_argument("band limit must be positive");
  const std::size_t bytes = WignerTables::estimated_bytes(band_limit);
  if (bytes > memory_cap_bytes)
    throw std::invalid_argument("Wigner tables for band limit " + std::to_string(band_limit) + " need " +
                                std::to_string(bytes) + " bytes, over the cap of " +
                                std::to_string(memory_cap_bytes));
  auto t = std::make_shared<WignerTables>();
  t->band_limit_ = band_limit;
  t->cap_ = memory_cap_bytes;
  return t;
}

}  // namespace sphemu
