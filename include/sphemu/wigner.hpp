// sphemu/wigner.hpp — drop-in for proj/include/sphemu/wigner.hpp:13-63. The
// Wigner recurrence runs on the device (sphemu_gpu_wigner_tables, the same
// tables the SHT plan builds); build_wigner_tables copies them out once and
// the object answers d_half_pi / q from host memory like the reference
// (wigner.cpp:136-175), with the reference's cap check and messages. The
// tables build_plan makes for itself (the device plan has its own copy in
// HBM) are filled on first host access only.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "detail_status.hpp"

namespace sphemu {

class WignerTables {
 public:
  int band_limit() const { return band_limit_; }

  // d^l_{m2,m}(pi/2) (wigner.cpp:136-150); any |m2|, |m| <= l < band_limit.
  double d_half_pi(int l, int m2, int m) const {
    if (l < 0 || l >= band_limit_) throw std::out_of_range("degree outside the table");
    ensure();
    return d_raw(l, m2, m);
  }

  // q(l, m, m2) = sqrt((2l+1)/(4 pi)) d^l_{m2,0} d^l_{m2,m} (wigner.cpp:152-170).
  double q(int l, int m, int m2) const {
    if (l < 0 || l >= band_limit_ || m < 0 || m > l || m2 < 0 || m2 >= band_limit_)
      throw std::out_of_range("q index outside the table");
    if (m2 > l) return 0.0;
    ensure();
    return q_[(static_cast<std::size_t>(l) * (l + 1) / 2 + m) * band_limit_ + m2];
  }

 private:
  // d_half_pi on filled tables (no ensure: build_q runs inside the fill)
  double d_raw(int l, int m2, int m) const {
    if (std::abs(m2) > l || std::abs(m) > l) return 0.0;
    int sign = 1;
    if (m2 < 0) {
      sign *= ((l + m) & 1) ? -1 : 1;
      m2 = -m2;
    }
    if (m < 0) {
      sign *= ((l + m2) & 1) ? -1 : 1;
      m = -m;
    }
    const std::size_t o = d_offset_[static_cast<std::size_t>(m2) * band_limit_ + m];
    return sign * d_[o + l - std::max(m2, m)];
  }

 public:

  std::size_t q_entry_count() const {
    ensure();
    return q_.size();
  }
  std::size_t memory_bytes() const {  // wigner.cpp:172-175
    ensure();
    return d_.size() * sizeof(double) + q_.size() * sizeof(double) + d_offset_.size() * sizeof(std::size_t);
  }
  // Rows whose recurrence drifted past |d| = 1 + 1e-9 and were renormalized.
  int renormalization_warnings() const {
    ensure();
    return renorm_warnings_;
  }
  // The cap the tables were built under (the device plan re-checks it).
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
  friend std::shared_ptr<const WignerTables> detail_lazy_wigner_tables(int, std::size_t);
  friend std::shared_ptr<const WignerTables> read_wigd(const std::string&);
  friend void write_wigd(const std::string&, const WignerTables&);

  void ensure() const {
    std::call_once(*once_, [this] { const_cast<WignerTables*>(this)->fill(); });
  }

  void fill() {
    const std::int64_t L = band_limit_;
    std::int64_t count = 0;
    for (std::int64_t k = 0; k < L; ++k) count += (2 * k + 1) * (L - k);
    std::vector<std::int64_t> off(static_cast<std::size_t>(L * L + 1));
    d_.resize(static_cast<std::size_t>(count));
    detail::check(sphemu_gpu_wigner_tables(band_limit_, cap_, off.data(), d_.data(), count, &renorm_warnings_));
    d_offset_.assign(off.begin(), off.end());
    build_q();
  }

  void build_q() {  // wigner.cpp:152-163
    const int big_l = band_limit_;
    q_.assign(static_cast<std::size_t>(big_l) * big_l * (big_l + 1) / 2, 0.0);
    for (int l = 0; l < big_l; ++l) {
      const double norm = std::sqrt((2.0 * l + 1.0) / (4.0 * 3.14159265358979323846));
      for (int m = 0; m <= l; ++m) {
        const std::size_t row = (static_cast<std::size_t>(l) * (l + 1) / 2 + m) * big_l;
        for (int m2 = 0; m2 <= l; ++m2) q_[row + m2] = norm * d_raw(l, m2, 0) * d_raw(l, m2, m);
      }
    }
  }

  int band_limit_ = 0;
  std::size_t cap_ = std::size_t{2} << 30;
  std::shared_ptr<std::once_flag> once_ = std::make_shared<std::once_flag>();
  int renorm_warnings_ = 0;
  std::vector<double> d_;
  std::vector<std::size_t> d_offset_;  // band_limit^2 + 1 entries
  std::vector<double> q_;
};

inline void check_wigner_cap(int band_limit, std::size_t memory_cap_bytes) {  // wigner.cpp:50-64
  if (band_limit < 1) throw std::invalid_argument("band limit must be positive");
  const std::size_t bytes = WignerTables::estimated_bytes(band_limit);
  if (bytes > memory_cap_bytes)
    throw std::invalid_argument("Wigner tables for band limit " + std::to_string(band_limit) + " need " +
                                std::to_string(bytes) + " bytes, over the cap of " +
                                std::to_string(memory_cap_bytes));
}

// Tables filled on first host access (build_plan's own; the device plan
// builds the same tables in HBM).
inline std::shared_ptr<const WignerTables> detail_lazy_wigner_tables(int band_limit, std::size_t memory_cap_bytes) {
  check_wigner_cap(band_limit, memory_cap_bytes);
  auto t = std::make_shared<WignerTables>();
  t->band_limit_ = band_limit;
  t->cap_ = memory_cap_bytes;
  return t;
}

// build_wigner_tables (wigner.cpp:49-134): the device recurrence, copied out.
inline std::shared_ptr<const WignerTables> build_wigner_tables(int band_limit,
                                                               std::size_t memory_cap_bytes = std::size_t{2} << 30) {
  auto t = detail_lazy_wigner_tables(band_limit, memory_cap_bytes);
  t->ensure();
  return t;
}

// Direct factorial-sum evaluation of d^l_{m2,m}(pi/2) (wigner.cpp:31-47).
inline double wigner_brute_force(int l, int m2, int m) {
  if (l < 0 || std::abs(m2) > l || std::abs(m) > l) return 0.0;
  auto lg = [](int k) { return std::lgamma(static_cast<long double>(k)); };
  const long double pref =
      0.5L * (lg(l + m2 + 1) + lg(l - m2 + 1) + lg(l + m + 1) + lg(l - m + 1)) - l * std::log(2.0L);
  const int s_lo = std::max(0, m - m2), s_hi = std::min(l + m, l - m2);
  long double sum = 0.0L;
  for (int s = s_lo; s <= s_hi; ++s) {
    const long double ln_den = lg(l + m - s + 1) + lg(s + 1) + lg(m2 - m + s + 1) + lg(l - m2 - s + 1);
    sum += (((m2 - m + s) & 1) ? -1 : 1) * std::exp(pref - ln_den);
  }
  return static_cast<double>(sum);
}

// Binary cache (wigner.cpp:177-218): "WIGD", u32 version 1, band_limit,
// renormalization warnings, then the d chains (little-endian); q rebuilt on load.
inline void write_wigd(const std::string& path, const WignerTables& tables) {
  tables.ensure();
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open " + path);
  const std::uint32_t head[3] = {1u, static_cast<std::uint32_t>(tables.band_limit()),
                                 static_cast<std::uint32_t>(tables.renormalization_warnings())};
  f.write("WIGD", 4);
  f.write(reinterpret_cast<const char*>(head), sizeof head);
  f.write(reinterpret_cast<const char*>(tables.d_.data()), static_cast<std::streamsize>(tables.d_.size() * 8));
  if (!f.good()) throw std::runtime_error("write failed for " + path);
}

inline std::shared_ptr<const WignerTables> read_wigd(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open " + path);
  char magic[4];
  std::uint32_t head[3];
  f.read(magic, 4);
  f.read(reinterpret_cast<char*>(head), sizeof head);
  if (!f || std::memcmp(magic, "WIGD", 4) != 0) throw std::runtime_error(path + ": not a WIGD file");
  if (head[0] != 1u) throw std::runtime_error(path + ": unsupported WIGD version");
  const int big_l = static_cast<int>(head[1]);
  if (big_l < 1 || big_l > (1 << 16)) throw std::runtime_error(path + ": implausible band limit");
  auto t = std::make_shared<WignerTables>();
  t->band_limit_ = big_l;
  t->cap_ = ~std::size_t{0};
  t->renorm_warnings_ = static_cast<int>(head[2]);
  t->d_offset_.assign(static_cast<std::size_t>(big_l) * big_l + 1, 0);
  std::size_t off = 0;
  for (int a = 0; a < big_l; ++a)
    for (int b = 0; b < big_l; ++b) {
      t->d_offset_[static_cast<std::size_t>(a) * big_l + b] = off;
      off += static_cast<std::size_t>(big_l - std::max(a, b));
    }
  t->d_offset_.back() = off;
  t->d_.resize(off);
  f.read(reinterpret_cast<char*>(t->d_.data()), static_cast<std::streamsize>(off * 8));
  if (!f || f.peek() != std::char_traits<char>::eof()) throw std::runtime_error(path + ": truncated or trailing bytes");
  t->build_q();
  std::call_once(*t->once_, [] {});  // filled: no device build on access
  return t;
}

// load_or_build_wigner (wigner.cpp:220-235).
inline std::shared_ptr<const WignerTables> load_or_build_wigner(int band_limit, const std::string& cache_path) {
  if (!cache_path.empty() && std::filesystem::exists(cache_path)) {
    try {
      auto t = read_wigd(cache_path);
      if (t->band_limit() == band_limit) return t;
    } catch (const std::exception&) {
      // fall through to a fresh build
    }
  }
  auto t = build_wigner_tables(band_limit);
  if (!cache_path.empty()) write_wigd(cache_path, *t);
  return t;
}

}  // namespace sphemu
