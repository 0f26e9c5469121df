// sphemu/mpchol.hpp — drop-in for proj/include/sphemu/mpchol.hpp:11-148 on
// the B200 path. The factorization entry points (tiled_cholesky,
// tiled_cholesky_dense, make_spd_test_matrix, assign_precisions) call the
// C-ABI (include/sphemu_gpu.h); the host-side containers and helpers keep the
// reference's semantics so existing call sites and tests compile unchanged.
#pragma once

#include <charconv>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <map>
#include <tuple>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "sphemu/detail_status.hpp"
#include "sphemu_gpu.h"

namespace sphemu {

enum class Precision : std::uint8_t { kDouble = 0, kSingle = 1, kHalf = 2 };
enum class PrecisionVariant : std::uint8_t { kDp = 0, kDpSp = 1, kDpSpHp = 2, kDpHp = 3 };

inline std::string to_string(Precision p) {
  return p == Precision::kDouble ? "dp" : (p == Precision::kSingle ? "sp" : "hp");
}
inline std::string to_string(PrecisionVariant v) {
  static const char* names[] = {"dp", "dpsp", "dpsphp", "dphp"};
  return names[static_cast<int>(v) & 3];
}
inline PrecisionVariant variant_from_string(const std::string& s) {
  static const std::map<std::string, PrecisionVariant> m{{"dp", PrecisionVariant::kDp},
                                                         {"dpsp", PrecisionVariant::kDpSp},
                                                         {"dpsphp", PrecisionVariant::kDpSpHp},
                                                         {"dphp", PrecisionVariant::kDpHp}};
  auto it = m.find(s);
  if (it == m.end()) throw std::invalid_argument("unknown precision variant: " + s);
  return it->second;
}

// MpCholConfig (mpchol.hpp:18-28) with the B200 fields appended; their
// defaults are the library's (FP16 HP storage as in the reference, tensor
// cores, lookahead on).
struct MpCholConfig {
  PrecisionVariant variant = PrecisionVariant::kDp;
  int tile_size = 128;
  int band_width_dp = 1;
  double sp_fraction = 0.05;
  int workers = 1;
  int hp_format = SPHEMU_HP_FP16;
  int compute = SPHEMU_COMPUTE_TENSOR;
  int lookahead = 1;
  int sp_compute = SPHEMU_SP_F16X3;

  void validate() const {
    if (tile_size < 1) throw std::invalid_argument("tile size must be positive");
    if (band_width_dp < 1) throw std::invalid_argument("double-precision band must be at least 1");
    if (sp_fraction < 0.0 || sp_fraction > 1.0) throw std::invalid_argument("sp fraction must lie in [0, 1]");
    if (workers < 1) throw std::invalid_argument("worker count must be positive");
  }
  sphemu_chol_config c_config() const {
    return sphemu_chol_config{static_cast<int>(variant), tile_size, band_width_dp, sp_fraction, workers,
                              hp_format, compute, lookahead, sp_compute};
  }
};

struct PrecisionMap {
  int n_tiles = 0;
  std::vector<Precision> tiles;  // packed i(i+1)/2 + j

  Precision at(int i, int j) const { return tiles[static_cast<std::size_t>(i) * (i + 1) / 2 + j]; }
  std::int64_t count(Precision p) const {
    std::int64_t c = 0;
    for (Precision t : tiles) c += t == p;
    return c;
  }
};

// assign_precisions (mpchol.cpp:67-93), computed by the library.
inline PrecisionMap assign_precisions(int n_tiles, const MpCholConfig& config) {
  config.validate();
  const sphemu_chol_config c = config.c_config();
  std::vector<std::uint8_t> raw(static_cast<std::size_t>(n_tiles) * (n_tiles + 1) / 2);
  detail::check(sphemu_gpu_assign_precisions(n_tiles, &c, raw.data()));
  PrecisionMap m;
  m.n_tiles = n_tiles;
  m.tiles.reserve(raw.size());
  for (std::uint8_t r : raw) m.tiles.push_back(static_cast<Precision>(r));
  return m;
}

// Lower-triangular tiles held as doubles on the host (mpchol.hpp:47-71).
class TiledMatrix {
 public:
  TiledMatrix() = default;
  TiledMatrix(int n, int tile_size) : n_(n), tile_size_(tile_size) {
    if (n < 1 || tile_size < 1) throw std::invalid_argument("matrix and tile sizes must be positive");
    n_tiles_ = (n + tile_size - 1) / tile_size;
    offset_.assign(static_cast<std::size_t>(n_tiles_) * (n_tiles_ + 1) / 2 + 1, 0);
    std::size_t o = 0, t = 0;
    for (int i = 0; i < n_tiles_; ++i)
      for (int j = 0; j <= i; ++j, ++t) {
        offset_[t] = o;
        o += static_cast<std::size_t>(tile_rows(i)) * tile_rows(j);
      }
    offset_[t] = o;
    data_.assign(o, 0.0);
  }
  static TiledMatrix from_dense(std::span<const double> a, int n, int tile_size) {
    if (a.size() != static_cast<std::size_t>(n) * n) throw std::invalid_argument("dense matrix has the wrong size");
    TiledMatrix m(n, tile_size);
    for (int i = 0; i < m.n_tiles_; ++i)
      for (int j = 0; j <= i; ++j) {
        auto t = m.tile(i, j);
        const int rows = m.tile_rows(i), cols = m.tile_rows(j);
        for (int r = 0; r < rows; ++r)
          for (int c = 0; c < cols; ++c)
            t[static_cast<std::size_t>(r) * cols + c] =
                a[static_cast<std::size_t>(i * tile_size + r) * n + j * tile_size + c];
      }
    return m;
  }
  std::vector<double> to_dense_lower() const {
    std::vector<double> out(static_cast<std::size_t>(n_) * n_, 0.0);
    for (int i = 0; i < n_tiles_; ++i)
      for (int j = 0; j <= i; ++j) {
        auto t = tile(i, j);
        const int rows = tile_rows(i), cols = tile_rows(j);
        for (int r = 0; r < rows; ++r)
          for (int c = 0; c < cols; ++c) {
            const int R = i * tile_size_ + r, Cc = j * tile_size_ + c;
            if (Cc <= R) out[static_cast<std::size_t>(R) * n_ + Cc] = t[static_cast<std::size_t>(r) * cols + c];
          }
      }
    return out;
  }
  int n() const { return n_; }
  int tile_size() const { return tile_size_; }
  int n_tiles() const { return n_tiles_; }
  int tile_rows(int i) const { return std::min(tile_size_, n_ - i * tile_size_); }
  std::span<double> tile(int i, int j) {
    const std::size_t t = static_cast<std::size_t>(i) * (i + 1) / 2 + j;
    return {data_.data() + offset_[t], offset_[t + 1] - offset_[t]};
  }
  std::span<const double> tile(int i, int j) const {
    const std::size_t t = static_cast<std::size_t>(i) * (i + 1) / 2 + j;
    return {data_.data() + offset_[t], offset_[t + 1] - offset_[t]};
  }

 private:
  int n_ = 0, tile_size_ = 0, n_tiles_ = 0;
  std::vector<std::size_t> offset_;
  std::vector<double> data_;
};

enum class TaskKind : std::uint8_t { kPotrf = 0, kTrsm = 1, kSyrk = 2, kGemm = 3 };

struct CholTask {
  TaskKind kind;
  int i = 0;
  int j = 0;
  int k = 0;
};

// The reference's CPU task DAG (mpchol.cpp:156-205). The device scheduler
// runs the same right-looking steps as streams/events, so this graph is a
// host-side description kept for callers and tests.
struct TaskGraph {
  std::vector<CholTask> tasks;
  std::vector<std::vector<std::int32_t>> successors;
  std::vector<std::int32_t> indegree;
  std::size_t size() const { return tasks.size(); }
};

inline TaskGraph build_task_graph(int nt) {
  if (nt < 1) throw std::invalid_argument("need at least one tile");
  TaskGraph g;
  std::vector<std::int32_t> potrf(nt), trsm(static_cast<std::size_t>(nt) * nt, -1), syrk(trsm);
  auto id = [&](TaskKind kind, int i, int j, int k) {
    g.tasks.push_back({kind, i, j, k});
    return static_cast<std::int32_t>(g.tasks.size() - 1);
  };
  auto at = [nt](int i, int k) { return static_cast<std::size_t>(i) * nt + k; };
  for (int k = 0; k < nt; ++k) {
    potrf[k] = id(TaskKind::kPotrf, k, k, k);
    for (int i = k + 1; i < nt; ++i) trsm[at(i, k)] = id(TaskKind::kTrsm, i, k, k);
    for (int i = k + 1; i < nt; ++i) syrk[at(i, k)] = id(TaskKind::kSyrk, i, i, k);
  }
  std::map<std::tuple<int, int, int>, std::int32_t> gemm;
  for (int k = 0; k < nt; ++k)
    for (int j = k + 1; j < nt; ++j)
      for (int i = j + 1; i < nt; ++i) gemm[{i, j, k}] = id(TaskKind::kGemm, i, j, k);
  g.successors.assign(g.tasks.size(), {});
  g.indegree.assign(g.tasks.size(), 0);
  auto edge = [&](std::int32_t a, std::int32_t b) {
    g.successors[a].push_back(b);
    ++g.indegree[b];
  };
  for (int k = 0; k < nt; ++k)
    for (int i = k + 1; i < nt; ++i) {
      edge(potrf[k], trsm[at(i, k)]);
      edge(trsm[at(i, k)], syrk[at(i, k)]);
      for (int j = k + 1; j < i; ++j) edge(trsm[at(i, k)], gemm[{i, j, k}]);
      for (int j = i + 1; j < nt; ++j) edge(trsm[at(i, k)], gemm[{j, i, k}]);
    }
  for (int i = 1; i < nt; ++i) {  // per-tile update chains in k order
    for (int k = 0; k + 1 < i; ++k) edge(syrk[at(i, k)], syrk[at(i, k + 1)]);
    edge(syrk[at(i, i - 1)], potrf[i]);
  }
  for (int i = 0; i < nt; ++i)
    for (int j = 1; j < i; ++j) {
      for (int k = 0; k + 1 < j; ++k) edge(gemm[{i, j, k}], gemm[{i, j, k + 1}]);
      edge(gemm[{i, j, j - 1}], trsm[at(i, j)]);
    }
  return g;
}

struct ConversionCounters {
  std::int64_t demotions_sp = 0;
  std::int64_t demotions_hp = 0;
  std::int64_t half_saturations = 0;
};

namespace detail {
// double -> float (RN) -> IEEE binary16 (RN-even), clamped to +-65504 with a
// count when the rounded magnitude would overflow (half.hpp:13-85 semantics).
inline double quantize_half(double x, std::int64_t* sat) {
  const float f = static_cast<float>(x);
  if (std::isnan(f)) return static_cast<double>(f);
  const double a = std::fabs(static_cast<double>(f));
  if (a >= 65520.0) {
    ++*sat;
    return std::signbit(f) ? -65504.0 : 65504.0;
  }
  double q;
  if (a < 0x1p-14) {
    q = std::nearbyint(a * 0x1p24) * 0x1p-24;  // subnormal grid
  } else {
    int e = 0;
    std::frexp(a, &e);                          // a = m 2^e, m in [0.5, 1)
    const double ulp = std::ldexp(1.0, e - 11);  // 11 significant bits
    q = std::nearbyint(a / ulp) * ulp;
  }
  return std::signbit(f) ? -q : q;
}
}  // namespace detail

// quantize_tile (mpchol.cpp:207-225).
inline void quantize_tile(std::span<double> tile, Precision p, ConversionCounters* counters) {
  if (p == Precision::kDouble) return;
  if (p == Precision::kSingle) {
    for (double& v : tile) v = static_cast<double>(static_cast<float>(v));
    if (counters) counters->demotions_sp += static_cast<std::int64_t>(tile.size());
    return;
  }
  std::int64_t sat = 0;
  for (double& v : tile) v = detail::quantize_half(v, &sat);
  if (counters) {
    counters->demotions_hp += static_cast<std::int64_t>(tile.size());
    counters->half_saturations += sat;
  }
}

struct FactorizationStats {
  int n = 0;
  int tile_size = 0;
  int n_tiles = 0;
  int workers = 0;
  PrecisionVariant variant = PrecisionVariant::kDp;
  std::int64_t tasks_potrf = 0, tasks_trsm = 0, tasks_syrk = 0, tasks_gemm = 0;
  std::int64_t tiles_dp = 0, tiles_sp = 0, tiles_hp = 0;
  std::int64_t bytes_dp = 0, bytes_sp = 0, bytes_hp = 0;
  ConversionCounters conversions;
  double wall_seconds = 0.0;
  double device_ms = 0.0;  // B200: factorization time on the device

  std::int64_t total_tasks() const { return tasks_potrf + tasks_trsm + tasks_syrk + tasks_gemm; }

  // mpchol.cpp:437-457: sorted keys, two-space indent, trailing newline.
  std::string to_json() const {
    auto num = [](double v) {
      char buf[64];
      auto r = std::to_chars(buf, buf + sizeof buf, v);
      std::string s(buf, r.ptr);
      if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
      return s;
    };
    auto obj = [](std::initializer_list<std::pair<const char*, std::string>> kv, int ind) {
      std::string pad(static_cast<std::size_t>(ind + 2), ' '), s = "{\n";
      bool first = true;
      for (auto& [k, v] : kv) {
        s += (first ? "" : ",\n") + pad + "\"" + k + "\": " + v;
        first = false;
      }
      return s + "\n" + std::string(static_cast<std::size_t>(ind), ' ') + "}";
    };
    auto I = [](std::int64_t v) { return std::to_string(v); };
    return obj({{"bytes", obj({{"dp", I(bytes_dp)}, {"hp", I(bytes_hp)}, {"sp", I(bytes_sp)},
                               {"total", I(bytes_dp + bytes_sp + bytes_hp)}}, 2)},
                {"conversions", obj({{"half_saturations", I(conversions.half_saturations)},
                                     {"to_hp", I(conversions.demotions_hp)}, {"to_sp", I(conversions.demotions_sp)}},
                                    2)},
                {"n", I(n)},
                {"n_tiles", I(n_tiles)},
                {"tasks", obj({{"gemm", I(tasks_gemm)}, {"potrf", I(tasks_potrf)}, {"syrk", I(tasks_syrk)},
                               {"total", I(total_tasks())}, {"trsm", I(tasks_trsm)}}, 2)},
                {"tile_size", I(tile_size)},
                {"tiles", obj({{"dp", I(tiles_dp)}, {"hp", I(tiles_hp)}, {"sp", I(tiles_sp)}}, 2)},
                {"variant", "\"" + to_string(variant) + "\""},
                {"wall_seconds", num(wall_seconds)},
                {"workers", I(workers)}},
               0) +
           "\n";
  }
};

namespace detail {
inline FactorizationStats from_c(const sphemu_chol_stats& s) {
  FactorizationStats f;
  f.n = s.n;
  f.tile_size = s.tile_size;
  f.n_tiles = s.n_tiles;
  f.workers = s.workers;
  f.variant = static_cast<PrecisionVariant>(s.variant);
  f.tasks_potrf = s.tasks_potrf;
  f.tasks_trsm = s.tasks_trsm;
  f.tasks_syrk = s.tasks_syrk;
  f.tasks_gemm = s.tasks_gemm;
  f.tiles_dp = s.tiles_dp;
  f.tiles_sp = s.tiles_sp;
  f.tiles_hp = s.tiles_hp;
  f.bytes_dp = s.bytes_dp;
  f.bytes_sp = s.bytes_sp;
  f.bytes_hp = s.bytes_hp;
  f.conversions = {s.demotions_sp, s.demotions_hp, s.half_saturations};
  f.wall_seconds = s.wall_seconds;
  f.device_ms = s.device_ms;
  return f;
}
}  // namespace detail

struct DenseCholResult {
  std::vector<double> factor;  // dense lower, exact zeros above the diagonal
  FactorizationStats stats;
};

// tiled_cholesky_dense (mpchol.cpp:412-417) on the device.
inline DenseCholResult tiled_cholesky_dense(std::span<const double> a, int n, const MpCholConfig& config) {
  config.validate();
  if (n < 1 || a.size() != static_cast<std::size_t>(n) * n)
    throw std::invalid_argument("dense matrix has the wrong size");
  const sphemu_chol_config c = config.c_config();
  DenseCholResult r;
  r.factor.resize(static_cast<std::size_t>(n) * n);
  sphemu_chol_stats st{};
  int failed = -1;
  const int rc =
      sphemu_gpu_tiled_cholesky_dense(a.data(), SPHEMU_HOST, n, &c, r.factor.data(), SPHEMU_HOST, &st, &failed);
  detail::check(rc, failed);
  r.stats = detail::from_c(st);
  return r;
}

// tiled_cholesky (mpchol.cpp:351-410): in place on the host tiles, factored on the device.
inline FactorizationStats tiled_cholesky(TiledMatrix& a, const MpCholConfig& config) {
  if (config.tile_size != a.tile_size()) throw std::invalid_argument("tile size does not match the matrix");
  const int n = a.n();
  std::vector<double> dense(static_cast<std::size_t>(n) * n, 0.0);
  for (int i = 0; i < a.n_tiles(); ++i)
    for (int j = 0; j <= i; ++j) {
      auto t = a.tile(i, j);
      const int rows = a.tile_rows(i), cols = a.tile_rows(j);
      for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c)
          dense[static_cast<std::size_t>(i * a.tile_size() + r) * n + j * a.tile_size() + c] =
              t[static_cast<std::size_t>(r) * cols + c];
    }
  DenseCholResult res = tiled_cholesky_dense(dense, n, config);
  for (int i = 0; i < a.n_tiles(); ++i)
    for (int j = 0; j <= i; ++j) {
      auto t = a.tile(i, j);
      const int rows = a.tile_rows(i), cols = a.tile_rows(j);
      for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c)
          t[static_cast<std::size_t>(r) * cols + c] =
              res.factor[static_cast<std::size_t>(i * a.tile_size() + r) * n + j * a.tile_size() + c];
    }
  return res.stats;
}

// make_spd_test_matrix (mpchol.cpp:419-435), generated on the device (bitwise the reference's values).
inline std::vector<double> make_spd_test_matrix(int n, std::uint64_t seed) {
  if (n < 1) throw std::invalid_argument("matrix size must be positive");
  MpCholConfig cfg;
  cfg.tile_size = n < 512 ? n : 512;
  cfg.compute = SPHEMU_COMPUTE_FP64;
  const sphemu_chol_config c = cfg.c_config();
  sphemu_chol_t h = nullptr;
  detail::check(sphemu_gpu_chol_create(n, &c, &h));
  std::vector<double> a(static_cast<std::size_t>(n) * n);
  int rc = sphemu_gpu_chol_generate_spd(h, seed);
  if (rc == SPHEMU_OK) rc = sphemu_gpu_chol_store_dense(h, a.data(), SPHEMU_HOST, n);
  sphemu_gpu_chol_destroy(h);
  detail::check(rc);
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j)
      a[static_cast<std::size_t>(i) * n + j] = a[static_cast<std::size_t>(j) * n + i];
  return a;
}

}  // namespace sphemu
