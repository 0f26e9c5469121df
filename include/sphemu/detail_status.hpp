// sphemu/detail_status.hpp — C-ABI status -> the reference's exception types
// (std::invalid_argument, NotPositiveDefiniteError, std::runtime_error), so
// callers of the C++ headers see exactly what the reference throws.
#pragma once

#include <stdexcept>
#include <string>

#include "sphemu_gpu.h"

namespace sphemu {

// mpchol.hpp:122-130: thrown by tiled_cholesky with the failing diagonal tile.
class NotPositiveDefiniteError : public std::runtime_error {
 public:
  NotPositiveDefiniteError(int tile_index, const std::string& what) : std::runtime_error(what), tile_(tile_index) {}
  int tile_index() const { return tile_; }

 private:
  int tile_ = 0;
};

namespace detail {
inline void check(int rc, int failed_tile = -1) {
  if (rc == SPHEMU_OK) return;
  const std::string msg = sphemu_gpu_last_error();
  if (rc == SPHEMU_ERR_INVALID_ARG) throw std::invalid_argument(msg);
  if (rc == SPHEMU_ERR_NOT_SPD) throw NotPositiveDefiniteError(failed_tile, msg);
  throw std::runtime_error(msg);
}
}  // namespace detail
}  // namespace sphemu
