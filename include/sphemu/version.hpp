// sphemu/version.hpp — drop-in for proj/include/sphemu/version.hpp:1-5.
#pragma once

namespace sphemu {
inline constexpr const char* kVersion = "0.1.0";
}
