#!/usr/bin/env bash
# Builds oracle/_ref/libsphemu_ref.so from the reference's OWN sources under
# /root/reference/proj (read in place, never copied): half.hpp, rng.hpp,
# wigner.cpp, grid.cpp, sht.cpp. FFTW (sht.cpp's one external dependency,
# through fft.hpp) is replaced by oracle/ref/fft_shim.cpp. mpchol.cpp and
# stochastic.cpp need Eigen (absent from this image) and are NOT built.
# Flags follow the reference's CMake Release build (-O3 -DNDEBUG, no -march,
# so no FMA contraction).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref="${SPHEMU_REFERENCE:-/root/reference/proj}"
out="$here/../_ref"
if [ ! -d "$ref/src" ]; then
  echo "reference sources not found at $ref; oracle/_ref not rebuilt" >&2
  exit 0
fi
mkdir -p "$out"
g++ -std=c++20 -O3 -DNDEBUG -fPIC -shared -I"$ref/include" \
  "$here/ref_wrap.cpp" "$here/fft_shim.cpp" \
  "$ref/src/wigner.cpp" "$ref/src/grid.cpp" "$ref/src/sht.cpp" \
  -o "$out/libsphemu_ref.so" -lpthread
echo "built $out/libsphemu_ref.so"
