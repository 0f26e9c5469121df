#!/usr/bin/env bash
# Builds oracle/_ref/libsphemu_ref.so from the reference's OWN sources under
# /root/reference/proj (read in place, never copied): half.hpp, rng.hpp,
# wigner.cpp, grid.cpp, sht.cpp. FFTW (sht.cpp's one external dependency,
# through fft.hpp) is replaced by oracle/ref/fft_shim.cpp. mpchol.cpp is built
# into a second library against oracle/ref/eigen_shim (the few Eigen calls it
# makes, with so_mpchol.c's loop order) and the nlohmann json header that
# ships with cudnn_frontend; stochastic.cpp needs real Eigen and is NOT built.
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
json_dir="$(python3 -c 'import os, sys; import site; [print(os.path.join(p, "include/cudnn_frontend/thirdparty/nlohmann")) for p in site.getsitepackages() if os.path.exists(os.path.join(p, "include/cudnn_frontend/thirdparty/nlohmann/json.hpp"))]' 2>/dev/null | head -1)"
if [ -n "$json_dir" ]; then
  g++ -std=c++20 -O3 -DNDEBUG -fPIC -shared -I"$here/eigen_shim" -I"$ref/include" -I"$json_dir" \
    "$here/ref_mpchol_wrap.cpp" "$ref/src/mpchol.cpp" -o "$out/libsphemu_ref_mpchol.so" -lpthread
  echo "built $out/libsphemu_ref_mpchol.so"
else
  echo "nlohmann json header not found; oracle/_ref/libsphemu_ref_mpchol.so not built" >&2
fi
