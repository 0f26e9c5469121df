#!/bin/bash
# Compiles the C++ drop-in API test against the built library (no GPU needed to build).
set -e
here=$(cd "$(dirname "$0")" && pwd)
root=$(cd "$here/../.." && pwd)
mkdir -p "$here/build"
g++ -std=c++20 -O2 -Wall -Wextra -I "$root/include" "$here/test_cpp_api.cpp" -o "$here/build/test_cpp_api" \
  -L "$root/paper_2408_04440_b200/lib" -lsphemu_gpu -Wl,-rpath,"$root/paper_2408_04440_b200/lib" \
  -Wl,-rpath-link,/usr/local/cuda/lib64 -Wl,--allow-shlib-undefined
echo "$here/build/test_cpp_api"
