#!/bin/bash
# Builds and installs the `dessim` CMake package (repo-root CMakeLists.txt,
# target dessim::dessim over the prebuilt libdesmoe.so), then builds the
# reference's own proj/tests/CMakeLists.txt against it through
# tests/cmake_consumer (test infrastructure). Output: tests/cpp/_cmake/
# (git-ignored; travels to the GPU box). Needs /root/reference and cmake.
#   tools/cmake_package.sh [outdir]
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=${1:-$ROOT/tests/cpp/_cmake}
GEN=""
command -v ninja >/dev/null && GEN="-G Ninja"
rm -rf "$OUT"
mkdir -p "$OUT"
cmake -S "$ROOT" -B "$OUT/pkg" $GEN -DDESMOE_PREBUILT="$ROOT/paper_2602_00879_b200/libdesmoe.so" > "$OUT/pkg.log"
cmake --build "$OUT/pkg" >> "$OUT/pkg.log"
cmake --install "$OUT/pkg" --prefix "$OUT/inst" >> "$OUT/pkg.log"
cmake -S "$ROOT/tests/cmake_consumer" -B "$OUT/consumer" $GEN -DCMAKE_PREFIX_PATH="$OUT/inst" > "$OUT/consumer.log"
cmake --build "$OUT/consumer" -j "$(nproc)" >> "$OUT/consumer.log"
echo "dessim package + reference tests built under $OUT"
