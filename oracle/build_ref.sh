#!/usr/bin/env bash
# Builds the CPU checkers (test infrastructure only):
#   oracle/_build/liboracle.so  — the C restatement (always; needs only gcc)
#   oracle/_ref/libraster_ref.so — the reference itself, compiled from its own
#       headers where they lie under /root/reference/proj/include, through
#       oracle/ref_shim.cpp. Skipped (previous build kept) when the reference
#       tree is absent, e.g. on the GPU box.
# Flags follow the reference's Release default (proj/CMakeLists.txt:6-8).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref_inc="${RASTER_REF_INCLUDE:-/root/reference/proj/include}"
mkdir -p "$here/_build" "$here/_ref"
gcc -std=c99 -O3 -fPIC -shared -Wall -Wextra -o "$here/_build/liboracle.so" \
    "$here/raster_oracle.c" -lm
if [ -d "$ref_inc/raster" ]; then
    g++ -std=c++20 -O3 -DNDEBUG -pthread -fPIC -shared -Wall \
        -I"$ref_inc" -I"$here" -o "$here/_ref/libraster_ref.so" "$here/ref_shim.cpp"
    echo "built $here/_ref/libraster_ref.so from $ref_inc"
else
    echo "reference headers not found at $ref_inc; keeping existing _ref build" >&2
fi
