#!/usr/bin/env bash
# Builds tests/cpp/_build/adapter_parity: the C++ drop-in header against the
# reference headers (test-only; needs /root/reference, so it is built in the
# build container and the binary travels to the GPU box with the snapshot).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
root="$(cd "$here/../.." && pwd)"
ref_inc="${RASTER_REF_INCLUDE:-/root/reference/proj/include}"
if [ ! -d "$ref_inc/raster" ]; then
    echo "reference headers not found at $ref_inc; skipping adapter test build" >&2
    exit 0
fi
mkdir -p "$here/_build"
g++ -std=c++20 -O2 -pthread -Wall -I"$ref_inc" -I"$root/include" \
    -o "$here/_build/adapter_parity" "$here/adapter_parity.cpp" \
    -L"$root/paper_1907_03620_b200" -lraster_b200 \
    -Wl,-rpath,'$ORIGIN/../../../paper_1907_03620_b200'
echo "built $here/_build/adapter_parity"
