#!/usr/bin/env bash
# Builds an experimental variant of libraster_b200.so with extra -D flags into
# build/variants/<name>.so (load it with RASTER_B200_LIB=...).
#   tools/build_variant.sh NAME -DRG_K8_FILL=32 ...
set -euo pipefail
root="$(cd "$(dirname "$0")/.." && pwd)"
name="$1"; shift
mkdir -p "$root/build/variants"
cd "$root/paper_1907_03620_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    -Xcompiler -O3 -shared "$@" -o "$root/build/variants/$name.so" \
    contract.cu agglomerate.cu agglomerate_sorted.cu label.cu points.cu dedupe.cu partition.cu api.cu
echo "built build/variants/$name.so"
