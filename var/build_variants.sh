#!/usr/bin/env bash
# A/B experiment builds of libraster_b200.so with K1 compile-time knobs
# (not part of the product; outputs are git-ignored .so files).
set -euo pipefail
root="$(cd "$(dirname "$0")/.." && pwd)"
csrc="$root/paper_1907_03620_b200/csrc"
build() {
    local name="$1"; shift
    (cd "$csrc" && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
        -Xcompiler -fPIC -Xcompiler -O3 -shared "$@" -o "$root/var/lib_$name.so" \
        contract.cu agglomerate.cu agglomerate_sorted.cu label.cu points.cu dedupe.cu partition.cu api.cu) &
}
rm -f "$root"/var/lib_*.so
for spec in "$@"; do
    name="${spec%%:*}"; flags="${spec#*:}"
    build "$name" $flags
done
wait
ls "$root/var/"
