#!/usr/bin/env bash
# A/B of variant builds on the GPU box: tools/ab_run.sh OUT.jsonl CONFIGS NAME...
# (each NAME is build/variants/NAME.so, run in its own process by tools/k1_ab.py)
out="$1"; cfgs="$2"; shift 2
: > "$out"
for v in "$@"; do
  RASTER_B200_LIB=build/variants/$v.so RG_K1=$v python tools/k1_ab.py $cfgs >> "$out" 2>> "$out.err"
done
cat "$out"
