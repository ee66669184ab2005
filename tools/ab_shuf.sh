#!/usr/bin/env bash
# A/B of variant builds on config 4 in random order: tools/ab_shuf.sh NAME...
for v in "$@"; do
  V=$v RASTER_B200_LIB=build/variants/$v.so python tools/shuf_ab.py 4 2>/dev/null | tail -1
done
