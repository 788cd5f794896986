#!/bin/bash
# Staggered start of the whole-tile rounds (MY_DGEMM_STAGGER phase groups):
# device time per shape for groups 1 (off), 2, 4, 8 (development aid).
cd "$(dirname "$0")/.."
out=gpurun_out/stagger_${1:-r02}.log
: > $out
SHAPES="16384x16384x256 16384x16384x128 8192x8192x512 12000x12000x100 4096x4096x4096 8192x8192x8192 4093x4099x2047 2048x2048x2048"
for g in 1 4 2 8 1; do
  MY_DGEMM_STAGGER=$g SHAPE_TAG="g=$g" timeout 600 python tools/shape_time.py $SHAPES >> $out 2>&1
  MY_DGEMM_STAGGER=$g SHAPE_TAG="g=$g" timeout 600 python tools/shape_time.py 16384x16384x256 --ldc-odd >> $out 2>&1
done
