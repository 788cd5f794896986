#!/bin/bash
# Split-boundary A/B (development aid): device time of short- and long-K shapes for the product
# library and build/variants/lib_sb*.so (-DMYD_SPLIT_BOUNDARY=0, -DMYD_SB_KSTEPS=...).
cd "$(dirname "$0")/.."
S="16384x16384x256 16384x16384x128 8192x8192x512 12000x12000x100 4096x4096x4096 8192x8192x8192 2048x2048x2048 4093x4099x2047"
for L in paper_1609_00076_b200/libmy_dgemm_b200.so build/variants/lib_sb*.so paper_1609_00076_b200/libmy_dgemm_b200.so; do
  echo "== $L"
  MY_DGEMM_LIB=$L SHAPE_TAG=$(basename $L .so) python tools/shape_time.py $S --reps=5
done
