#!/bin/bash
# A/B of library builds on one box (development aid): shape_time.py for each build/variants/*.so
# and the product library, twice in alternating order.
cd "$(dirname "$0")/.."
S=${SHAPES:-"16384x16384x256 8192x8192x512 12000x12000x100 8192x8192x8192"}
for pass in 1 2; do
  for L in paper_1609_00076_b200/libmy_dgemm_b200.so build/variants/*.so; do
    MY_DGEMM_LIB=$L SHAPE_TAG="p$pass $(basename $L .so)" python tools/shape_time.py $S --reps=5
  done
done
