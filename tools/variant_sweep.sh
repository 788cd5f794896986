#!/usr/bin/env bash
# Time the product library and every build/variants/*.so on a few shapes.
cd "$(dirname "$0")/.."
for lib in paper_1609_00076_b200/libmy_dgemm_b200.so build/variants/*.so; do
  echo "== $lib"
  MY_DGEMM_LIB=$PWD/$lib PYTHONPATH=. timeout 120 python tools/perf_probe.py --quick "$@"
done
