#!/usr/bin/env bash
cd "$(dirname "$0")/.."
for lib in paper_1609_00076_b200/libmy_dgemm_b200.so build/variants/*.so; do
  echo "== $lib"
  MY_DGEMM_LIB=$PWD/$lib PYTHONPATH=. timeout 60 python tools/skinny_probe.py
done
