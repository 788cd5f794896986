#!/bin/bash
# L2 eviction-priority hints and raster band height (development aid):
# device time and DRAM bytes of the main launch at 8192^3 and cfg4 for each
# variant library (build/variants/lib_*.so, built with -DMYD_L2_HINTS=...,
# -DMYD_FAST_GROUP_M=...).  Output: gpurun_out/l2_hints_*.log
cd "$(dirname "$0")/.."
out=gpurun_out/l2_hints_${1:-r02}.log
: > $out
for lib in build/variants/lib_h3g8.so build/variants/lib_h4g8.so build/variants/lib_h3g12.so build/variants/lib_h2g8.so; do
  [ -f $lib ] || continue
  echo "== $lib" >> $out
  MY_DGEMM_LIB=$lib timeout 300 python tools/perf_probe.py --quick 8192 >> $out 2>&1
  MY_DGEMM_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none --kernel-name regex:dgemm_fast_kernel -c 3 --csv python tools/profile_one.py 8192 8192 8192 2>/dev/null | grep -E "dram__|gpu__time|lts__" >> $out
done
