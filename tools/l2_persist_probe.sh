#!/bin/bash
# Persisting-L2 carve-out + eviction hints (development aid): device time and
# DRAM bytes of the 8192^3 call's launches for the product library and each
# variant build/variants/lib_h<hint>g<GROUP_M>p<persist MB>.so
# (-DMYD_L2_HINTS, -DMYD_FAST_GROUP_M, -DMYD_L2_PERSIST_MB).
cd "$(dirname "$0")/.."
out=gpurun_out/l2_persist_${1:-r02}.log
: > $out
for lib in paper_1609_00076_b200/libmy_dgemm_b200.so build/variants/lib_h*p*.so; do
  [ -f $lib ] || continue
  echo "== $lib" >> $out
  MY_DGEMM_LIB=$lib timeout 300 python tools/perf_probe.py --quick 8192 >> $out 2>&1
  MY_DGEMM_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --kernel-name regex:dgemm_fast_kernel -c 2 --csv python tools/profile_one.py 8192 8192 8192 2>/dev/null | grep -E "dram__|gpu__time|lts__|dmma" >> $out
done
