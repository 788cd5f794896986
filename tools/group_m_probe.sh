# DRAM traffic / time of the 8192^3 call for raster and L2-policy variants
# (build/variants/lib*.so built with -DMYD_FAST_GROUP_M=... / -DMYD_C_EVICT_FIRST).
for L in paper_1609_00076_b200/libmy_dgemm_b200.so "$@"; do
  echo "== $L"
  MY_DGEMM_LIB=$L timeout 120 python tools/perf_probe.py 8192 2>&1 | grep "8192x8192x8192 {}"
  MY_DGEMM_LIB=$L timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:dgemm_fast -s 2 -c 1 python tools/profile_one.py 8192 8192 8192 2>&1 | grep -E "dram__|gpu__time|hit_rate"
done
