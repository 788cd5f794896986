# few-row kernel variants (UNROLL, WARPS, KC, CTAs/SM) (development aid)
for L in paper_1609_00076_b200/libmy_dgemm_b200.so "$@"; do
  echo "== $L"
  MY_DGEMM_LIB=$L timeout 120 python tools/msmall_probe.py 2x8192x8192 4x8192x8192 8x4096x4096 3x5000x777 8x2048x2048 4x16384x4000 2>&1
done
