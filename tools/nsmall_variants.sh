# few-column kernel variants (ROWS, WARPS, KW) at n = 8 and 16 (development aid)
for L in paper_1609_00076_b200/libmy_dgemm_b200.so "$@"; do
  echo "== $L"
  MY_DGEMM_LIB=$L timeout 120 python tools/nsmall_probe.py 2>&1 | grep -E "^8192x(12|16)x|^4096x16"
done
