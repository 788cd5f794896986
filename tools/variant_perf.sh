# perf_probe --quick for the default library and each variant given
for L in paper_1609_00076_b200/libmy_dgemm_b200.so "$@"; do
  echo "== $L"
  MY_DGEMM_LIB=$L timeout 200 python tools/perf_probe.py 4096 8192 2>&1 | grep -v exact
done
