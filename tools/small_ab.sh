for L in build/variants/lib_base.so paper_1609_00076_b200/libmy_dgemm_b200.so; do
  echo "== $L"
  MY_DGEMM_LIB=$L PLANS=0:heur,65:s1,66:s2,67:s3,70:s6,73:s9,74:s10 python tools/small_kernel_probe.py 17x17x4096 18x18x4096 128x128x2048 256x256x4096 256x256x256 128x128x128 384x384x384 512x512x512 37x53x71 1000x1000x64 100x300x1000 2>&1
done
