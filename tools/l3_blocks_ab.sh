# level-3 block-size / looking-direction A/B (development aid)
for cfg in "512,128" "512,0" "256,0" "1024,128" "256,64" "512,64"; do
  for L in 0 1; do
    echo "== blocks $cfg left_looking=$L"
    MY_DGEMM_L3_BLOCKS=$cfg MY_DGEMM_L3_LEFT=$L  # (the right-looking order, L=0, was removed after this A/B) timeout 120 python tools/level3_probe.py 4096 8192 2>&1 | grep -v dsyrk
  done
done
