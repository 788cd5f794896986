#!/bin/bash
# Round re-alignment A/B (MY_DGEMM_ROUND_SYNC=R, an experiment build in git history): time (shape_time.py) and DRAM bytes of the
# whole-tile launch (ncu) for cfg5 and 16384^2 x 32768, R = 0 (off) / 32 / 16 / 8 (development aid).
cd "$(dirname "$0")/.."
for R in 0 32 16 8; do
  echo "== MY_DGEMM_ROUND_SYNC=$R"
  MY_DGEMM_ROUND_SYNC=$R SHAPE_TAG=R$R python tools/shape_time.py 16384x16384x32768 32768x32768x32768 --reps=2
  for s in "16384 16384 32768" "32768 32768 32768"; do
    MY_DGEMM_ROUND_SYNC=$R ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:dgemm_fast -c 1 --csv python tools/profile_one.py $s --launches 1 2>/dev/null | grep -E "dram__|gpu__time|dmma" | awk -F'","' -v s="$s" '{print "   ", s, $(NF-3), $NF}'
  done
done
