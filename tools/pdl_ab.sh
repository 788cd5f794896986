for v in 0 1; do
  echo "== MY_DGEMM_NO_PDL=$v"
  MY_DGEMM_NO_PDL=$v timeout 300 python tools/sweep.py --quick 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['config'], d['best_us'], d['frac_fp64_peak'])"
  MY_DGEMM_NO_PDL=$v LD_LIBRARY_PATH=$PWD/paper_1609_00076_b200 tools/microbench/host_overhead 512 512
  MY_DGEMM_NO_PDL=$v LD_LIBRARY_PATH=$PWD/paper_1609_00076_b200 tools/microbench/host_overhead 2048 2048
done
