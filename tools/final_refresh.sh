set -x
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_final.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_final.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:dgemm_fast -c 2 -o gpurun_out/prof_fast_final python tools/profile_one.py 8192 8192 8192 --launches 1 > gpurun_out/ncu_full.log 2>&1
timeout 1200 python tools/sweep.py --json gpurun_out/sweep_final.json > gpurun_out/sweep_final.log 2>&1
