set -x
python -m pytest tests -q -m gpu > gpurun_out/gputest_r02b.log 2>&1; tail -3 gpurun_out/gputest_r02b.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02b.log 2>&1; tail -1 gpurun_out/smoke_r02b.log
python bench.py > gpurun_out/bench_r02f.log 2> gpurun_out/bench_r02f.err; tail -1 gpurun_out/bench_r02f.log | cut -c1-300
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02f.log 2>&1; tail -1 gpurun_out/bench_ref_r02f.log | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_r02f.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_r02f.log 2>&1; echo "ncu launch rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dgemm_fast -c 2 -o gpurun_out/prof_cfg5_r02f python tools/profile_one.py 32768 32768 32768 --launches 1 > gpurun_out/ncu_cfg5_r02f.log 2>&1; echo "ncu cfg5 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:dgemm_small -c 2 -o gpurun_out/prof_small_r02f python tools/plan_once.py 256 256 256 0 > gpurun_out/ncu_small_r02f.log 2>&1; echo "ncu small rc=$?"
