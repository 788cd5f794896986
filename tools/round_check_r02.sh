# Round-2 end-of-session check on one B200 (gpurun): GPU tests, smoke, bench (default cfg5),
# reference arm, ncu launch list of the bench command, the full sweep.
set -x
python -m pytest tests -q -m gpu > gpurun_out/gputest_r02d.log 2>&1; tail -3 gpurun_out/gputest_r02d.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02d.log 2>&1; tail -1 gpurun_out/smoke_r02d.log
python bench.py > gpurun_out/bench_r02j.log 2> gpurun_out/bench_r02j.err; tail -1 gpurun_out/bench_r02j.log | cut -c1-300
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r02j.log 2>&1; tail -1 gpurun_out/bench_ref_r02j.log | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_r02j.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_r02j.log 2>&1; echo "ncu launch rc=$?"
python tools/sweep.py --json gpurun_out/sweep_r02j.json > gpurun_out/sweep_r02j.log 2>&1; tail -2 gpurun_out/sweep_r02j.log
