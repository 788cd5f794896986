# Round-2 end-of-session check on one B200 (gpurun): GPU tests, smoke, bench (default cfg5),
# reference arm, ncu launch list of the bench command, the full sweep.  TAG names the outputs.
TAG=${TAG:-r02p}
set -x
python -m pytest tests -q -m gpu > gpurun_out/gputest_$TAG.log 2>&1; tail -3 gpurun_out/gputest_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; tail -1 gpurun_out/smoke_$TAG.log
python bench.py > gpurun_out/bench_$TAG.log 2> gpurun_out/bench_$TAG.err; tail -1 gpurun_out/bench_$TAG.log | cut -c1-300
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; tail -1 gpurun_out/bench_ref_$TAG.log | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench_$TAG.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launch rc=$?"
python tools/sweep.py --json gpurun_out/sweep_$TAG.json > gpurun_out/sweep_$TAG.log 2>&1; tail -2 gpurun_out/sweep_$TAG.log | cut -c1-200
# ncu --set full captures (one per gpurun call: a report is ~30 MB and gpurun_out/ carries 64 MB back):
#   gpurun -- 'python tools/profile_one.py 1024 1024 1024 --launches 2 && ncu --set full --clock-control none --import-source on \
#     -k regex:dgemm_fast -c 2 -f -o gpurun_out/prof_1024_sk_r02p python tools/profile_one.py 1024 1024 1024 --launches 2'
