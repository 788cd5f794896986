"""Device-resident performance sweep over every BASELINE.json config.

  python tools/sweep.py [--quick] [--json out.json]

cfg1 512^3; cfg2 256..8192 step 256; cfg3 (4093,4099,2047), (1,8192,8192),
(8192,1,8192), (37,53,71) with lda=m+7, ldb=k+5, ldc=m+3; cfg4 16384^2 x 256;
cfg5 32768^3 (1 GPU).  Operands come from the device generator (seed 42).
Timing: CUDA events on the launch stream, 2 warm-ups, best and median of
`reps`; C is reset from a pristine copy outside the timed region when the
operands fit in L2-sized budgets, else left accumulating (same work).
Reports GFLOP/s, fraction of 37.22 TF FP64 peak, the median SM clock and
throttle reasons nvidia-smi saw while timing, and GB/s over the
algorithmic bytes 8(mk + kn + 2mn) against the 6550.7 GB/s measured HBM copy.
Launch-bound shapes (several calls per event) are also timed replayed from a
CUDA graph of the same calls (graph_us: device time per call).
"""

import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402  (nvidia-smi sampling, as the bench line does)
from paper_1609_00076_b200 import engine  # noqa: E402

PEAK_TF = 37.22
HBM_GBS = 6550.7
SEED = 42


def run(name, m, n, k, lda=None, ldb=None, ldc=None, reps=5):
    lda, ldb, ldc = lda or m, ldb or k, ldc or m
    st = torch.cuda.current_stream().cuda_stream
    a = torch.empty(lda * k, dtype=torch.float64, device="cuda")
    b = torch.empty(ldb * n, dtype=torch.float64, device="cuda")
    c = torch.empty(ldc * n, dtype=torch.float64, device="cuda")
    seeds = [engine.operand_seed(SEED, r, m, n, k) for r in (1, 2, 3)]
    engine.fill_random_device(a.data_ptr(), m, k, lda, seeds[0], 0, st)
    engine.fill_random_device(b.data_ptr(), k, n, ldb, seeds[1], 0, st)
    engine.fill_random_device(c.data_ptr(), m, n, ldc, seeds[2], 0, st)

    flop = 2.0 * m * n * k
    inner = int(min(200, max(1, 2e10 / flop)))  # amortise host launch gaps for tiny shapes

    def go():
        for _ in range(inner):
            engine.dgemm_device(m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), ldc, st)

    for _ in range(2):
        go()
    torch.cuda.synchronize()
    # enough timed reps for >= ~0.4 s under the clock sampler (100 ms period),
    # so short configs report their SM clock and throttle reasons too
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    go()
    e1.record()
    torch.cuda.synchronize()
    reps = max(reps, min(200, int(0.4 / max(e0.elapsed_time(e1) * 1e-3, 1e-6)) + 1))
    times = []
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        go()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3 / inner)
    clk = clocks.stop()
    best, med = min(times), statistics.median(times)
    graph_us = None
    if inner > 1:
        # launch-bound shapes: the same calls replayed from a CUDA graph (device
        # time without the Python/ctypes launch path between calls)
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        with torch.cuda.stream(s2):
            with torch.cuda.graph(g, stream=s2):
                for _ in range(inner):
                    engine.dgemm_device(m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), ldc,
                                        s2.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        gt = []
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            gt.append(e0.elapsed_time(e1) * 1e-3 / inner)
        graph_us = round(min(gt) * 1e6, 2)
        del g
    byts = 8.0 * (m * k + k * n + 2 * m * n)
    rec = {"config": name, "m": m, "n": n, "k": k, "lda": lda, "ldb": ldb, "ldc": ldc,
           "launches_per_event": inner, "best_us": round(best * 1e6, 2), "median_us": round(med * 1e6, 2),
           "gflops": round(flop / best / 1e9, 2), "frac_fp64_peak": round(flop / best / 1e12 / PEAK_TF, 4),
           "gbs": round(byts / best / 1e9, 1), "frac_hbm": round(byts / best / 1e9 / HBM_GBS, 4),
           "sm_mhz": clk.get("sm_mhz"), "clock_reasons": clk.get("reasons")}
    if graph_us is not None:
        rec["graph_us"] = graph_us
        rec["graph_frac_fp64_peak"] = round(flop / (graph_us * 1e-6) / 1e12 / PEAK_TF, 4)
    print(json.dumps(rec), flush=True)
    del a, b, c
    torch.cuda.empty_cache()
    return rec


def main():
    quick = "--quick" in sys.argv
    out = []
    out.append(run("cfg1", 512, 512, 512))
    sizes = range(256, 8192 + 1, 256) if not quick else (256, 1024, 2048, 4096, 8192)
    for s in sizes:
        out.append(run(f"cfg2_{s}", s, s, s, reps=3 if s >= 4096 else 5))
    out.append(run("cfg3a", 4093, 4099, 2047, 4093 + 7, 2047 + 5, 4093 + 3))
    out.append(run("cfg3b", 1, 8192, 8192, 1 + 7, 8192 + 5, 1 + 3))
    out.append(run("cfg3c", 8192, 1, 8192, 8192 + 7, 8192 + 5, 8192 + 3))
    out.append(run("cfg3d", 37, 53, 71, 37 + 7, 71 + 5, 37 + 3))
    out.append(run("cfg4", 16384, 16384, 256))
    if not quick:
        out.append(run("cfg5_1gpu", 32768, 32768, 32768, reps=2))
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
