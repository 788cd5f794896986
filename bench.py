"""bench.py -- the driver contract for the my_dgemm path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload cfg2_8192|cfg5|cfg4|cfg3a] [--no-cpu-baseline]

For N>1 launch under torchrun (one rank per GPU, NCCL).  One JSON line on
rank 0.

Workload (BASELINE.json configs[1], the size sweep's headline point): DGEMM
C := A*B + C, m = k = 8192, fp64, column-major, tight leading dimensions,
operands from the reference generator (seed 42, splitmix64-v1, generated on
the device bit-exactly).  At N ranks the problem grows by columns (weak
scaling): n = 8192*N, rank g owns columns [8192g, 8192(g+1)) of B and C, A
lives on rank 0 and is broadcast over NCCL inside every step before the
per-rank GEMM (--overlap: in k-chunks under the GEMM; paper_1609_00076_b200/
multi.py explains why that is not the default).  A step
is one full C += A*B.  Inputs (3 x 512 MiB per rank) exceed the 126 MB L2,
so no flush is needed between steps.

value  = 2*m*n*k * K / max-over-ranks device time (CUDA events), GFLOP/s.
e2e    = the same metric through the public host API (my_dgemm_ex with host
         pointers from pinned memory: H2D of A, B, C and D2H of C inside every
         step), wall-clock, rank 0 / per-rank host call at N>1.
roofline: dominant kernel = dgemm_fast_kernel; bound "tensor" (the FP64 DMMA
         pipe); achieved = 2mnk per launch / mean launch time (CUDA events on
         the launch stream); peak = 37.22 TFLOP/s nominal FP64
         (148 SM x 128 flop/clk x 1.965 GHz; our DMMA microbenchmark
         measured 37.10, profiles/fp64_peak_r01.txt).  MEASURED_PEAKS.json
         holds no FP64 figure.
cpu_baseline: the reference's own CPU path (oracle/_ref: gemmforge
         gemm_goto_parallel, compiled backend, all host threads) on a column
         slab of the same workload; "port" (oracle/ C restatement) if the
         reference package is absent.
`--impl reference` times that CPU path as the reference arm.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

FP64_PEAK_TFLOPS = 37.22  # nominal: 148 SM x 128 flop/clk x 1.965 GHz
FP64_PEAK_MEASURED = 37.10  # DMMA.8x8x4 microbenchmark on this pool (profiles/fp64_peak_r01.txt)
SEED = 42
METRIC = "DGEMM GFLOPS (2mnk/s)"
UNIT = "GFLOP/s"

WORKLOADS = {
    # name: (m, n_per_rank, k)
    "cfg2_8192": (8192, 8192, 8192),
    "cfg5": (32768, 32768, 32768),  # n is per rank here; --strong splits the 32768^3 problem
    "cfg4": (16384, 16384, 256),
    "cfg3a": (4093, 4099, 2047),
}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, pw, reasons = [], None, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
                pw.append(float(parts[3]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------- CPU legs


class CpuReference:
    """The reference's CPU path on column slabs of the workload.

    kind "reference": gemmforge.parallel.gemm_goto_parallel from oracle/_ref
    (the unmodified reference, compiled backend, GotoParams() defaults, all
    host threads, loop ic when ceil(m/64) >= T else jr -- BASELINE.md 4),
    timed per the reference protocol (bench.py:109-123: C reset outside the
    timed region).  kind "port": oracle/liboracle.so's C restatement of the
    same five-loop algorithm.  A (m x k) is generated once and reused.
    """

    def __init__(self, m: int, n: int, k: int):
        self.m, self.n, self.k = m, n, k
        self.threads = len(os.sched_getaffinity(0))
        ref_path = os.path.join(REPO, "oracle", "_ref")
        use_ref = os.path.isdir(os.path.join(ref_path, "gemmforge"))
        if use_ref:
            if ref_path not in sys.path:
                sys.path.insert(0, ref_path)
            from gemmforge.backends import available_backends
            use_ref = "c" in available_backends()
        self.use_ref = use_ref
        self._a = None
        self._slabs = {}

    def _operands(self, ns):
        m, n, k = self.m, self.n, self.k
        if self.use_ref:
            from gemmforge.bench import _operand_seed
            from gemmforge.matrix import alloc_matrix, fill_random

            if self._a is None:
                self._a = fill_random(alloc_matrix(m, k), _operand_seed(SEED, 1, m, n, k))
            if ns not in self._slabs:
                self._slabs = {ns: (fill_random(alloc_matrix(k, ns), _operand_seed(SEED, 2, m, n, k)),
                                    fill_random(alloc_matrix(m, ns), _operand_seed(SEED, 3, m, n, k)))}
        else:
            import oracle

            if self._a is None:
                self._a = oracle.fill(oracle.alloc(m, k), m, k, m, oracle.operand_seed(SEED, 1, m, n, k))
            if ns not in self._slabs:
                self._slabs = {ns: (
                    oracle.fill(oracle.alloc(k, ns), k, ns, k, oracle.operand_seed(SEED, 2, m, n, k)),
                    oracle.fill(oracle.alloc(m, ns), m, ns, m, oracle.operand_seed(SEED, 3, m, n, k)))}
        return (self._a, *self._slabs[ns])

    def time_slab(self, ns: int) -> float:
        a, b, c0 = self._operands(ns)
        m, k, T = self.m, self.k, self.threads
        if self.use_ref:
            from gemmforge.goto import GotoParams
            from gemmforge.matrix import copy_matrix
            from gemmforge.parallel import gemm_goto_parallel, make_plan

            p = GotoParams()
            plan = (make_plan("ic", T, m, p.mc) if -(-m // p.mc) >= T else make_plan("jr", T, ns, p.nr))
            c = copy_matrix(c0)  # reset outside the timed region
            t0 = time.perf_counter()
            gemm_goto_parallel(a, b, c, p, plan)
            return time.perf_counter() - t0
        import oracle

        c = c0.copy()
        t0 = time.perf_counter()
        oracle.goto(m, ns, k, a, m, b, k, c, m, threads=T)
        return time.perf_counter() - t0

    def slab_for(self, seconds: float) -> int:
        """Columns for ~`seconds` of work, calibrated on a 16-column slab."""
        ns0 = max(1, min(self.n, 16))
        t0 = self.time_slab(ns0)
        rate = 2.0 * self.m * ns0 * self.k / t0
        return int(max(ns0, min(self.n, seconds * rate / (2.0 * self.m * self.k))))

    def info(self, ns: int, t: float, reps: int) -> dict:
        m, k = self.m, self.k
        return {"kind": "reference" if self.use_ref else "port", "cores": self.threads,
                "sample": f"column slab B[:, :{ns}] of m={m} k={k} (n={self.n}); "
                          f"{2.0 * m * ns * k:.3e} flop per run; best {t:.2f} s of {reps}; "
                          + ("gemmforge gemm_goto_parallel (oracle/_ref, compiled backend), GotoParams() defaults"
                             if self.use_ref else "oracle/liboracle.so oracle_goto (C port of goto/parallel)")}


def cpu_reference_rate(m: int, n: int, k: int, target_s: float = 12.0, reps: int = 1):
    ref = CpuReference(m, n, k)
    ns = ref.slab_for(target_s / max(1, reps))
    t = min(ref.time_slab(ns) for _ in range(max(1, reps)))
    return 2.0 * m * ns * k / t / 1e9, ref.info(ns, t, reps)


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    m, n_rank, k = WORKLOADS[args.workload]
    n = n_rank if args.strong else n_rank * max(world, args.gpus)  # the GPU arm's whole-job problem
    # each step a bounded slab so W+K steps finish within a few minutes
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    ref = CpuReference(m, n, k)
    ns = ref.slab_for(per_step)
    rates, times = [], []
    for s in range(args.warmup + args.steps):
        t = ref.time_slab(ns)
        if s >= args.warmup:
            rates.append(2.0 * m * ns * k / t / 1e9)
            times.append(t)
    info = ref.info(ns, min(times), len(times))
    value = sum(rates) / len(rates)
    flop_step = 2.0 * m * n * k
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(flop_step / (value * 1e9) * 1e3, 3),
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, seed 42)",
        "config": {"workload": args.workload, "m": m, "n": n, "k": k, "lda": m, "ldb": k, "ldc": m,
                   "layout": "column-major", "note": "each step times a column slab (cpu_baseline.sample)"},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, **info},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm


def run_b200_arm(args):
    import torch
    import torch.distributed as dist

    from paper_1609_00076_b200 import _capi, engine
    from paper_1609_00076_b200.multi import ShardedDgemm, make_shard_plan

    rank, world, local = env_rank()
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _capi.load()

    m, n_rank, k = WORKLOADS[args.workload]
    n_total = n_rank if args.strong else n_rank * world  # strong: the workload's n split over the ranks
    plan = make_shard_plan(m, n_total, k, world, root=0, k_chunk=args.k_chunk)
    j0, j1 = plan.local(rank)
    nloc = j1 - j0
    stream = torch.cuda.current_stream(dev)
    st = stream.cuda_stream

    A = torch.empty(m * k, dtype=torch.float64, device=dev)
    B = torch.empty(k * nloc, dtype=torch.float64, device=dev)
    C = torch.empty(m * nloc, dtype=torch.float64, device=dev)
    seeds = [engine.operand_seed(SEED, r, m, n_total, k) for r in (1, 2, 3)]
    if rank == 0:
        engine.fill_random_device(A.data_ptr(), m, k, m, seeds[0], 0, st)
    else:
        A.fill_(float("nan"))  # must be overwritten by the broadcast
    engine.fill_random_device(B.data_ptr(), k, nloc, k, seeds[1], j0, st)
    engine.fill_random_device(C.data_ptr(), m, nloc, m, seeds[2], j0, st)
    torch.cuda.synchronize()

    # per-launch timing of the dominant kernel: events around each GEMM launch
    launch_events: list[tuple] = []

    def timed_compute(mm, nl, kc, A_, lda, B_, ldb, C_, ldc):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        engine.dgemm_device(mm, nl, kc, A_.data_ptr(), lda, B_.data_ptr(), ldb, C_.data_ptr(), ldc,
                            st, path=drv.path)
        e1.record(stream)
        launch_events.append((e0, e1, kc))

    drv = ShardedDgemm(plan, rank, compute=timed_compute, overlap=args.overlap, reserve_sms=args.reserve_sms)
    close_chain = None
    if world > 1 and args.exchange == "chain":  # A over NVLink by the copy engines (peer.py)
        from paper_1609_00076_b200.peer import connect_chain

        chain, close_chain = connect_chain(A, drv.chain_spans(m), rank, world, root=0)
        drv.attach_chain(chain)

    def step():
        drv.step(A, m, B, k, C, m)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    launch_events.clear()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = lib.my_dgemm_kernel_launches()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    barrier()
    t_start.record(stream)
    for _ in range(args.steps):
        step()
    t_end.record(stream)
    barrier()
    launches = lib.my_dgemm_kernel_launches() - launches0
    clk = clocks.stop()
    ms = t_start.elapsed_time(t_end)
    kern_ms = [e0.elapsed_time(e1) for e0, e1, _ in launch_events]
    kern_flop = [2.0 * m * nloc * kc for _, _, kc in launch_events]
    if world > 1:
        t = torch.tensor([ms, float(launches)], dtype=torch.float64, device=dev)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, launches_total = float(mx[0]), int(sm[1])
    else:
        ms_max, launches_total = ms, int(launches)
    flop_step = 2.0 * m * n_total * k
    value = flop_step * args.steps / (ms_max * 1e-3) / 1e9

    exchange_name = ("copy-engine chain over NVLink peer memory" if args.exchange == "chain"
                     else "NCCL broadcast")
    if close_chain is not None:
        close_chain()
    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(args, m, nloc, k, seeds, j0, rank, world, n_total)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        gf, info = cpu_reference_rate(m, n_total, k, target_s=args.cpu_seconds)
        cpu = {"value": round(gf, 3), "unit": UNIT, **info}

    if rank == 0:
        mean_kernel_s = sum(kern_ms) / len(kern_ms) * 1e-3
        achieved = (sum(kern_flop) / len(kern_flop)) / mean_kernel_s / 1e12
        traffic = load_traffic(args.workload)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4),
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference splitmix64-v1 generator, seed 42, generated on device bit-exactly)",
            "config": {"workload": args.workload, "m": m, "n": n_total, "k": k,
                       "n_per_gpu": nloc, "lda": m, "ldb": k, "ldc": m, "layout": "column-major",
                       "parallelism": f"jc-shard x{world}" + (
                           (f", {exchange_name} of A in {len(drv.plan.chunks)} k-chunks under the GEMM" if args.overlap
                            else f", {exchange_name} of A, then the GEMM") if world > 1 else ""),
                       "l2": "inputs larger than L2 (no flush)"},
            "roofline": {"bound": "tensor", "achieved": round(achieved, 3), "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                         "traffic": traffic, "kernel": "dgemm_fast_kernel<2,128,128,32> whole-tile rounds + stream-K tail (one call = both launches)",
                         "peak_source": "nominal FP64 148SMx128flop/clkx1.965GHz (not in MEASURED_PEAKS.json); "
                                        f"DMMA microbench {FP64_PEAK_MEASURED}",
                         "launches_timed": len(kern_ms), "mean_launch_ms": round(mean_kernel_s * 1e3, 4)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_total,
            "clocks": clk,
            "fp64_frac_at_sampled_clock": (round(value / 1e3 / (FP64_PEAK_TFLOPS * clk["sm_mhz"] / 1965.0)
                                                 / world, 4) if clk.get("sm_mhz") else None),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def measure_e2e(args, m, nloc, k, seeds, j0, rank, world, n_total):
    """Same metric through the public host API: my_dgemm_ex on pinned host
    buffers (H2D of A, B_g, C_g and D2H of C_g every step), wall clock, max
    over ranks.  At N>1 every rank stages its own copy of A (a host-memory
    broadcast is outside the API); the device broadcast path is `value`."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1609_00076_b200 import _capi

    lib = _capi.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    # operands generated on device, copied once into pinned host buffers (setup, untimed)
    hA = torch.empty(m * k, dtype=torch.float64, pin_memory=True)
    hB = torch.empty(k * nloc, dtype=torch.float64, pin_memory=True)
    hC = torch.empty(m * nloc, dtype=torch.float64, pin_memory=True)
    from paper_1609_00076_b200 import engine

    for h, (rows, cols, seed, c0) in zip((hA, hB, hC), ((m, k, seeds[0], 0), (k, nloc, seeds[1], j0),
                                                       (m, nloc, seeds[2], j0))):
        d = torch.empty(rows * cols, dtype=torch.float64, device=dev)
        engine.fill_random_device(d.data_ptr(), rows, cols, rows, seed, c0,
                                  torch.cuda.current_stream().cuda_stream)
        h.copy_(d)
        del d
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, args.e2e_steps))

    def call():
        _capi.check(lib.my_dgemm_ex(m, nloc, k, hA.data_ptr(), m, hB.data_ptr(), k, hC.data_ptr(), m,
                                    _capi.FORCE_PATH(engine.path(m, n_total, False)), None))

    for _ in range(2):
        call()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t[0])
    lib.my_dgemm_release_workspace()
    flop = 2.0 * m * n_total * k * steps
    return {"value": round(flop / dt / 1e9, 3), "unit": UNIT,
            "h2d_bytes_per_step": 8 * (m * k * world + (k + m) * n_total),
            "d2h_bytes_per_step": 8 * m * n_total, "steps": steps,
            "api": "my_dgemm_ex(host pointers, pinned) -> panel-pipelined H2D/GEMM/D2H"}


def load_traffic(workload):
    """dram bytes per call of dgemm_fast_kernel from the committed ncu --set
    full summary (profiles/traffic.json) when it was captured on this
    workload, else None."""
    p = os.path.join(REPO, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    return t.get("dram_bytes_per_launch") if str(t.get("workload", "")).startswith(workload + " ") else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2_8192")
    ap.add_argument("--k-chunk", type=int, default=2048)
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: the workload's n is the total, split over the ranks (e.g. "
                         "--workload cfg5 --strong: SURVEY 8e's 32768^3 on 1/2/4/8 GPUs)")
    ap.add_argument("--overlap", action="store_true",
                    help="broadcast A in k-chunks under the GEMM instead of before it (N>1)")
    ap.add_argument("--exchange", choices=("nccl", "chain"), default="nccl",
                    help="N > 1: how A reaches the ranks -- NCCL broadcast, or the copy-engine chain over "
                         "NVLink peer memory (no SMs; paper_1609_00076_b200/peer.py)")
    ap.add_argument("--reserve-sms", type=int, default=0,
                    help="with --overlap: SMs kept free of the GEMM for NCCL's kernels")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: the contract requires --warmup >= 3", file=sys.stderr)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200_arm(args)


if __name__ == "__main__":
    sys.exit(main())
