"""bench.py -- the driver contract for the my_dgemm path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload cfg5|cfg2_8192|cfg4|cfg3a] [--scaling strong|weak]
                  [--exchange all|nccl|chain] [--no-cpu-baseline] [--no-e2e]

N > 1 outside torchrun: bench.py starts the N ranks itself (torch.distributed
.run on 127.0.0.1, one process per GPU, NCCL); under torchrun WORLD_SIZE must
equal --gpus.  One JSON line on rank 0.

Workload (default): SURVEY 8e's scaling problem, BASELINE configs[4] -- DGEMM
C := A*B + C, m = n = k = 32768, fp64, column-major, tight leading
dimensions, operands from the reference generator (seed 42, splitmix64-v1,
generated on the device bit-exactly; 8.6 GB per matrix).  Strong scaling:
rank g owns the column panel split_columns(32768, N)[g] of B and C; A lives
on rank 0 and reaches the others inside every timed step.  At N > 1 every
exchange schedule is timed in the same run -- the serialized NCCL broadcast,
the chunked NCCL broadcast under the GEMM (with and without SMs reserved
for NCCL) and the copy-engine chain over NVLink peer memory -- and the
fastest is the value (the others under alt_exchange).  A step is one full
C += A*B.  Inputs exceed the 126 MB L2, so no flush is needed.

value  = 2*m*n*k * K / max-over-ranks device time (CUDA events), GFLOP/s.
e2e    = the same metric through the public host API, host buffers pinned,
         wall clock, max over ranks: N = 1 my_dgemm_ex with host pointers
         (H2D of A, B, C and D2H of C inside every call); N > 1
         ShardedDgemm.step_host (B / C panels per rank, A from the root's
         host memory into the exchange, C panels back).
roofline: dominant kernel = dgemm_fast_kernel; bound "tensor" (the FP64 DMMA
         pipe); achieved = 2mnk per launch / mean launch time (CUDA events on
         the launch stream); peak = 37.22 TFLOP/s nominal FP64
         (148 SM x 128 flop/clk x 1.965 GHz; our DMMA microbenchmark
         measured 37.10, profiles/fp64_peak_r01.txt).  MEASURED_PEAKS.json
         holds no FP64 figure.
cpu_baseline: the reference's own CPU path (oracle/_ref: gemmforge
         gemm_goto_parallel, compiled backend, all host threads) on a k-slab
         of the same workload (see CpuReference); "port" (oracle/ C
         restatement) if the reference package is absent.
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

import numpy as np

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
    """The reference's CPU path on a k-slab of the workload.

    kind "reference": gemmforge.parallel.gemm_goto_parallel from oracle/_ref
    (the unmodified reference, compiled backend, GotoParams() defaults, all
    host threads, loop ic when ceil(m/64) >= T else jr -- BASELINE.md 4).
    kind "port": oracle/liboracle.so's C restatement of the same algorithm.

    A sample is d (a multiple of kc = 256) consecutive pc iterations of the
    reference's own loop nest over the WHOLE m x n problem: C += A[:, :d] *
    B[:d, :] with every jc panel (nc = 4096 columns), every ic block, the same
    packing, barriers and C traffic per pc iteration as the full call, which
    is k/kc such iterations (goto.py:212-229, parallel.py:183-199).  So the
    sample's rate is the full problem's rate, which a column slab narrower
    than nc would understate (each packed A block would feed fewer columns).
    Operands come from the reference generator at their positions in the full
    matrices: A's first d columns, B's first d rows (ld = k, so the strides
    are the full problem's), C whole.  C is not reset between runs (the
    values do not change the work).
    """

    KC = 256  # GotoParams().kc

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
        self._c = None
        self._ab = (0, None, None)

    def _operands(self, d):
        m, n, k = self.m, self.n, self.k
        if self.use_ref:
            from gemmforge.bench import _operand_seed
            from gemmforge.matrix import Matrix, alloc_matrix, fill_random, random_values

            if self._c is None:
                self._c = fill_random(alloc_matrix(m, n), _operand_seed(SEED, 3, m, n, k))
            if self._ab[0] < d:
                a = fill_random(alloc_matrix(m, d), _operand_seed(SEED, 1, m, n, k))  # A[:, :d]
                b = alloc_matrix(d, n, k)  # B[:d, :] with the full problem's ld
                sb = _operand_seed(SEED, 2, m, n, k)
                for j in range(n):
                    b.data[j * k:j * k + d] = random_values(sb, d, start=j * k)
                self._ab = (d, a, b)
            _, a, b = self._ab
            return Matrix(m, d, m, a.data[:m * d]), Matrix(d, n, k, b.data), self._c
        import oracle

        if self._c is None:
            self._c = oracle.fill(oracle.alloc(m, n), m, n, m, oracle.operand_seed(SEED, 3, m, n, k))
        if self._ab[0] < d:
            a = oracle.fill(oracle.alloc(m, d), m, d, m, oracle.operand_seed(SEED, 1, m, n, k))
            b = np.zeros(k * (n - 1) + d)
            sb = oracle.operand_seed(SEED, 2, m, n, k)
            for j in range(n):
                b[j * k:j * k + d] = oracle.random_values(sb, d, start=j * k)
            self._ab = (d, a, b)
        return self._ab[1], self._ab[2], self._c

    def time_sample(self, d: int) -> float:
        a, b, c = self._operands(d)
        m, n, k, T = self.m, self.n, self.k, self.threads
        if self.use_ref:
            from gemmforge.goto import GotoParams
            from gemmforge.parallel import gemm_goto_parallel, make_plan

            p = GotoParams()
            plan = (make_plan("ic", T, m, p.mc) if -(-m // p.mc) >= T else make_plan("jr", T, n, p.nr))
            t0 = time.perf_counter()
            gemm_goto_parallel(a, b, c, p, plan)
            return time.perf_counter() - t0
        import oracle

        t0 = time.perf_counter()
        oracle.goto(m, n, d, a, m, b, k, c, m, threads=T)
        return time.perf_counter() - t0

    def flop(self, d: int) -> float:
        return 2.0 * self.m * self.n * d

    def depth_for(self, seconds: float) -> int:
        """k-slab depth (a multiple of kc, at most k) for ~`seconds` of work,
        calibrated on one pc iteration."""
        d0 = min(self.k, self.KC)
        t0 = self.time_sample(d0)
        want = seconds * self.flop(d0) / t0 / (2.0 * self.m * self.n)
        d = int(want // self.KC) * self.KC
        return max(d0, min(self.k, d))

    def info(self, d: int, t: float, reps: int) -> dict:
        m, n, k = self.m, self.n, self.k
        iters = -(-k // self.KC)
        return {"kind": "reference" if self.use_ref else "port", "cores": self.threads,
                "sample": f"k-slab C += A[:, :{d}] B[:{d}, :] over the whole {m}x{n} C (k={k}): "
                          f"{-(-d // self.KC)} of the full call's {iters} pc iterations, every jc panel and ic "
                          f"block; {self.flop(d):.3e} flop per run; best {t:.2f} s of {reps}; "
                          + ("gemmforge gemm_goto_parallel (oracle/_ref, compiled backend), GotoParams() defaults"
                             if self.use_ref else "oracle/liboracle.so oracle_goto (C port of goto/parallel)")}


def cpu_reference_rate(m: int, n: int, k: int, target_s: float = 12.0, reps: int = 1):
    ref = CpuReference(m, n, k)
    d = ref.depth_for(target_s / max(1, reps))
    t = min(ref.time_sample(d) for _ in range(max(1, reps)))
    return ref.flop(d) / t / 1e9, ref.info(d, t, reps)


def run_reference_arm(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    m, n_rank, k = WORKLOADS[args.workload]
    n = n_rank if args.scaling == "strong" else n_rank * max(world, args.gpus)  # the GPU arm's whole-job problem
    # each step a bounded slab so W+K steps finish within a few minutes
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    ref = CpuReference(m, n, k)
    d = ref.depth_for(per_step)
    rates, times = [], []
    for s in range(args.warmup + args.steps):
        t = ref.time_sample(d)
        if s >= args.warmup:
            rates.append(ref.flop(d) / t / 1e9)
            times.append(t)
    info = ref.info(d, min(times), len(times))
    value = sum(rates) / len(rates)
    flop_step = 2.0 * m * n * k
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # a step is one timed k-slab of the whole problem (d of its k/256 pc
        # iterations); the whole problem's time is extrapolated from its rate
        "ms_per_step": round(sum(times) / len(times) * 1e3, 3),
        "ms_per_step_full_problem_extrapolated": round(flop_step / (value * 1e9) * 1e3, 3),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, seed 42)",
        "config": {"workload": args.workload, "m": m, "n": n, "k": k, "lda": m, "ldb": k, "ldc": m,
                   "layout": "column-major", "sample_k_depth": d,
                   "note": "each step times the k-slab C += A[:, :sample_k_depth] B[:sample_k_depth, :] of this "
                           "problem (cpu_baseline.sample)"},
        "cpu_baseline": {"value": round(value, 3), "unit": UNIT, **info},
        "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_ms": [round(t * 1e3, 1) for t in times],
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- GPU arm


def _schedules(args, world):
    """Exchange schedules the run times.  N = 1: no exchange.  N > 1: the
    serialized NCCL broadcast, the chunked NCCL broadcast under the GEMM
    (with and without SMs reserved for NCCL), and the copy-engine chain
    over NVLink peer memory -- or only the one --exchange names."""
    if world == 1:
        return [("single", dict(exchange="nccl", overlap=False, reserve_sms=0))]
    every = [
        ("nccl", dict(exchange="nccl", overlap=False, reserve_sms=0)),
        ("nccl-overlap", dict(exchange="nccl", overlap=True, reserve_sms=0)),
        (f"nccl-overlap-reserve{args.reserve_sms or 8}",
         dict(exchange="nccl", overlap=True, reserve_sms=args.reserve_sms or 8)),
        ("chain", dict(exchange="chain", overlap=True, reserve_sms=0)),
    ]
    if args.exchange == "all":
        return every
    if args.exchange == "chain":
        return [("chain", dict(exchange="chain", overlap=True, reserve_sms=0))]
    name = "nccl-overlap" if args.overlap else "nccl"
    if args.overlap and args.reserve_sms:
        name += f"-reserve{args.reserve_sms}"
    return [(name, dict(exchange="nccl", overlap=args.overlap, reserve_sms=args.reserve_sms))]


def run_b200_arm(args):
    import torch
    import torch.distributed as dist

    from paper_1609_00076_b200 import _capi, engine
    from paper_1609_00076_b200.multi import ShardedDgemm, make_shard_plan

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # --emulate-world W (tests, one GPU): a one-rank NCCL group runs rank 0's
    # share of a W-way split through every N > 1 code path (schedules,
    # chunked broadcasts on NCCL's stream, step_host, the line's N > 1 keys);
    # no data moves and the numbers describe rank 0's panel only.
    pw = args.emulate_world or world  # the world the plan is cut for
    use_pg = world > 1 or args.emulate_world > 0
    if use_pg:
        # rank 0 logs NCCL's communicator setup ("nRanks N"); the others stay quiet
        os.environ.setdefault("NCCL_DEBUG", "INFO" if rank == 0 else "WARN")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29577")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    lib = _capi.load()

    m, n_rank, k = WORKLOADS[args.workload]
    strong = args.scaling == "strong"
    n_total = n_rank if strong else n_rank * pw
    plan = make_shard_plan(m, n_total, k, pw, root=0, k_chunk=args.k_chunk)
    j0, j1 = plan.local(rank)
    nloc = j1 - j0
    stream = torch.cuda.current_stream(dev)
    st = stream.cuda_stream

    A = torch.empty(m * k, dtype=torch.float64, device=dev)
    B = torch.empty(k * nloc, dtype=torch.float64, device=dev)
    C = torch.empty(m * nloc, dtype=torch.float64, device=dev)
    seeds = [engine.operand_seed(SEED, r, m, n_total, k) for r in (1, 2, 3)]

    def fill_a():
        if rank == 0:
            engine.fill_random_device(A.data_ptr(), m, k, m, seeds[0], 0, st)
        else:
            A.fill_(float("nan"))  # must be overwritten by the exchange

    fill_a()
    engine.fill_random_device(B.data_ptr(), k, nloc, k, seeds[1], j0, st)
    engine.fill_random_device(C.data_ptr(), m, nloc, m, seeds[2], j0, st)
    torch.cuda.synchronize()

    def barrier():
        if use_pg:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(vals):
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        if use_pg:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t]

    def sum_over_ranks(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        if use_pg:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return int(t[0])

    launch_events: list[tuple] = []

    def make_driver(opts):
        def timed_compute(mm, nl, kc, A_, lda, B_, ldb, C_, ldc):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream(dev)
            e0.record(cur)
            engine.dgemm_device(mm, nl, kc, A_.data_ptr(), lda, B_.data_ptr(), ldb, C_.data_ptr(), ldc,
                                cur.cuda_stream, path=drv.path)
            e1.record(cur)
            launch_events.append((e0, e1, kc))

        drv = ShardedDgemm(plan, rank, compute=timed_compute, overlap=opts["overlap"],
                           reserve_sms=opts["reserve_sms"])
        close = None
        if world > 1 and opts["exchange"] == "chain":  # A over NVLink by the copy engines (peer.py)
            from paper_1609_00076_b200.peer import connect_chain

            chain, close = connect_chain(A, drv.chain_spans(m), rank, world, root=0)
            drv.attach_chain(chain)
        return drv, close

    def time_steps(step_fn, steps):
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(steps):
            step_fn()
        t1.record(stream)
        barrier()
        return t0.elapsed_time(t1)

    results = {}  # name -> dict(ms, kern_ms, kern_flop, launches)
    clock_lines = {}
    flop_step = 2.0 * m * (n_total if pw == world else nloc) * k  # emulated: rank 0's share only
    done = threading.Event()
    partial: dict = {}

    def emit_partial():  # watchdog: a schedule that never completes still leaves a line
        if not done.is_set():
            if rank == 0 and partial.get("line"):
                line = dict(partial["line"])
                line.setdefault("alt_exchange", {})[partial.get("running", "?")] = "timeout"
                print(json.dumps(line), flush=True)
            os._exit(0 if partial.get("line") else 3)

    schedules = _schedules(args, pw)
    if world == 1:  # emulated: no peers for the copy-engine chain
        schedules = [(nm, o) for nm, o in schedules if o["exchange"] != "chain"]
    for name, opts in schedules:
        partial["running"] = name
        watchdog = threading.Timer(args.schedule_timeout, emit_partial) if pw > 1 else None
        if watchdog:
            watchdog.daemon = True
            watchdog.start()
        drv, close = make_driver(opts)
        step = lambda: drv.step(A, m, B, k, C, m)  # noqa: E731
        for _ in range(args.warmup):
            step()
        barrier()
        launch_events.clear()
        sampler = ClockSampler(local)
        sampler.start()
        time.sleep(0.3)
        l0 = lib.my_dgemm_kernel_launches()
        ms = time_steps(step, args.steps)
        launches = lib.my_dgemm_kernel_launches() - l0
        clock_lines[name] = sampler.stop()
        kern = [(e0.elapsed_time(e1), 2.0 * m * nloc * kc) for e0, e1, kc in launch_events]
        ms_max, = max_over_ranks([ms])
        results[name] = {"ms": ms_max, "kern": kern, "launches": sum_over_ranks(launches)}
        if close is not None:
            close()
        if watchdog:
            watchdog.cancel()
        fill_a()  # the next schedule starts from A on the root only
        torch.cuda.synchronize()
        best = min(results, key=lambda nm: results[nm]["ms"])
        partial["line"] = _gpu_line(args, world, pw, m, n_total, k, nloc, results, best, clock_lines, flop_step,
                                    None, None, None)

    best = min(results, key=lambda nm: results[nm]["ms"])
    done.set()
    compute_ms = None
    if pw > 1:  # the per-rank GEMM alone, A resident: what the exchange costs on top of it
        drv, _ = make_driver(dict(exchange="nccl", overlap=False, reserve_sms=0))
        dist.broadcast(A, src=0)
        ms = time_steps(lambda: drv.step(A, m, B, k, C, m, broadcast_a=False), args.steps)
        compute_ms, = max_over_ranks([ms])

    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(args, m, nloc, k, seeds, j0, rank, pw, n_total, plan, A, B, C, best)
    cpu = None
    if rank == 0 and pw == 1 and not args.no_cpu_baseline:
        gf, info = cpu_reference_rate(m, n_total, k, target_s=args.cpu_seconds)
        cpu = {"value": round(gf, 3), "unit": UNIT, **info}
    line = _gpu_line(args, world, pw, m, n_total, k, nloc, results, best, clock_lines, flop_step, compute_ms, e2e,
                     cpu)
    if use_pg:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


def _gpu_line(args, world, pw, m, n_total, k, nloc, results, best, clock_lines, flop_step, compute_ms, e2e, cpu):
    r = results[best]
    value = flop_step * args.steps / (r["ms"] * 1e-3) / 1e9
    kern_ms = [t for t, _ in r["kern"]]
    kern_flop = [f for _, f in r["kern"]]
    mean_kernel_s = sum(kern_ms) / len(kern_ms) * 1e-3 if kern_ms else float("nan")
    achieved = (sum(kern_flop) / len(kern_flop)) / mean_kernel_s / 1e12 if kern_ms else None
    clk = clock_lines[best]
    exchanges = {"single": "none (one GPU)", "nccl": "NCCL broadcast of A, then the GEMM",
                 "nccl-overlap": "NCCL broadcast of A in k-chunks under the GEMM",
                 "chain": "copy-engine chain of A over NVLink peer memory, k-chunks under the GEMM"}
    desc = exchanges.get(best, f"NCCL broadcast of A in k-chunks under the GEMM, {best.rsplit('reserve', 1)[-1]} "
                               "SMs reserved for NCCL")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(r["ms"] / args.steps, 4),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference splitmix64-v1 generator, seed 42, generated on device bit-exactly)",
        "config": {"workload": args.workload, "m": m, "n": n_total, "k": k,
                   "n_per_gpu": nloc, "lda": m, "ldb": k, "ldc": m, "layout": "column-major",
                   "parallelism": f"jc-shard x{pw}" + (f", {desc}" if pw > 1 else ""),
                   "exchange": best, "k_chunk": args.k_chunk if pw > 1 else None,
                   "l2": "inputs larger than L2 (no flush)"},
        "roofline": {"bound": "tensor", "achieved": round(achieved, 3) if achieved else None,
                     "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": round(achieved / FP64_PEAK_TFLOPS, 4) if achieved else None,
                     "traffic": load_traffic(args.workload, pw),
                     "kernel": "dgemm_fast_kernel whole-tile rounds + stream-K tail (one my_dgemm call = "
                               "both launches; per rank and k-chunk at N > 1)",
                     "peak_source": "nominal FP64 148SMx128flop/clkx1.965GHz (not in MEASURED_PEAKS.json); "
                                    f"DMMA microbench {FP64_PEAK_MEASURED}",
                     "launches_timed": len(kern_ms), "mean_launch_ms": round(mean_kernel_s * 1e3, 4)},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": r["launches"],
        "clocks": clk,
        "fp64_frac_at_sampled_clock": (round(value / 1e3 / (FP64_PEAK_TFLOPS * clk["sm_mhz"] / 1965.0) / world, 4)
                                       if clk.get("sm_mhz") else None),
        "fp64_frac_per_gpu": round(value / 1e3 / (FP64_PEAK_TFLOPS * world), 4),
    }
    if pw != world:
        line["emulated_world"] = pw
        line["note"] = "--emulate-world: rank 0's share of the split on a one-rank NCCL group (code-path test)"
    if pw > 1:
        line["alt_exchange"] = {nm: round(flop_step * args.steps / (x["ms"] * 1e-3) / 1e9, 3)
                                for nm, x in results.items() if nm != best}
        if compute_ms is not None:
            line["compute_only_ms_per_step"] = round(compute_ms / args.steps, 4)
            line["exchange_overhead_frac"] = round(1.0 - compute_ms / r["ms"], 4)
    return line


def measure_e2e(args, m, nloc, k, seeds, j0, rank, world, n_total, plan, A, B, C, best):
    """The same metric through the public host API, host buffers pinned,
    wall clock, max over ranks.  N = 1: my_dgemm_ex with host pointers (the
    drop-in; H2D of A, B, C and D2H of C inside every call, panel-pipelined).
    N > 1: ShardedDgemm.step_host -- every rank uploads its B / C panel, the
    root uploads A chunk by chunk into the exchange, the GEMM, D2H of the C
    panel -- with the fastest NCCL schedule (the chain falls back to the
    chunked NCCL broadcast here)."""
    import torch
    import torch.distributed as dist

    from paper_1609_00076_b200 import _capi, engine
    from paper_1609_00076_b200.multi import ShardedDgemm

    lib = _capi.load()
    dev = torch.device("cuda", torch.cuda.current_device())
    st = torch.cuda.current_stream().cuda_stream
    steps = max(1, min(args.steps, args.e2e_steps))
    hB = torch.empty(k * nloc, dtype=torch.float64, pin_memory=True)
    hC = torch.empty(m * nloc, dtype=torch.float64, pin_memory=True)
    hA = torch.empty(m * k if rank == 0 else 0, dtype=torch.float64, pin_memory=True)
    if rank == 0:
        engine.fill_random_device(A.data_ptr(), m, k, m, seeds[0], 0, st)
        hA.copy_(A)
    engine.fill_random_device(C.data_ptr(), m, nloc, m, seeds[2], j0, st)
    hB.copy_(B)
    hC.copy_(C)
    torch.cuda.synchronize()

    if world == 1:
        def call():
            _capi.check(lib.my_dgemm_ex(m, nloc, k, hA.data_ptr(), m, hB.data_ptr(), k, hC.data_ptr(), m,
                                        _capi.FORCE_PATH(engine.path(m, n_total, False)), None))
        api = "my_dgemm_ex(host pointers, pinned) -> panel-pipelined H2D/GEMM/D2H"
    else:
        overlap = best != "nccl"
        reserve = int(best.rsplit("reserve", 1)[-1]) if "reserve" in best else 0
        drv = ShardedDgemm(plan, rank, overlap=overlap, reserve_sms=reserve)

        def call():
            drv.step_host(hA, A, m, hB, B, k, hC, C, m)
        api = (f"ShardedDgemm.step_host (pinned host panels; root uploads A chunk by chunk into the "
               f"{'chunked ' if overlap else ''}NCCL broadcast{f', {reserve} SMs reserved' if reserve else ''})")

    for _ in range(1 if m * k > (1 << 28) else 2):
        call()
    if dist.is_initialized():
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    dt = time.perf_counter() - t0
    if dist.is_initialized():
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t[0])
    lib.my_dgemm_release_workspace()
    flop = 2.0 * m * (n_total if dist.is_initialized() and dist.get_world_size() == world else nloc) * k * steps
    return {"value": round(flop / dt / 1e9, 3), "unit": UNIT,
            "h2d_bytes_per_step": 8 * (m * k + (k + m) * n_total),
            "d2h_bytes_per_step": 8 * m * n_total, "steps": steps, "ms_per_step": round(dt / steps * 1e3, 3),
            "api": api}


def load_traffic(workload, world=1):
    """dram bytes per call of dgemm_fast_kernel from the committed ncu --set
    full summary (profiles/traffic.json, one entry per workload) when it was
    captured on this workload at one GPU (the per-rank call differs at
    N > 1), else None."""
    p = os.path.join(REPO, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    if world != 1:
        return None
    entry = t.get("workloads", {}).get(workload) if "workloads" in t else t
    if not entry or not str(entry.get("workload", "")).startswith(workload + " "):
        return None
    return entry.get("dram_bytes_per_launch")


def under_launcher() -> bool:
    """True inside a torchrun / torch.distributed.run worker."""
    return "WORLD_SIZE" in os.environ and "LOCAL_RANK" in os.environ


def self_launch(args) -> int:
    """`python bench.py --gpus N` outside torchrun: start the N ranks
    ourselves (one process per GPU through torch.distributed.run on
    127.0.0.1), as the reference's threaded engine creates its own workers
    (parallel.py:224-234).  Rank 0's JSON line is the output; the exit code
    is the launcher's."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def run_dry(args) -> int:
    """--dry-run: the launcher and the collective plumbing without GPU work
    (gloo): every rank joins, the world size is checked, rank 0 prints the
    line it would time."""
    import torch
    import torch.distributed as dist

    rank, world, _ = env_rank()
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        assert int(t[0]) == world
        dist.destroy_process_group()
    if rank == 0:
        m, n_rank, k = WORKLOADS[args.workload]
        n = n_rank if args.scaling == "strong" else n_rank * world
        print(json.dumps({"dry_run": True, "metric": METRIC, "unit": UNIT, "n_gpus": world, "ranks_joined": world,
                          "scaling": args.scaling, "config": {"workload": args.workload, "m": m, "n": n, "k": k},
                          "schedules": [nm for nm, _ in _schedules(args, world)]}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg5",
                    help="default cfg5: SURVEY 8e's 32768^3 problem (BASELINE configs[4]), split over the GPUs")
    ap.add_argument("--scaling", choices=("strong", "weak"), default="strong",
                    help="strong: the workload's n is the whole job, split over the ranks; weak: n per rank")
    ap.add_argument("--strong", action="store_true", help="same as --scaling strong (kept for old command lines)")
    ap.add_argument("--k-chunk", type=int, default=2048)
    ap.add_argument("--exchange", choices=("all", "nccl", "chain"), default="all",
                    help="N > 1: how A reaches the ranks -- 'all' times every schedule (serialized NCCL "
                         "broadcast, chunked NCCL broadcast under the GEMM with and without SMs reserved, the "
                         "copy-engine chain over NVLink peer memory, paper_1609_00076_b200/peer.py) and reports "
                         "the fastest as the value, the others under alt_exchange")
    ap.add_argument("--overlap", action="store_true",
                    help="with --exchange nccl: broadcast A in k-chunks under the GEMM instead of before it")
    ap.add_argument("--reserve-sms", type=int, default=0,
                    help="with the overlapped NCCL schedule: SMs kept free of the GEMM for NCCL's kernels")
    ap.add_argument("--schedule-timeout", type=float, default=300.0,
                    help="N > 1: seconds one exchange schedule may take before rank 0 reports what it has")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--emulate-world", type=int, default=0,
                    help="tests on one GPU: run rank 0's share of a W-way split through the N > 1 code paths "
                         "on a one-rank NCCL group")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch the ranks and check the collective plumbing (gloo), no GPU work")
    args = ap.parse_args()
    if args.strong:
        args.scaling = "strong"
    if args.warmup < 3:
        print("warning: the contract requires --warmup >= 3", file=sys.stderr)
    if args.gpus < 1:
        print(f"error: --gpus must be >= 1, got {args.gpus}", file=sys.stderr)
        return 2
    if not under_launcher():
        if args.gpus > 1:
            return self_launch(args)
    else:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            print(f"error: launched with WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
            return 2
    if args.dry_run:
        return run_dry(args)
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200_arm(args)


if __name__ == "__main__":
    sys.exit(main())
