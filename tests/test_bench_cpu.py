"""bench.py's CPU-side pieces without a GPU: the reference-arm timer (the
unmodified reference from oracle/_ref when built, else the C port) on a tiny
slab, and the clock sampler's degraded mode."""

import importlib.util
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(REPO, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_cpu_reference_rate_tiny():
    bench = load_bench()
    gf, info = bench.cpu_reference_rate(64, 64, 64, target_s=0.05)
    assert gf > 0
    assert info["kind"] in ("reference", "port") and info["cores"] >= 1
    assert "k-slab" in info["sample"]


def test_cpu_reference_port_matches_reference_kind_semantics():
    """The C port (kind "port") times the same algorithm: bitwise-equal C to
    the naive oracle on the slab it times."""
    import numpy as np

    import oracle

    m, n, k = 70, 9, 33
    a, b, c = oracle.make_operands(42, m, n, k)
    want = oracle.naive(m, n, k, a, m, b, k, c.copy(), m)
    got = oracle.goto(m, n, k, a, m, b, k, c.copy(), m, threads=3)
    assert np.array_equal(got, want)


def test_clock_sampler_without_nvidia_smi(monkeypatch):
    bench = load_bench()
    monkeypatch.setenv("PATH", "/nonexistent")
    s = bench.ClockSampler(0)
    s.start()
    out = s.stop()
    assert out["sm_mhz"] is None and out["reasons"]


def test_reference_arm_prints_contract_line(tmp_path):
    """`bench.py --impl reference` under a non-zero RANK exits 0 without work
    (torchrun N>1: only rank 0 times the CPU path)."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.slow
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--workload", "cfg2_8192"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GFLOP/s" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_self_launch_starts_n_ranks_dry_run():
    """`python bench.py --gpus 2` outside torchrun launches the two ranks
    itself (torch.distributed.run on 127.0.0.1); --dry-run stands in for the
    GPU arm (gloo all-reduce across the ranks), so rank 0's line must say
    n_gpus 2 and that both ranks joined."""
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["dry_run"] and line["n_gpus"] == 2 and line["ranks_joined"] == 2
    assert line["scaling"] == "strong" and line["config"]["workload"] == "cfg5"
    assert line["config"]["n"] == 32768
    assert line["schedules"] == ["nccl", "nccl-overlap", "nccl-overlap-reserve8", "chain"]


def test_world_size_must_match_gpus():
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "4", "--dry-run"],
                       capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr


def test_schedules_and_line_shape():
    """The N > 1 line: value from the fastest schedule, the others under
    alt_exchange, the exchange overhead against the compute-only time."""
    import argparse

    bench = load_bench()
    args = argparse.Namespace(exchange="all", overlap=False, reserve_sms=0, steps=4, warmup=3, workload="cfg5",
                              scaling="strong", k_chunk=2048)
    names = [nm for nm, _ in bench._schedules(args, 8)]
    assert names == ["nccl", "nccl-overlap", "nccl-overlap-reserve8", "chain"]
    assert [nm for nm, _ in bench._schedules(args, 1)] == ["single"]
    m = n = k = 32768
    flop = 2.0 * m * n * k
    results = {nm: {"ms": ms, "kern": [(ms / 4 / 16, flop / 8 / 16)] * 64, "launches": 128}
               for nm, ms in zip(names, (1100.0, 1000.0, 1050.0, 990.0))}
    clk = {nm: {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": []} for nm in names}
    line = bench._gpu_line(args, 8, 8, m, n, k, 4096, results, "chain", clk, flop, 960.0, None, None)
    assert line["n_gpus"] == 8 and line["config"]["exchange"] == "chain"
    assert line["value"] == round(flop * 4 / 0.99 / 1e9, 3)
    assert set(line["alt_exchange"]) == {"nccl", "nccl-overlap", "nccl-overlap-reserve8"}
    assert line["exchange_overhead_frac"] == round(1 - 960.0 / 990.0, 4)
    assert line["roofline"]["traffic"] is None  # the ncu capture is per 1-GPU call
    assert "emulated_world" not in line


def test_reference_arm_reports_timed_slab(monkeypatch, capsys):
    """The reference arm's ms_per_step is the timed slab's; the whole
    problem's extrapolated time has its own key."""
    import argparse

    bench = load_bench()

    class FakeRef:
        def __init__(self, m, n, k):
            self.m, self.n, self.k = m, n, k

        def depth_for(self, s):
            return 512

        def time_sample(self, d):
            return 0.5

        def flop(self, d):
            return 2.0 * self.m * self.n * d

        def info(self, d, t, reps):
            return {"kind": "reference", "cores": 16, "sample": f"k-slab {d}"}

    monkeypatch.setattr(bench, "CpuReference", FakeRef)
    monkeypatch.setattr(bench, "env_rank", lambda: (0, 1, 0))
    args = argparse.Namespace(workload="cfg5", scaling="strong", gpus=1, steps=3, warmup=3)
    assert bench.run_reference_arm(args) == 0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["ms_per_step"] == 500.0 and line["config"]["sample_k_depth"] == 512
    gf = 2.0 * 32768 * 32768 * 512 / 0.5 / 1e9
    assert line["value"] == round(gf, 3)
    assert line["ms_per_step_full_problem_extrapolated"] == round(2.0 * 32768**3 / (gf * 1e9) * 1e3, 3)


def test_cpu_reference_k_slab_is_the_reference_computation():
    """The CPU baseline's sample is C += A[:, :d] B[:d, :] on the full
    problem's operands (reference generator positions, B with ld = k): its
    result is bitwise the oracle's on the same slices."""
    import numpy as np

    import oracle

    bench = load_bench()
    m, n, k, d = 70, 50, 600, 256
    ref = bench.CpuReference(m, n, k)
    a, b, c = ref._operands(d)
    data = lambda x: np.asarray(x.data if hasattr(x, "data") and not isinstance(x, np.ndarray) else x)  # noqa: E731
    A, Bf, C0 = data(a).copy(), data(b).copy(), data(c).copy()
    full_a = oracle.fill(oracle.alloc(m, k), m, k, m, oracle.operand_seed(42, 1, m, n, k))
    full_b = oracle.fill(oracle.alloc(k, n), k, n, k, oracle.operand_seed(42, 2, m, n, k))
    assert np.array_equal(A[:m * d], full_a[:m * d])
    for j in range(n):
        assert np.array_equal(Bf[j * k:j * k + d], full_b[j * k:j * k + d])
    want = oracle.naive(m, n, d, A, m, Bf, k, C0.copy(), m)
    ref.time_sample(d)
    assert np.array_equal(data(ref._c)[:m * n], want[:m * n])
