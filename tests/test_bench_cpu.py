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
    assert "column slab" in info["sample"]


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
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, env=env, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.mark.slow
def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GFLOP/s" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
