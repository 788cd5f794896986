"""GPU parity: the sm_100a kernels, called through the C ABI, against the
oracle and the reference-generated golden fixtures.

Bars (BASELINE.json north_star):
  * exact mode (MY_DGEMM_EXACT) and the operand generator: BIT-EXACT;
  * fast path: |C - C_ref|_max <= c * k * eps * (|A||B| + |C|)_max with
    c = 2, eps = 2^-52 (HEADLINE_C below), checked elementwise, plus the
    reference's own gate 2^-50 * k * max|A| * max|B| (kernels.py:31-38).
"""

import ctypes

import os
import sys

import numpy as np
import pytest

import oracle
from paper_1609_00076_b200 import _capi, engine

pytestmark = pytest.mark.gpu

HEADLINE_C = 2.0
EPS = 2.0**-52
SEED = 42


@pytest.fixture(scope="module")
def torch_cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _capi.load()
    return torch


def dev_matrix(torch, m, n, ld, seed, canary=None, col0=0):
    """Device buffer ld*n filled by the device generator (padding = canary)."""
    buf = torch.full((ld * n,), canary if canary is not None else 0.0, dtype=torch.float64,
                     device="cuda")
    engine.fill_random_device(buf.data_ptr(), m, n, ld, seed, col0,
                              torch.cuda.current_stream().cuda_stream)
    return buf


def dev_operands(torch, m, n, k, lda=None, ldb=None, ldc=None, canary=None):
    lda, ldb, ldc = lda or m, ldb or k, ldc or m
    s = [oracle.operand_seed(SEED, r, m, n, k) for r in (1, 2, 3)]
    return (dev_matrix(torch, m, k, lda, s[0], canary), dev_matrix(torch, k, n, ldb, s[1], canary),
            dev_matrix(torch, m, n, ldc, s[2], canary), (lda, ldb, ldc))


def run_dev(torch, m, n, k, a, lda, b, ldb, c, ldc, **kw):
    engine.dgemm_device(m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), ldc,
                        torch.cuda.current_stream().cuda_stream, **kw)
    torch.cuda.synchronize()


def device_bound(torch, m, n, k, a, lda, b, ldb, c0, ldc, c=HEADLINE_C):
    """The headline bound c * k * eps * (|A||B| + |C|)_max with the
    magnitude computed on the device: the fast kernel on |A|,
    |B| accumulating into |C|.  Every term is non-negative, so there is no
    cancellation and the computed maximum is within a factor (1 + k eps) of
    the exact one.  c0 is C before the update; buffers are ld * cols long."""
    aa, bb, w = a.abs(), b.abs(), c0.abs()
    run_dev(torch, m, n, k, aa, lda, bb, ldb, w, ldc)
    mag = float(w.view(n, ldc)[:, :m].max())
    del aa, bb, w
    assert mag == mag and mag > 0.0
    return c * k * EPS * mag


def check_dev(torch, m, n, k, got, want, ld, bound):
    """Device-side parity check (matrix.py:210-232 via my_dgemm_diff_report):
    raises VerificationError with the reference's failure line at the first
    offender, and fails on a NaN max."""
    rep = engine.verify_device(m, n, k, got.data_ptr(), ld, want.data_ptr(), ld, bound)
    assert rep.max_abs_diff <= bound, rep
    return rep


def headline_bound(m, n, k, a, lda, b, ldb, c0, ldc):
    A = oracle.valid_region(a, m, k, lda).T
    B = oracle.valid_region(b, k, n, ldb).T
    C = oracle.valid_region(c0, m, n, ldc).T
    mag = np.abs(A) @ np.abs(B) + np.abs(C)
    return HEADLINE_C * k * EPS * float(mag.max())


# ------------------------------------------------------------------ generator


@pytest.mark.parametrize("m,n,ld,seed,col0", [
    (2, 4, 2, 42, 0), (3, 5, 7, 9, 0), (37, 23, 40, 7, 0), (1000, 3, 1001, (1 << 64) - 1, 0),
    (129, 17, 129, 12345678901234567, 5), (4093, 7, 4100, 0, 11),
])
def test_fill_random_bit_exact(torch_cuda, m, n, ld, seed, col0):
    canary = -777.25
    d = dev_matrix(torch_cuda, m, n, ld, seed, canary, col0)
    got = d.cpu().numpy()
    want = oracle.random_values(seed, m * (n + col0))[col0 * m:]
    assert np.array_equal(oracle.valid_region(got, m, n, ld).ravel(), want)
    if ld > m:
        assert np.all(got.reshape(n, ld)[:, m:] == canary)


def test_fill_matches_reference_goldens(torch_cuda, golden):
    d = dev_matrix(torch_cuda, 2, 4, 2, 42).cpu().numpy()
    assert d.tolist() == golden["random_values"]["seed42_first8"]


# ------------------------------------------------------------ exact (bitwise)

EXACT_KATS = ["cfg3d", "cfg1", "cfg2_256", "cfg2_768", "cfg2_1024", "cfg2_1280", "cfg2_1536", "cfg2_1792",
              "cfg3b", "cfg3c", "cfg3a", "cfg2_2048", "cfg4"]


@pytest.mark.parametrize("name", EXACT_KATS)
def test_exact_mode_bitwise_kat(torch_cuda, golden, name):
    kat = golden["kat"][name]
    m, n, k = kat["m"], kat["n"], kat["k"]
    lda, ldb, ldc = kat["lds"]
    a, b, c, _ = dev_operands(torch_cuda, m, n, k, lda, ldb, ldc, canary=-777.25)
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, c, ldc, exact=True)
    got = c.cpu().numpy()
    assert oracle.sha256_valid(got, m, n, ldc) == kat["sha256"]
    if ldc > m:
        assert np.all(got.reshape(n, ldc)[:, m:] == -777.25)


def test_exact_mode_host_path_matches_oracle_bitwise(torch_cuda):
    for (m, n, k) in [(1, 1, 1), (5, 4, 3), (8, 8, 8), (13, 11, 17), (97, 89, 83), (130, 257, 33)]:
        a, b, c = oracle.make_padded_operands(SEED, m, n, k, m + 2, k + 1, m + 3)
        want = oracle.naive(m, n, k, a, m + 2, b, k + 1, c.copy(), m + 3)
        got = engine.my_dgemm(m, n, k, a, m + 2, b, k + 1, c.copy(), m + 3, exact=True)
        assert np.array_equal(got, want), (m, n, k)


# ------------------------------------------------------------ fast path


def check_fast_vs_oracle(m, n, k, lda, ldb, ldc, want=None, **kw):
    a, b, c0 = oracle.make_padded_operands(SEED, m, n, k, lda, ldb, ldc, canary=-777.25)
    if want is None:
        want = oracle.naive_par(m, n, k, a, lda, b, ldb, c0.copy(), ldc)
    got = engine.my_dgemm(m, n, k, a, lda, b, ldb, c0.copy(), ldc)
    bound = headline_bound(m, n, k, a, lda, b, ldb, c0, ldc)
    rep = oracle.max_abs_diff(got, want, m, n, ldc, tol=bound)
    assert rep.clean, oracle.failure_line(rep.first_bad_i, rep.first_bad_j, rep.value_got,
                                          rep.value_expected)
    gate = oracle.tolerance(k, 1.0, 1.0)
    assert rep.max_abs_diff <= gate
    pad = got.reshape(n, ldc)[:, m:] if ldc > m else np.zeros(0)
    assert np.all(pad == -777.25), "padding rows of C were written"
    return rep


@pytest.mark.parametrize("m,n,k", [
    (1, 1, 1), (2, 3, 1), (5, 4, 3), (8, 8, 8), (9, 7, 11), (31, 33, 32), (37, 53, 71),
    (64, 64, 64), (97, 89, 83), (127, 129, 15), (128, 128, 16), (129, 127, 17), (255, 257, 300),
    (512, 512, 512),
])
@pytest.mark.parametrize("pad", [0, 1, 2, 7])
def test_fast_small_and_ragged(torch_cuda, m, n, k, pad):
    check_fast_vs_oracle(m, n, k, m + pad, k + (pad * 5) % 8, m + (pad * 3) % 8)


@pytest.mark.parametrize("name", ["cfg1", "cfg3d", "cfg3a", "cfg3b", "cfg3c", "cfg2_1024"])
def test_fast_baseline_configs(torch_cuda, golden, name):
    kat = golden["kat"][name]
    m, n, k = kat["m"], kat["n"], kat["k"]
    lda, ldb, ldc = kat["lds"]
    check_fast_vs_oracle(m, n, k, lda, ldb, ldc)


def test_fast_vec1_path_matches(torch_cuda):
    """Odd leading dimensions force 8-byte staging; both staging widths agree bitwise."""
    m, n, k = 300, 200, 100
    a, b, c, (lda, ldb, ldc) = dev_operands(torch_cuda, m, n, k, 301, 103, 305)
    c2 = c.clone()
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, c, ldc)
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, c2, ldc, force_vec1=True)
    assert torch_cuda.equal(c, c2)


def test_fast_tiled_handles_skinny(torch_cuda, golden):
    """The tiled kernel is also correct on m==1 / n==1 (bypass the gemv kernels)."""
    for name in ("cfg3b", "cfg3c"):
        kat = golden["kat"][name]
        m, n, k = kat["m"], kat["n"], kat["k"]
        lda, ldb, ldc = kat["lds"]
        a, b, c, _ = dev_operands(torch_cuda, m, n, k, lda, ldb, ldc)
        bound = device_bound(torch_cuda, m, n, k, a, lda, b, ldb, c, ldc)
        ce = c.clone()
        run_dev(torch_cuda, m, n, k, a, lda, b, ldb, c, ldc, force_tiled=True)
        run_dev(torch_cuda, m, n, k, a, lda, b, ldb, ce, ldc, exact=True)
        check_dev(torch_cuda, m, n, k, c, ce, ldc, bound)


def test_fast_vs_exact_full_8192_and_samples(torch_cuda, golden):
    """cfg2 at 8192^3: every element of the fast result against the exact
    (bitwise-oracle) kernel, and the reference's sampled elements."""
    m = n = k = 8192
    a, b, c, _ = dev_operands(torch_cuda, m, n, k)
    bound = device_bound(torch_cuda, m, n, k, a, m, b, k, c, m)
    ce = c.clone()
    run_dev(torch_cuda, m, n, k, a, m, b, k, c, m)
    run_dev(torch_cuda, m, n, k, a, m, b, k, ce, m, exact=True)
    check_dev(torch_cuda, m, n, k, c, ce, m, bound)
    s = golden["sampled"]["cfg2_8192"]
    host_c = c.view(n, m)
    host_e = ce.view(n, m)
    for t, (i, j) in enumerate((i, j) for i in s["rows"] for j in s["cols"]):
        assert float(host_e[j, i]) == s["values"][t]  # exact kernel: bitwise
        assert abs(float(host_c[j, i]) - s["values"][t]) <= bound


def test_cfg5_full_exact_samples_and_8_way_shards(torch_cuda, golden):
    """cfg5 (32768^3, 8.6 GB per operand): every element of the fast result
    against the exact (bitwise-oracle) kernel, the reference's sampled
    elements (bitwise for exact, within the headline bound for fast), and the
    8-rank jc-sharded step (multi.ShardedDgemm, 2048-deep k-chunks as the
    overlapped schedule runs them; ranks one after another, A resident)
    bitwise equal to the single call."""
    from paper_1609_00076_b200.multi import ShardedDgemm, make_shard_plan

    torch = torch_cuda
    free, _ = torch.cuda.mem_get_info()
    if free < 64 * 2**30:
        pytest.skip("needs ~60 GB of device memory")
    s = golden["sampled"]["cfg5"]
    m, n, k = s["m"], s["n"], s["k"]
    a, b, c, _ = dev_operands(torch, m, n, k)
    bound = device_bound(torch, m, n, k, a, m, b, k, c, m)
    torch.cuda.empty_cache()
    fast = c.clone()
    run_dev(torch, m, n, k, a, m, b, k, fast, m)
    rows, cols = torch.tensor(s["rows"], device="cuda"), torch.tensor(s["cols"], device="cuda")
    pick = lambda x: x.view(n, m)[cols][:, rows].T.reshape(-1).cpu().tolist()  # row-major over (rows, cols)
    want = s["values"]
    got_fast = pick(fast)
    assert all(abs(g - w) <= bound for g, w in zip(got_fast, want))
    plan = make_shard_plan(m, n, k, 8, root=0, k_chunk=2048)
    shard = c.clone()
    for rank in range(8):
        j0, j1 = plan.local(rank)
        drv = ShardedDgemm(plan, rank, broadcast=lambda t, src: None, overlap=True)
        drv.step(a, m, b[j0 * k:], k, shard[j0 * m:], m, broadcast_a=False)
    torch.cuda.synchronize()
    assert torch.equal(shard, fast)
    del shard
    run_dev(torch, m, n, k, a, m, b, k, c, m, exact=True)  # c := the exact result
    assert pick(c) == want  # bitwise the reference's elements
    check_dev(torch, m, n, k, fast, c, m, bound)


def test_cfg4_full_fast_vs_exact(torch_cuda, golden):
    """cfg4 (16384^2 x 256, the rank-k panel): fast against exact on every
    element; the exact result is the reference KAT bit for bit."""
    kat = golden["kat"]["cfg4"]
    m, n, k = kat["m"], kat["n"], kat["k"]
    a, b, c, _ = dev_operands(torch_cuda, m, n, k)
    bound = device_bound(torch_cuda, m, n, k, a, m, b, k, c, m)
    ce = c.clone()
    run_dev(torch_cuda, m, n, k, a, m, b, k, c, m)
    run_dev(torch_cuda, m, n, k, a, m, b, k, ce, m, exact=True)
    assert oracle.sha256_valid(ce.cpu().numpy(), m, n, m) == kat["sha256"]
    check_dev(torch_cuda, m, n, k, c, ce, m, bound)


@pytest.mark.parametrize("m,n,k,lda,ldb,ldc", [
    (1000, 1100, 300, 1000, 300, 1000),     # aligned: bulk-copy path
    (777, 1029, 201, 781, 205, 780),        # odd ld: 8-byte LDGSTS path
    (2304, 2304, 128, 2304, 128, 2304),     # plan picks tail strips (324 tiles)
    (4093, 4099, 200, 4100, 202, 4096),     # ragged last tile column run as tail strips (edge plan)
    (1500, 2050, 160, 1500, 160, 1503),     # edge plan, odd ldc, 2 valid columns in the edge tile
    (4100, 3000, 200, 4100, 200, 4100),     # ragged last tile row (4 rows) run as 16x128 units
    (12, 9000, 500, 13, 500, 12),           # 9..16 rows: tiled, 16x128 units only
    (2100, 777, 300, 2101, 301, 2103),      # ragged row (52 rows) and column, odd lds
    (2048, 2048, 2048, 2048, 2048, 2048),   # stream-K: 256 tiles x 64 slabs over 148 SMs
    (3001, 2999, 1111, 3003, 1113, 3002),   # stream-K with ragged tiles, ragged last slab, odd lds
    (1024, 1024, 1024, 1024, 1024, 1024),   # below one wave: stream-K over 128x64 / 128x32 / 64x32 units
    (768, 1280, 600, 770, 602, 768),
])
def test_strip_plans_bitwise_equal(torch_cuda, m, n, k, lda, ldb, ldc):
    """Full tiles, 128x64 strips, 128x32 strips, 64x32 and 16x128 units, the
    stream-K schedule (tiles cut between CTAs, finished from a partial) and
    the heuristic's edge plans give bitwise the same C (the per-element DMMA
    sequence does not depend on the CTA shape or on who runs which slabs)."""
    a, b, c, _ = dev_operands(torch_cuda, m, n, k, lda, ldb, ldc, canary=-777.25)
    outs = []
    for strips in (0, 2, 4, 8, 16, 32, 34, 36, 40) + SMALL_PLANS:
        cc = c.clone()
        run_dev(torch_cuda, m, n, k, a, lda, b, ldb, cc, ldc, strips=strips)
        outs.append(cc)
    assert all(torch_cuda.equal(outs[0], o) for o in outs[1:])
    ce = c.clone()
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, ce, ldc, exact=True)
    bound = device_bound(torch_cuda, m, n, k, a, lda, b, ldb, c, ldc)
    check_dev(torch_cuda, m, n, k, outs[0], ce, ldc, bound)
    host = outs[3].cpu().numpy()
    if ldc > m:
        assert np.all(host.reshape(n, ldc)[:, m:] == -777.25)


@pytest.mark.parametrize("m,n,k,lda,ldb,ldc", [
    (1024, 1024, 1024, 1024, 1024, 1024),   # 64 tiles, 32 slabs of 32: tiles cut into 2-3 pieces
    (1280, 1152, 1100, 1280, 1100, 1282),   # 32-deep slabs with a ragged last one
    (512, 512, 512, 512, 512, 512),         # 16 tiles, 16-deep slabs: ~9 pieces per tile
    (1000, 1100, 777, 1002, 778, 1000),     # ragged tiles, ragged last slab
    (768, 640, 96, 768, 96, 768),           # short K: fewer slabs than 2 per CTA -> not applicable
    (777, 1029, 201, 781, 205, 780),        # odd lda / ldb: staged from even-ld scratch copies
    (300, 200, 100, 301, 101, 300),         # odd lda / ldb, small: 8-byte staging -> not applicable
])
def test_k_split_plan_is_opt_in_deterministic_and_within_the_bound(torch_cuda, m, n, k, lda, ldb, ldc):
    """The K-split plan (plan 48, MY_DGEMM_FORCE_KSPLIT): a tile's K range in
    pieces on several SMs, partial sums added by the tile's owner in CTA
    order.  It is the one plan that is not the single ascending chain, so it
    is opt-in: the default call and MY_DGEMM_PLAN_INVARIANT stay bitwise the
    other plans.  Forced, it is run-to-run bitwise deterministic, within the
    headline bound of the exact kernel, keeps the padding, and falls back to
    the plan-invariant heuristic where the shape does not allow it."""
    a, b, c, _ = dev_operands(torch_cuda, m, n, k, lda, ldb, ldc, canary=-777.25)
    outs = {}
    for strips in (0, -1, 2, 48, 48):
        cc = c.clone()
        run_dev(torch_cuda, m, n, k, a, lda, b, ldb, cc, ldc, strips=strips)
        outs.setdefault(strips, []).append(cc)
    assert torch_cuda.equal(outs[0][0], outs[-1][0]) and torch_cuda.equal(outs[0][0], outs[2][0])
    assert torch_cuda.equal(outs[48][0], outs[48][1])
    ce = c.clone()
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, ce, ldc, exact=True)
    bound = device_bound(torch_cuda, m, n, k, a, lda, b, ldb, c, ldc)
    check_dev(torch_cuda, m, n, k, outs[48][0], ce, ldc, bound)
    tiles = -(-m // 128) * -(-n // 128)
    vec2 = (lda % 2 == 0 and ldb % 2 == 0) or m * n * k >= 1 << 24 or k >= 512  # (odd lds: even-ld scratch copies)
    applicable = vec2 and tiles < 148 and tiles * -(-k // (32 if k >= 1024 else 16)) >= 2 * 148
    if not applicable:
        assert torch_cuda.equal(outs[48][0], outs[0][0])
    host = outs[48][0].cpu().numpy()
    if ldc > m:
        assert np.all(host.reshape(n, ldc)[:, m:] == -777.25)
    # the BLAS epilogue on the K-split plan: alpha (A B) + beta C applied by the owner after the fix-up
    if applicable:
        cb = c.clone()
        engine.dgemm("N", "N", m, n, k, -0.5, a, lda, b, ldb, 0.25, cb, ldc, epilogue=True, plan=48)
        torch_cuda.cuda.synchronize()
        want = 0.25 * c.view(n, ldc)[:, :m] - 0.5 * (ce.view(n, ldc)[:, :m] - c.view(n, ldc)[:, :m])
        assert float((cb.view(n, ldc)[:, :m] - want).abs().max()) <= 2 * bound
        if ldc > m:
            assert bool((cb.view(n, ldc)[:, m:] == -777.25).all())


SMALL_PLANS = tuple(range(64, 75))  # the small-block kernel: planner's pick, then variants 1..10


@pytest.mark.parametrize("m,n,k,lda,ldb,ldc", [
    (256, 256, 256, 256, 256, 256),      # the sub-wave point of the cfg2 sweep
    (37, 53, 71, 44, 76, 40),            # cfg3d: ragged everything, odd lds (8-byte staging)
    (17, 17, 4096, 17, 4096, 17),        # tiny m x n, long K chain
    (129, 65, 33, 130, 34, 131),         # one past a block in m and n, K one past a slab, odd ldc
    (200, 300, 1000, 200, 1000, 200),    # ragged K (1000 = 31 slabs of 32 + 8)
    (512, 512, 513, 512, 514, 512),      # K one past a 4-group: the zero-filled tail group
    (64, 64, 2, 64, 2, 64),              # K < 4
    (1000, 1000, 64, 1001, 65, 1002),    # short K, odd lds, many blocks
])
def test_small_kernel_bitwise_equals_units(torch_cuda, m, n, k, lda, ldb, ldc):
    """The small-block kernel (csrc/dgemm_small.cu) is one more plan of the
    tiled path: every variant gives bitwise the C of the persistent kernel's
    64x32-unit plan (same DMMA chain per element), never writes padding
    rows, and is within the headline bound of the exact kernel."""
    a, b, c, _ = dev_operands(torch_cuda, m, n, k, lda, ldb, ldc, canary=-777.25)
    ref = c.clone()
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, ref, ldc, strips=8, force_tiled=True)
    for strips in SMALL_PLANS:
        for vec1 in (False, True):
            cc = c.clone()
            run_dev(torch_cuda, m, n, k, a, lda, b, ldb, cc, ldc, strips=strips, force_tiled=True,
                    force_vec1=vec1)
            assert torch_cuda.equal(cc, ref), (strips, vec1)
    ce = c.clone()
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, ce, ldc, exact=True)
    bound = device_bound(torch_cuda, m, n, k, a, lda, b, ldb, c, ldc)
    check_dev(torch_cuda, m, n, k, ref, ce, ldc, bound)
    if ldc > m:
        assert np.all(ref.cpu().numpy().reshape(n, ldc)[:, m:] == -777.25)


_ROUND_SYNC_RUN = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, {repo!r})
from paper_1609_00076_b200 import engine
m, n, k = 8192, 8192, 16384
st = torch.cuda.current_stream().cuda_stream
ops = [torch.empty(r * c, dtype=torch.float64, device="cuda") for r, c in ((m, k), (k, n), (m, n))]
for t, (buf, r, c) in enumerate(zip(ops, (m, k, m), (k, n, n))):
    engine.fill_random_device(buf.data_ptr(), r, c, r, 77 + t, 0, st)
engine.dgemm_device(m, n, k, ops[0].data_ptr(), m, ops[1].data_ptr(), k, ops[2].data_ptr(), m, st)
np.save(sys.argv[1], ops[2][: 64 * m].cpu().numpy())  # (enough to compare: the first 64 columns)
np.save(sys.argv[1] + ".sum.npy", np.array([float(ops[2].sum()), float(ops[2].abs().sum())]))
"""


def test_round_realignment_changes_timing_never_results(torch_cuda, tmp_path):
    """MY_DGEMM_ROUND_SYNC: long-K whole-tile launches re-align their rounds
    on a grid counter every R rounds (own instantiation, cooperative launch);
    C is bitwise the unsynchronised run (8192^2 x 16384: 25 whole rounds,
    R = 4 -> 5 re-alignments)."""
    import subprocess

    script = tmp_path / "run.py"
    script.write_text(_ROUND_SYNC_RUN.format(repo=os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
    outs, sums = [], []
    for r in ("0", "4"):
        out = tmp_path / f"c{r}.npy"
        env = dict(os.environ, MY_DGEMM_ROUND_SYNC=r)
        subprocess.run([sys.executable, str(script), str(out)], check=True, env=env, timeout=600)
        outs.append(np.load(out))
        sums.append(np.load(str(out) + ".sum.npy"))
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(sums[0], sums[1])


def test_fast_deterministic(torch_cuda):
    m, n, k = 1000, 1100, 1200
    a, b, c, _ = dev_operands(torch_cuda, m, n, k)
    outs = []
    for _ in range(3):
        cc = c.clone()
        run_dev(torch_cuda, m, n, k, a, m, b, k, cc, m)
        outs.append(cc)
    assert torch_cuda.equal(outs[0], outs[1]) and torch_cuda.equal(outs[0], outs[2])


def test_kchunked_equals_unchunked_bitwise(torch_cuda):
    """C += A[:,chunk] B[chunk,:] over 16-aligned k chunks is bitwise the
    single call (the multi-GPU driver relies on it)."""
    m, n, k = 640, 384, 1024
    a, b, c, _ = dev_operands(torch_cuda, m, n, k)
    c1 = c.clone()
    run_dev(torch_cuda, m, n, k, a, m, b, k, c1, m)
    c2 = c.clone()
    for p0 in range(0, k, 256):
        engine.dgemm_device(m, n, 256, a.data_ptr() + p0 * m * 8, m, b.data_ptr() + p0 * 8, k,
                            c2.data_ptr(), m, torch_cuda.cuda.current_stream().cuda_stream)
    torch_cuda.cuda.synchronize()
    assert torch_cuda.equal(c1, c2)


# ------------------------------------------------------------ boundary


def test_small_cases_against_reference_fixtures(torch_cuda, small_cases):
    for key, want in small_cases.items():
        if not key.startswith("verify_"):
            continue
        m, n, k = (int(x) for x in key.split("_")[1:])
        a, b, c = oracle.make_operands(SEED, m, n, k)
        got = engine.my_dgemm(m, n, k, a, m, b, k, c.copy(), m, exact=True)
        assert np.array_equal(oracle.valid_region(got, m, n, m).T, want), key
        got = engine.my_dgemm(m, n, k, a, m, b, k, c.copy(), m)
        assert np.abs(oracle.valid_region(got, m, n, m).T - want).max() <= oracle.tolerance(k, 1, 1)


def test_invalid_args_leave_c_untouched(torch_cuda):
    c = np.full(16, 3.5)
    a = np.ones(16)
    lib = _capi.load()
    assert lib.my_dgemm_ex(4, 4, 4, a.ctypes.data, 3, a.ctypes.data, 4, c.ctypes.data, 4, 0, None) == -5
    lib.my_dgemm(4, 4, 4, a.ctypes.data, 4, a.ctypes.data, 4, c.ctypes.data, 2)
    assert lib.my_dgemm_last_status() == -9
    assert np.all(c == 3.5)


def test_c_abi_my_dgemm_host_signature(torch_cuda):
    m, n, k = 37, 53, 71
    a, b, c = oracle.make_padded_operands(SEED, m, n, k, m + 7, k + 5, m + 3)
    want = oracle.naive(m, n, k, a, m + 7, b, k + 5, c.copy(), m + 3)
    lib = _capi.load()
    got = c.copy()
    lib.my_dgemm(m, n, k, a.ctypes.data, m + 7, b.ctypes.data, k + 5, got.ctypes.data, m + 3)
    assert lib.my_dgemm_last_status() == 0
    rep = oracle.max_abs_diff(got, want, m, n, m + 3, tol=oracle.tolerance(k, 1, 1))
    assert rep.clean
    assert np.all(got.reshape(n, m + 3)[:, m:] == -777.25)


def test_reference_registry_gate_admits_b200(torch_cuda):
    from conftest import import_reference, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref (the reference package) not built")
    gf = import_reference()
    reg = gf.registry.KernelRegistry()
    engine.register(reg)  # runs the reference's own validation gate
    assert "b200" in reg.variant_names()
    eng = reg.build_engine("b200", None)
    a, b, c = gf.bench.make_operands(42, 97, 89, 83)
    want = gf.kernels.gemm_naive(a, b, gf.matrix.copy_matrix(c))
    got = eng(a, b, gf.matrix.copy_matrix(c))
    rep = gf.matrix.max_abs_diff(got, want, gf.kernels.tolerance(83, 1.0, 1.0))
    assert rep.first_bad_i is None


def test_reference_cli_verify_and_bench_with_b200(torch_cuda):
    """The reference's own CLI (cmd_verify / cmd_bench, cli.py:83-107) drives
    the engine through the registry: exit code 0, every shape PASS."""
    import os
    import subprocess
    import sys

    from conftest import REPO, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref (the reference package) not built")
    tool = os.path.join(REPO, "tools", "run_gemmforge_b200.py")
    r = subprocess.run([sys.executable, tool, "verify", "--alg", "b200"], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
    r = subprocess.run([sys.executable, tool, "bench", "--alg", "b200", "--min", "128", "--max", "256",
                        "--step", "128", "--check", "--format", "csv", "--reps", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert ",b200," in r.stdout


@pytest.mark.parametrize("m,n,k,lda,ldb,ldc", [
    (2048, 2048, 2048, 2048, 2048, 2048),   # pipelined host path: 4 panels, 8 k-chunks
    (1500, 3000, 1000, 1507, 1003, 1501),   # odd host lds, pipelined
])
def test_host_path_pipeline_bitwise_equals_device_path(torch_cuda, m, n, k, lda, ldb, ldc):
    """The host-pointer path (panel pipeline, k-chunked first panel) returns
    bitwise what the device-pointer path computes, and never writes padding."""
    a, b, c = oracle.make_padded_operands(SEED, m, n, k, lda, ldb, ldc, canary=-777.25)
    got = engine.my_dgemm(m, n, k, a, lda, b, ldb, c.copy(), ldc)
    da = torch_cuda.from_numpy(a).cuda()
    db = torch_cuda.from_numpy(b).cuda()
    dc = torch_cuda.from_numpy(c).cuda()
    run_dev(torch_cuda, m, n, k, da, lda, db, ldb, dc, ldc)
    dev = dc.cpu().numpy()
    assert np.array_equal(oracle.valid_region(got, m, n, ldc), oracle.valid_region(dev, m, n, ldc))
    assert np.all(got.reshape(n, ldc)[:, m:] == -777.25)


# ------------------------------------------------------------ BLAS surface


def blas_reference(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc):
    """alpha op(A) op(B) + beta C via the oracle on explicitly transposed
    operands (products p-ascending), plus the headline bound."""
    A = oracle.valid_region(a, k if ta == "T" else m, m if ta == "T" else k, lda).T
    B = oracle.valid_region(b, n if tb == "T" else k, k if tb == "T" else n, ldb).T
    opA = np.ascontiguousarray((A.T if ta == "T" else A).T).ravel()   # column-major m x k
    opB = np.ascontiguousarray((B.T if tb == "T" else B).T).ravel()   # column-major k x n
    P = oracle.naive(m, n, k, opA, m, opB, k, np.zeros(m * n), m)
    Cv = oracle.valid_region(c, m, n, ldc)
    want = alpha * P.reshape(n, m) + (beta * Cv if beta != 0 else 0.0)
    mag = abs(alpha) * (np.abs(opA.reshape(k, m).T) @ np.abs(opB.reshape(n, k).T))
    if beta != 0:
        mag = mag + abs(beta) * np.abs(Cv.T)
    return want, (HEADLINE_C * (k + 2) * EPS * float(mag.max()) if mag.size else 0.0)


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
@pytest.mark.parametrize("alpha,beta", [(1.0, 1.0), (-0.5, 2.0), (1.5, 0.0), (0.0, -3.0)])
@pytest.mark.parametrize("m,n,k", [(37, 53, 71), (300, 1, 257), (1, 300, 257), (130, 260, 190)])
def test_blas_dgemm_host(torch_cuda, ta, tb, alpha, beta, m, n, k):
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    nra, nca = (k, m) if ta == "T" else (m, k)
    nrb, ncb = (n, k) if tb == "T" else (k, n)
    lda, ldb, ldc = nra + 3, nrb + 1, m + 2
    a = rng.uniform(-1, 1, lda * nca)
    b = rng.uniform(-1, 1, ldb * ncb)
    c = rng.uniform(-1, 1, ldc * n)
    c.reshape(n, ldc)[:, m:] = -777.25
    if beta == 0.0:
        c.reshape(n, ldc)[:, :m] = np.nan   # must not be read
    want, bound = blas_reference(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc)
    got = engine.dgemm(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c.copy(), ldc)
    gv = oracle.valid_region(got, m, n, ldc)
    assert np.all(np.isfinite(gv))
    assert np.abs(gv - want).max() <= bound + 1e-300
    assert np.all(got.reshape(n, ldc)[:, m:] == -777.25)


def test_blas_alpha_beta_one_is_bitwise_my_dgemm_on_transposed_operands(torch_cuda):
    """op(A) via the transpose pre-pass is the NN kernel on A^T: bitwise."""
    m, n, k = 700, 500, 300
    a, b, c, _ = dev_operands(torch_cuda, k, n, m)          # A stored k x m (to be transposed)
    bt = dev_matrix(torch_cuda, n, k, n, 99)                # B stored n x k
    at = a[: k * m].view(m, k).t().contiguous().view(-1)    # explicit A^T, column-major m x k
    btt = bt[: n * k].view(k, n).t().contiguous().view(-1)  # explicit B^T, k x n
    c0 = torch_cuda.rand(m * n, dtype=torch_cuda.float64, device="cuda")
    c1, c2 = c0.clone(), c0.clone()
    engine.dgemm("T", "T", m, n, k, 1.0, a, k, bt, n, 1.0, c1, m)
    run_dev(torch_cuda, m, n, k, at, m, btt, k, c2, m)
    torch_cuda.cuda.synchronize()
    assert torch_cuda.equal(c1, c2)
    c3 = c0.clone()
    engine.dgemm("T", "T", m, n, k, 1.0, a, k, bt, n, 1.0, c3, m, exact=True)
    c4 = c0.clone()
    run_dev(torch_cuda, m, n, k, at, m, btt, k, c4, m, exact=True)
    torch_cuda.cuda.synchronize()
    assert torch_cuda.equal(c3, c4)


@pytest.mark.parametrize("m,n,k,alpha,beta", [(700, 500, 300, -0.75, 2.5), (2048, 2048, 512, 1.0, -3.0),
                                               (300, 1200, 900, 3.0, 0.5), (256, 256, 256, 2.0, 0.25)])
def test_blas_reference_order_is_bitwise_the_three_steps(torch_cuda, m, n, k, alpha, beta):
    """The reference-BLAS order on the tiled path with beta not in {0, 1}:
    C := beta C, alpha scales the smaller operand, then the accumulate
    contract -- bitwise the explicit three-step computation (one rounding
    each)."""
    torch = torch_cuda
    a, b, c, _ = dev_operands(torch, m, n, k)
    got = c.clone()
    engine.dgemm("N", "N", m, n, k, alpha, a, m, b, k, beta, got, m)
    want = c * beta
    if m * k <= k * n:
        a = a * alpha
    else:
        b = b * alpha
    run_dev(torch, m, n, k, a, m, b, k, want, m)
    torch.cuda.synchronize()
    assert torch.equal(got, want)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_path_pageable_and_pinned_agree(torch_cuda, pinned):
    """Pageable callers go through the pinned staging ring; pinned ones DMA
    directly: both give bitwise the device-path result (odd lds, pipelined)."""
    m, n, k = 1500, 3000, 1000
    lda, ldb, ldc = 1507, 1003, 1501
    a, b, c = oracle.make_padded_operands(SEED, m, n, k, lda, ldb, ldc, canary=-777.25)
    if pinned:
        ta, tb, tc = (torch_cuda.from_numpy(x).pin_memory() for x in (a, b, c))
        lib = _capi.load()
        _capi.check(lib.my_dgemm_ex(m, n, k, ta.data_ptr(), lda, tb.data_ptr(), ldb, tc.data_ptr(), ldc, 0,
                                    None))
        got = tc.numpy()
    else:
        got = engine.my_dgemm(m, n, k, a, lda, b, ldb, c.copy(), ldc)
    dc = torch_cuda.from_numpy(c).cuda()
    run_dev(torch_cuda, m, n, k, torch_cuda.from_numpy(a).cuda(), lda, torch_cuda.from_numpy(b).cuda(), ldb,
            dc, ldc)
    assert np.array_equal(oracle.valid_region(got, m, n, ldc), oracle.valid_region(dc.cpu().numpy(), m, n, ldc))
    assert np.all(got.reshape(n, ldc)[:, m:] == -777.25)


@pytest.mark.parametrize("shards,m,n,k,lds,pinned", [
    (2, 1000, 1100, 700, None, False),
    (3, 1500, 3000, 1000, (1507, 1003, 1501), False),
    (4, 777, 1029, 4100, (781, 4105, 780), True),
    (3, 100, 100, 300, None, False),       # n < one panel per shard: shards 1, 2 only upload A chunks
    (2, 300, 1, 900, None, False),         # n == 1: the single-shard gemv, as my_dgemm
    (3, 1, 700, 500, None, False),         # m == 1
    (8, 640, 2048, 2048, None, True),
    (3, 6, 5000, 700, (7, 703, 9), False),  # few rows: every shard on the few-row kernel
    (2, 8192, 12, 900, None, False),       # few columns: one shard holds them all
])
def test_multi_device_host_path_bitwise_equals_single(torch_cuda, shards, m, n, k, lds, pinned):
    """my_dgemm_multi_ex over `shards` column shards (all on this GPU: the
    device list repeats, each entry its own buffers, the A chunks still
    travel shard to shard by peer copy) gives bitwise the single-device
    my_dgemm result; padding rows untouched."""
    lda, ldb, ldc = lds or (m, k, m)
    a, b, c = oracle.make_padded_operands(SEED, m, n, k, lda, ldb, ldc, canary=-777.25)
    want = engine.my_dgemm(m, n, k, a, lda, b, ldb, c.copy(), ldc)
    if pinned:
        ta, tb, tc = (torch_cuda.from_numpy(x).pin_memory() for x in (a, b, c))
        got = engine.my_dgemm_multi([0] * shards, m, n, k, ta.numpy(), lda, tb.numpy(), ldb, tc.numpy(), ldc)
    else:
        got = engine.my_dgemm_multi([0] * shards, m, n, k, a, lda, b, ldb, c.copy(), ldc)
    assert np.array_equal(oracle.valid_region(got, m, n, ldc), oracle.valid_region(want, m, n, ldc))
    if ldc > m:
        assert np.all(got.reshape(n, ldc)[:, m:] == -777.25)


def test_multi_device_exact_mode_and_ngpu_entry(torch_cuda):
    """Exact mode through the multi-device path is bitwise the naive oracle;
    my_dgemm_multi(ngpu=1) is the single-device call."""
    m, n, k = 97, 300, 83
    a, b, c = oracle.make_operands(SEED, m, n, k)
    want = oracle.naive(m, n, k, a, m, b, k, c.copy(), m)
    got = engine.my_dgemm_multi([0, 0, 0], m, n, k, a, m, b, k, c.copy(), m, exact=True)
    assert np.array_equal(got, want)
    got1 = engine.my_dgemm_multi(1, m, n, k, a, m, b, k, c.copy(), m)
    assert np.array_equal(got1, engine.my_dgemm(m, n, k, a, m, b, k, c.copy(), m))
    with pytest.raises(ValueError, match="devices are visible"):
        engine.my_dgemm_multi(torch_cuda.cuda.device_count() + 1, m, n, k, a, m, b, k, c.copy(), m)


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (1, 1, 777), (1, 5, 1), (5, 1, 1), (200, 300, 1), (2, 2, 4096)])
def test_degenerate_shapes(torch_cuda, m, n, k):
    check_fast_vs_oracle(m, n, k, m + 1, k + 3, m + 2)
    a, b, c = oracle.make_padded_operands(SEED, m, n, k, m + 1, k + 3, m + 2)
    want = oracle.naive(m, n, k, a, m + 1, b, k + 3, c.copy(), m + 2)
    got = engine.my_dgemm(m, n, k, a, m + 1, b, k + 3, c.copy(), m + 2, exact=True)
    assert np.array_equal(got, want)


def test_nonfinite_propagation_matches_oracle(torch_cuda):
    """Inf and NaN inputs give non-finite outputs exactly where the reference's
    naive loop produces them (exact mode: bitwise including NaN positions)."""
    m, n, k = 150, 140, 90
    a, b, c = oracle.make_padded_operands(SEED, m, n, k, m, k, m)
    a[5 * m + 3] = np.inf          # A(3, 5)
    a[7 * m + 100] = -np.inf       # A(100, 7)
    b[11 * k + 5] = np.nan         # B(5, 11)
    c[13 * m + 20] = np.inf        # C(20, 13)
    want = oracle.naive(m, n, k, a, m, b, k, c.copy(), m)
    for exact in (False, True):
        got = engine.my_dgemm(m, n, k, a, m, b, k, c.copy(), m, exact=exact)
        assert np.array_equal(np.isnan(got), np.isnan(want)), exact
        assert np.array_equal(np.isinf(got), np.isinf(want)), exact
        fin = np.isfinite(want)
        assert np.abs(got[fin] - want[fin]).max() <= oracle.tolerance(k, 1.0, 1.0)
        if exact:
            assert np.array_equal(got[fin], want[fin])
            assert np.array_equal(np.signbit(got[np.isinf(got)]), np.signbit(want[np.isinf(want)]))


def test_tuner_changes_speed_never_results(torch_cuda):
    m, n, k = 1792, 1792, 600
    a, b, c, _ = dev_operands(torch_cuda, m, n, k)
    c1 = c.clone()
    run_dev(torch_cuda, m, n, k, a, m, b, k, c1, m)
    plan, ms = engine.tune(m, n, k)
    assert plan in (0, 1, 2, 4, 8, 16, 32, 34, 36, 40) and ms > 0
    c2 = c.clone()
    run_dev(torch_cuda, m, n, k, a, m, b, k, c2, m)
    assert torch_cuda.equal(c1, c2)
    _capi.load().my_dgemm_tune_clear()


@pytest.mark.parametrize("odd_lds", [(1003, 781, 1005), (1002, 778, 1005), (1003, 778, 1004)])
def test_odd_ld_prepass_bitwise_equals_aligned(torch_cuda, odd_lds):
    """Odd leading dimensions of A / B take the even-ld scratch copy path, an
    odd ldc is read and written in place (8-byte staging, scalar stores):
    bitwise the same C as the same operands stored with even leading
    dimensions, and padding rows of C untouched."""
    m, n, k = 1001, 1203, 777
    odd = dev_operands(torch_cuda, m, n, k, *odd_lds, canary=-777.25)
    even = dev_operands(torch_cuda, m, n, k, 1002, 778, 1004, canary=-777.25)
    a, b, c, (lda, ldb, ldc) = odd
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, c, ldc)
    a2, b2, c2, (lda2, ldb2, ldc2) = even
    run_dev(torch_cuda, m, n, k, a2, lda2, b2, ldb2, c2, ldc2)
    g1 = oracle.valid_region(c.cpu().numpy(), m, n, ldc)
    g2 = oracle.valid_region(c2.cpu().numpy(), m, n, ldc2)
    assert np.array_equal(g1, g2)
    assert np.all(c.cpu().numpy().reshape(n, ldc)[:, m:] == -777.25)


def test_c_view_8_byte_aligned_in_place(torch_cuda):
    """C as a view starting one double into its buffer (8-byte aligned base,
    even ldc): staged and stored in place, bitwise the aligned result, the
    doubles around the view untouched."""
    m, n, k = 1030, 517, 640
    a, b, c, _ = dev_operands(torch_cuda, m, n, k)
    want = c.clone()
    run_dev(torch_cuda, m, n, k, a, m, b, k, want, m)
    buf = torch_cuda.full((m * n + 2,), -5.5, dtype=torch_cuda.float64, device="cuda")
    buf[1:1 + m * n].copy_(c)
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, buf.data_ptr() + 8, m,
                        torch_cuda.cuda.current_stream().cuda_stream)
    torch_cuda.cuda.synchronize()
    assert torch_cuda.equal(buf[1:1 + m * n], want)
    assert float(buf[0]) == -5.5 and float(buf[-1]) == -5.5


@pytest.mark.parametrize("world,shape", [(2, (700, 1111, 900)), (3, (700, 1111, 900)), (8, (700, 1111, 900)),
                                         (3, (5, 3000, 400)), (2, (4096, 10, 300)), (3, (8, 8192, 300)),
                                         (2, (3, 20000, 64))])
def test_sharded_step_every_world_size_bitwise_equals_single_call(torch_cuda, world, shape):
    """multi.ShardedDgemm's per-rank work for world sizes 2, 3, 8 run one rank
    after another on this GPU (A already resident: the broadcast is the
    identity here, no rank waits on another), C panels assembled: bitwise the
    single-GPU call.  The NCCL path then only moves A (tests/test_multi.py
    covers the exchange with gloo)."""
    from paper_1609_00076_b200.multi import ShardedDgemm, make_shard_plan

    m, n, k = shape
    a, b, c, _ = dev_operands(torch_cuda, m, n, k)
    want = c.clone()
    run_dev(torch_cuda, m, n, k, a, m, b, k, want, m)  # the single call, its own path
    plan = make_shard_plan(m, n, k, world, root=0, k_chunk=256)
    for overlap in (False, True):  # whole-k GEMM / k-chunked GEMMs
        got = c.clone()
        for rank in range(world):
            j0, j1 = plan.local(rank)
            drv = ShardedDgemm(plan, rank, broadcast=lambda t, src: None, overlap=overlap)
            drv.step(a, m, b[j0 * k:], k, got[j0 * m:], m, broadcast_a=False)
        torch_cuda.cuda.synchronize()
        assert torch_cuda.equal(got, want), overlap


def test_device_flag_rejects_host_pointers(torch_cuda):
    a = np.ones(16)
    d = torch_cuda.ones(16, dtype=torch_cuda.float64, device="cuda")
    lib = _capi.load()
    st = lib.my_dgemm_ex(4, 4, 4, a.ctypes.data, 4, d.data_ptr(), 4, d.data_ptr(), 4, _capi.DEVICE_PTRS, None)
    assert st == -4 and "device pointer" in _capi.last_error()
    st = lib.my_dgemm_ex(4, 4, 4, d.data_ptr(), 4, d.data_ptr(), 4, a.ctypes.data, 4, _capi.DEVICE_PTRS, None)
    assert st == -8


@pytest.mark.parametrize("m,n,k", [(300, 257, 129), (2048, 2048, 512), (1280, 1280, 300)])
def test_cuda_graph_capture_and_replay(torch_cuda, m, n, k):
    """The device path is capture-safe: a CUDA graph of several my_dgemm_ex
    calls replays, twice, to the same result as eager calls -- small units,
    the stream-K schedule (workspace, zeroed flags and epoch baked into the
    graph) and stream-K over units."""
    torch = torch_cuda
    a, b, c, _ = dev_operands(torch, m, n, k)
    eager = c.clone()
    for _ in range(3):
        run_dev(torch, m, n, k, a, m, b, k, eager, m)
    graphed = c.clone()
    s = torch.cuda.Stream()
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, graphed.data_ptr(), m, s.cuda_stream)  # warm
    torch.cuda.synchronize()
    graphed.copy_(c)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, graphed.data_ptr(), m,
                                torch.cuda.current_stream().cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(graphed, eager)
    graphed.copy_(c)
    g.replay()  # the flags of the previous replay must not satisfy this one's waits
    torch.cuda.synchronize()
    assert torch.equal(graphed, eager)


@pytest.mark.timeout(300)
def test_stream_k_workspace_is_per_stream(torch_cuda):
    """Stream-K calls keep their partials and flags in a block owned by the
    call's stream (up to 8 streams per device; further streams take a pooled
    block with zeroed flags).  Ten streams issue interleaved stream-K calls
    (1280^3: stream-K over units; 1792 x 1664 x 512: full-tile stream-K) on
    their own C at the same time, twice over: every result is bitwise the
    single-stream one, so no call ever saw another stream's partials or a
    stale flag."""
    torch = torch_cuda
    shapes = [(1280, 1280, 1280), (1792, 1664, 512)]
    ops, want = [], []
    for (m, n, k) in shapes:
        a, b, c, _ = dev_operands(torch, m, n, k)
        w = c.clone()
        run_dev(torch, m, n, k, a, m, b, k, w, m)
        run_dev(torch, m, n, k, a, m, b, k, w, m)
        ops.append((m, n, k, a, b, c))
        want.append(w)
    streams = [torch.cuda.Stream() for _ in range(10)]
    outs = [[c.clone() for (_, _, _, _, _, c) in ops] for _ in streams]
    torch.cuda.synchronize()
    for rep in range(2):
        for si, st in enumerate(streams):
            for oi, (m, n, k, a, b, _) in enumerate(ops):
                engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, outs[si][oi].data_ptr(), m,
                                    st.cuda_stream)
    torch.cuda.synchronize()
    for si in range(len(streams)):
        for oi in range(len(ops)):
            assert torch.equal(outs[si][oi], want[oi]), (si, oi)


def test_more_than_2_31_elements_of_c(torch_cuda):
    """C with 2.15e9 elements (> 2^31: every index is 64-bit): fast path vs the
    exact kernel over the whole matrix within the headline bound, and the last
    column's last element against a CPU evaluation of the same operands."""
    m = n = 46341  # m * n = 2,147,488,281 > 2^31
    k = 16
    st = torch_cuda.cuda.current_stream().cuda_stream
    free, _ = torch_cuda.cuda.mem_get_info()
    if free < 4 * m * n * 8 + (1 << 30):
        pytest.skip("needs ~70 GB of free device memory")
    a = dev_matrix(torch_cuda, m, k, m, 101)
    b = dev_matrix(torch_cuda, k, n, k, 102)
    c0 = dev_matrix(torch_cuda, m, n, m, 103)
    cf = c0.clone()
    run_dev(torch_cuda, m, n, k, a, m, b, k, cf, m)
    bound = device_bound(torch_cuda, m, n, k, a, m, b, k, c0, m)
    torch_cuda.cuda.empty_cache()
    ce = c0
    run_dev(torch_cuda, m, n, k, a, m, b, k, ce, m, exact=True)
    check_dev(torch_cuda, m, n, k, cf, ce, m, bound)
    # last element, bitwise against the naive order evaluated on the host
    row = a.view(k, m)[:, m - 1].cpu().numpy()
    col = b.view(n, k)[n - 1].cpu().numpy()
    del cf
    want = float(dev_matrix(torch_cuda, m, n, m, 103)[(n - 1) * m + m - 1])
    for p in range(k):
        want = want + float(row[p]) * float(col[p])
    assert float(ce[(n - 1) * m + m - 1]) == want


@pytest.mark.parametrize("shape", [(2048, 2048, 2048), (1000, 1100, 700), (4093, 4099, 300)])
def test_back_to_back_dependent_calls_stream_ordered(torch_cuda, shape):
    """Consecutive calls on one stream with no host sync between them, each
    reading the previous call's output (RAW) or overwriting its input (WAR):
    programmatic dependent launch must keep stream semantics, including a
    call's early-starting tail launch.  Compared with the same chain run with
    a device sync after every call."""
    m, n, k = shape
    st = torch_cuda.cuda.current_stream().cuda_stream
    base = [dev_matrix(torch_cuda, r, c, r, 300 + t) for t, (r, c) in
            enumerate(((m, k), (k, n), (m, n), (m, n), (n, n)))]

    def chain(sync):
        a, b, c1, c2, b2 = (x.clone() for x in base)
        calls = [
            lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c1.data_ptr(), m, st),
            # RAW: c1 (just written) is the A operand
            lambda: engine.dgemm_device(m, n, n, c1.data_ptr(), m, b2.data_ptr(), n, c2.data_ptr(), m, st),
            # WAR: c1 (just read as A) is overwritten as C
            lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c1.data_ptr(), m, st),
            # RAW again, chained through c2
            lambda: engine.dgemm_device(m, n, n, c2.data_ptr(), m, b2.data_ptr(), n, c1.data_ptr(), m, st),
        ]
        for call in calls:
            call()
            if sync:
                torch_cuda.cuda.synchronize()
        torch_cuda.cuda.synchronize()
        return c1, c2

    want = chain(True)
    for _ in range(3):
        got = chain(False)
        assert torch_cuda.equal(got[0], want[0]) and torch_cuda.equal(got[1], want[1])


@pytest.mark.parametrize("shape", [(4093, 4099, 300), (2048, 2048, 512), (700, 900, 1000), (256, 256, 256)])
def test_sm_cap_changes_speed_never_results(torch_cuda, shape):
    """my_dgemm_set_max_ctas: the persistent grid on 100, 37 or 1 SMs gives
    bitwise the all-SM result (different plans and unit assignment, same
    per-element arithmetic); 256^3 runs on the small-block kernel without a
    cap and on the persistent grid under one."""
    m, n, k = shape
    a, b, c, _ = dev_operands(torch_cuda, m, n, k)
    want = c.clone()
    run_dev(torch_cuda, m, n, k, a, m, b, k, want, m)
    try:
        for cap in (100, 37, 1):
            engine.set_max_ctas(cap)
            got = c.clone()
            run_dev(torch_cuda, m, n, k, a, m, b, k, got, m)
            assert torch_cuda.equal(got, want), cap
    finally:
        engine.set_max_ctas(0)


def test_concurrent_host_threads_disjoint_c(torch_cuda):
    """Re-entrancy for disjoint C: host threads calling the
    host-pointer path and the device path (each on its own stream) at the
    same time get the results of sequential calls."""
    import threading

    shapes = [(700, 900, 500), (1024, 512, 768), (333, 1200, 257), (1500, 700, 900)]
    ops = [oracle.make_operands(SEED + i, *s) for i, s in enumerate(shapes)]
    want = [engine.my_dgemm(m, n, k, a, m, b, k, c.copy(), m) for (m, n, k), (a, b, c) in zip(shapes, ops)]
    dev = []
    for (m, n, k), (a, b, c) in zip(shapes, ops):
        dev.append(tuple(torch_cuda.from_numpy(x).cuda() for x in (a, b, c)))
    results, errors = {}, []

    def host_worker(i):
        try:
            (m, n, k), (a, b, c) = shapes[i], ops[i]
            for _ in range(3):
                results[("h", i)] = engine.my_dgemm(m, n, k, a, m, b, k, c.copy(), m)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    def dev_worker(i):
        try:
            (m, n, k) = shapes[i]
            a, b, c = dev[i]
            s = torch_cuda.cuda.Stream()
            with torch_cuda.cuda.stream(s):
                cc = c.clone()
                engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, cc.data_ptr(), m, s.cuda_stream)
                s.synchronize()
            results[("d", i)] = cc.cpu().numpy()
        except Exception as e:  # pragma: no cover
            errors.append(e)

    threads = [threading.Thread(target=host_worker, args=(i,)) for i in range(len(shapes))]
    threads += [threading.Thread(target=dev_worker, args=(i,)) for i in range(len(shapes))]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    for i in range(len(shapes)):
        assert np.array_equal(results[("h", i)], want[i]), i
        assert np.array_equal(results[("d", i)], want[i]), i


@pytest.mark.parametrize("m,n,k,lda,ldb,ldc", [
    (4096, 2, 3000, 4096, 3000, 4096),      # k split over CTAs, ordered fix-up
    (5000, 7, 1000, 5003, 1001, 5002),      # odd lds, ragged row block
    (8192, 16, 2048, 8192, 2048, 8195),
    (4100, 3, 100, 4100, 100, 4100),        # single k chunk
])
def test_few_columns_kernel(torch_cuda, m, n, k, lda, ldb, ldc):
    """2 <= n <= 16 with a tall A runs on the bandwidth kernel: within the
    headline bound of the exact kernel, deterministic, padding untouched;
    the BLAS epilogue (beta = 0 on a NaN-filled C) through the same kernel."""
    a, b, c, _ = dev_operands(torch_cuda, m, n, k, lda, ldb, ldc, canary=-777.25)
    cf, ce = c.clone(), c.clone()
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, cf, ldc)
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, ce, ldc, exact=True)
    bound = device_bound(torch_cuda, m, n, k, a, lda, b, ldb, c, ldc)
    check_dev(torch_cuda, m, n, k, cf, ce, ldc, bound)
    again = c.clone()
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, again, ldc)
    assert torch_cuda.equal(again, cf)
    host = cf.cpu().numpy().reshape(n, ldc)
    if ldc > m:
        assert np.all(host[:, m:] == -777.25)
    cn = torch_cuda.full_like(c, float("nan"))
    engine.dgemm("N", "N", m, n, k, 1.0, a.view(-1), lda, b.view(-1), ldb, 0.0, cn, ldc)
    torch_cuda.cuda.synchronize()
    prod = (cf - c).cpu().numpy().reshape(n, ldc)[:, :m]
    got = cn.cpu().numpy().reshape(n, ldc)[:, :m]
    assert np.all(np.isfinite(got)) and np.abs(got - prod).max() <= 2 * bound


@pytest.mark.parametrize("m,n,k,lda,ldb,ldc", [
    (4, 8192, 3000, 4, 3000, 4),
    (7, 5000, 1000, 9, 1003, 8),            # odd / padded lds, ragged column groups
    (16, 8192, 700, 16, 701, 19),
    (2, 4100, 100, 2, 100, 2),
])
def test_few_rows_kernel(torch_cuda, m, n, k, lda, ldb, ldc):
    """2 <= m <= 16 on the FMA few-row kernel (PATH_FEW_ROWS; the default up
    to m = 4): within the headline bound of the exact kernel, deterministic,
    padding untouched, and the BLAS epilogue (beta = 0 on a NaN-filled C)
    through the default path."""
    a, b, c, _ = dev_operands(torch_cuda, m, n, k, lda, ldb, ldc, canary=-777.25)
    cf, ce = c.clone(), c.clone()
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, cf, ldc, path=_capi.PATH_FEW_ROWS)
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, ce, ldc, exact=True)
    bound = device_bound(torch_cuda, m, n, k, a, lda, b, ldb, c, ldc)
    check_dev(torch_cuda, m, n, k, cf, ce, ldc, bound)
    again = c.clone()
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, again, ldc, path=_capi.PATH_FEW_ROWS)
    assert torch_cuda.equal(again, cf)
    if ldc > m:
        assert np.all(cf.cpu().numpy().reshape(n, ldc)[:, m:] == -777.25)
    cn = torch_cuda.full_like(c, float("nan"))
    engine.dgemm("N", "N", m, n, k, 1.0, a.view(-1), lda, b.view(-1), ldb, 0.0, cn, ldc)
    torch_cuda.cuda.synchronize()
    cd = c.clone()
    run_dev(torch_cuda, m, n, k, a, lda, b, ldb, cd, ldc)  # default path (m > 4: the DMMA row kernel)
    prod = (cd - c).cpu().numpy().reshape(n, ldc)[:, :m]
    got = cn.cpu().numpy().reshape(n, ldc)[:, :m]
    assert np.all(np.isfinite(got)) and np.abs(got - prod).max() <= 2 * bound


@pytest.mark.parametrize("m,n,k,lda,ldb,ldc", [
    (8, 8192, 3000, 8, 3000, 8),
    (16, 8192, 700, 16, 701, 19),           # odd ldb: 8-byte B loads
    (5, 5000, 1001, 9, 1004, 8),            # k % 4 == 1, ragged column blocks
    (12, 4100, 3, 12, 3, 12),               # k < 4: only the partial group
    (16, 33, 8192, 16, 8192, 16),           # one CTA, long k split over the warps
    (24, 2000, 515, 27, 516, 25),           # forced: 17..32 rows (4 row tiles)
    (32, 9000, 256, 32, 256, 32),
    (2, 3000, 64, 2, 64, 2),
])
def test_rows_dmma_kernel(torch_cuda, m, n, k, lda, ldb, ldc):
    """The DMMA row kernel (PATH_ROWS_DMMA; default for 5 <= m <= 16, forced
    up to 32 rows): within the headline bound of the exact kernel,
    deterministic, bitwise invariant to splitting the columns (what the
    sharded drivers rely on), padding untouched, and the BLAS epilogue
    (beta = 0 on a NaN-filled C) through it."""
    torch = torch_cuda
    P = _capi.PATH_ROWS_DMMA
    a, b, c, _ = dev_operands(torch, m, n, k, lda, ldb, ldc, canary=-777.25)
    cf, ce = c.clone(), c.clone()
    run_dev(torch, m, n, k, a, lda, b, ldb, cf, ldc, path=P)
    run_dev(torch, m, n, k, a, lda, b, ldb, ce, ldc, exact=True)
    bound = device_bound(torch, m, n, k, a, lda, b, ldb, c, ldc)
    check_dev(torch, m, n, k, cf, ce, ldc, bound)
    again = c.clone()
    run_dev(torch, m, n, k, a, lda, b, ldb, again, ldc, path=P)
    assert torch.equal(again, cf)
    # column shards (ragged widths, B and C views at column offsets) give the same bits
    split = c.clone()
    j0 = 0
    for w in (n // 3 + 1, 7, n):
        w = min(w, n - j0)
        if w <= 0:
            break
        engine.dgemm_device(m, w, k, a.data_ptr(), lda, b.data_ptr() + 8 * j0 * ldb, ldb,
                            split.data_ptr() + 8 * j0 * ldc, ldc, torch.cuda.current_stream().cuda_stream, path=P)
        j0 += w
    torch.cuda.synchronize()
    assert torch.equal(split, cf)
    if ldc > m:
        assert np.all(cf.cpu().numpy().reshape(n, ldc)[:, m:] == -777.25)
    if 5 <= m <= 16:
        assert engine.path(m, n) == P
        cd = c.clone()
        run_dev(torch, m, n, k, a, lda, b, ldb, cd, ldc)
        assert torch.equal(cd, cf)
        cn = torch.full_like(c, float("nan"))
        engine.dgemm("N", "N", m, n, k, 1.0, a.view(-1), lda, b.view(-1), ldb, 0.0, cn, ldc)
        torch.cuda.synchronize()
        prod = (cf - c).cpu().numpy().reshape(n, ldc)[:, :m]
        got = cn.cpu().numpy().reshape(n, ldc)[:, :m]
        assert np.all(np.isfinite(got)) and np.abs(got - prod).max() <= 2 * bound


def test_rows_dmma_keeps_negative_zero(torch_cuda):
    """C = -0, A = +0, B = -1: every product is -0 and the reference keeps
    -0 (acc = C, acc += a*b); the row kernel's accumulators start at -0, the
    additive identity, so -0 survives the slice sum and the add onto C."""
    torch = torch_cuda
    m, n, k = 12, 3000, 203
    a = torch.zeros(m * k, dtype=torch.float64, device="cuda")
    b = torch.full((k * n,), -1.0, dtype=torch.float64, device="cuda")
    c = torch.full((m * n,), -0.0, dtype=torch.float64, device="cuda")
    run_dev(torch, m, n, k, a, m, b, k, c, m, path=_capi.PATH_ROWS_DMMA)
    assert bool(torch.signbit(c).all())


@pytest.mark.parametrize("m,n,k,alpha,beta", [(2048, 2048, 512, 1.5, -0.5), (2048, 2304, 700, 2.0, 0.0),
                                               (1280, 1280, 300, -1.0, 1.0)])
@pytest.mark.parametrize("epilogue", [False, True])
def test_blas_epilogue_under_stream_k(torch_cuda, m, n, k, alpha, beta, epilogue):
    """alpha / beta through the stream-K schedule (these shapes' tiles do not
    fill the last wave).  Large tiled calls with beta != 0 default to the
    reference-BLAS order (C := beta C, alpha folded into an operand, then the
    accumulate contract), so `epilogue=True` (MY_DGEMM_BLAS_EPILOGUE) forces
    the kernel epilogue for every case: cut tiles carry the partial product
    from zero, the last segment applies alpha and beta once (reading C when
    beta != 0); beta = 0 never reads a NaN C on either route."""
    torch = torch_cuda
    a, b, c, _ = dev_operands(torch, m, n, k)
    cin = c.clone() if beta != 0 else torch.full_like(c, float("nan"))
    out = cin.clone()
    engine.dgemm("N", "N", m, n, k, alpha, a, m, b, k, beta, out, m, epilogue=epilogue)
    torch.cuda.synchronize()
    A = a.view(k, m).T
    B = b.view(n, k).T
    want = alpha * (A @ B) + (beta * c.view(n, m).T if beta != 0 else 0.0)
    got = out.view(n, m).T
    bound = HEADLINE_C * (k + 2) * EPS * (abs(alpha) * k + abs(beta))
    assert torch.isfinite(got).all()
    assert float((got - want).abs().max()) <= bound


def _fuzz_shapes(seed, count):
    """Seeded random shapes spanning every kernel family: m or n of 1, few
    rows / columns, ragged tiles, short and long k, padded / odd lds."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        kind = rng.integers(0, 6)
        if kind == 0:
            m, n = 1, int(rng.integers(1, 3000))
        elif kind == 1:
            m, n = int(rng.integers(1, 3000)), 1
        elif kind == 2:
            m, n = int(rng.integers(2, 17)), int(rng.integers(16, 6000))
        elif kind == 3:
            m, n = int(rng.integers(4096, 9000)), int(rng.integers(2, 17))
        else:
            m, n = int(rng.integers(1, 1500)), int(rng.integers(1, 1500))
        k = int(rng.choice([1, 3, 15, 16, 17, 64, 255, 256, 700, 1031, 2048]))
        pads = [int(p) for p in rng.integers(0, 9, size=3)]
        out.append((m, n, k, m + pads[0], k + pads[1], m + pads[2]))
    return out


@pytest.mark.parametrize("seed", [11, 12, 13, 14])
def test_fuzz_random_shapes_fast_vs_exact(torch_cuda, seed):
    """Random shapes (seeded): the default path (whatever kernel family and
    plan it picks) within the headline bound of the bitwise-oracle exact
    kernel, every full-tile plan bitwise equal to the default tiled call, and
    padding canaries intact."""
    torch = torch_cuda
    for (m, n, k, lda, ldb, ldc) in _fuzz_shapes(seed, 40):
        a, b, c, _ = dev_operands(torch, m, n, k, lda, ldb, ldc, canary=-777.25)
        fast, exact = c.clone(), c.clone()
        run_dev(torch, m, n, k, a, lda, b, ldb, fast, ldc)
        run_dev(torch, m, n, k, a, lda, b, ldb, exact, ldc, exact=True)
        bound = device_bound(torch, m, n, k, a, lda, b, ldb, c, ldc)
        check_dev(torch, m, n, k, fast, exact, ldc, bound)
        if ldc > m:
            assert bool((fast.view(n, ldc)[:, m:] == -777.25).all()), (m, n, k)
        tiled = []
        for strips in (0, 2, 8, 32):
            cc = c.clone()
            run_dev(torch, m, n, k, a, lda, b, ldb, cc, ldc, strips=strips, force_tiled=True)
            tiled.append(cc)
        assert all(torch.equal(tiled[0], t) for t in tiled[1:]), (m, n, k, lda, ldb, ldc)


@pytest.mark.parametrize("m,n,k,lds", [(300, 260, 100, (300, 100, 300)), (257, 300, 20, (257, 21, 259)),
                                       (1024, 1024, 1028, (1024, 1028, 1024))])
def test_signed_zero_is_plan_invariant_and_matches_the_oracle(torch_cuda, m, n, k, lds):
    """C = -0, A = +0, B = -1: every real product is -0, so the reference's
    loop (acc = acc + a*b from acc = C) keeps -0.  K is ragged, so the last
    K slab carries all-zero k-steps; the kernels skip them in every unit
    shape and plan (computing them would turn -0 into +0), so every plan
    returns -0 everywhere, bitwise the exact kernel."""
    torch = torch_cuda
    lda, ldb, ldc = lds
    a = torch.zeros(lda * k, dtype=torch.float64, device="cuda")
    b = torch.full((ldb * n,), -1.0, dtype=torch.float64, device="cuda")
    c = torch.full((ldc * n,), -0.0, dtype=torch.float64, device="cuda")
    ce = c.clone()
    run_dev(torch, m, n, k, a, lda, b, ldb, ce, ldc, exact=True)
    assert bool(torch.signbit(ce.view(n, ldc)[:, :m]).all())
    for strips in (0, 2, 4, 8, 16, 32, 34, 36, 40) + SMALL_PLANS:
        cc = c.clone()
        run_dev(torch, m, n, k, a, lda, b, ldb, cc, ldc, strips=strips, force_tiled=True)
        assert bool(torch.signbit(cc.view(n, ldc)[:, :m]).all()), strips


# ------------------------------------------- the device checker's own controls


def _host_report(got, want, m, n, ld, tol):
    return oracle.max_abs_diff(got.cpu().numpy(), want.cpu().numpy(), m, n, ld, tol=tol)


def _same_report(dev, host):
    same_max = (dev.max_abs_diff == host.max_abs_diff
                or (dev.max_abs_diff != dev.max_abs_diff and host.max_abs_diff != host.max_abs_diff))
    assert same_max, (dev, host)
    assert (dev.first_bad_i, dev.first_bad_j) == (host.first_bad_i, host.first_bad_j), (dev, host)
    if not host.clean:
        assert np.array_equal(np.float64(dev.value_got), np.float64(host.value_got), equal_nan=True)
        assert dev.value_expected == host.value_expected
        assert (engine.failure_line(dev.first_bad_i, dev.first_bad_j, dev.value_got, dev.value_expected)
                == oracle.failure_line(host.first_bad_i, host.first_bad_j, host.value_got, host.value_expected))


TOL = 2.0**-30


def _plants(m, n):
    """Planted (i, j, kind) mismatch sets; kinds: 'at' = difference exactly
    the tolerance (not an offender under the strict > rule), 'above' = one ulp
    of 0.5 past it, 'big', 'nan', 'inf'.  Positions: first and last element,
    a 128-row tile boundary, an 8-way jc shard boundary, the last column."""
    sh = (n // 8) if n >= 8 else n - 1
    return {
        "first": [(0, 0, "big")],
        "last": [(m - 1, n - 1, "big")],
        "tile_edge": [(127, 1, "at"), (128, 1, "above"), (m - 1, n - 1, "big")],
        "shard_edge": [(0, sh - 1, "at"), (5, sh, "above")],
        "just_above_after_at": [(3, 0, "at"), (4, 0, "at"), (m - 2, n - 1, "above")],
        "only_at": [(1, 1, "at"), (m - 1, n - 1, "at")],
        "nan_only": [(7, 2, "nan")],
        "nan_then_above": [(2, 0, "nan"), (9, n - 1, "above")],
        "inf": [(m // 2, n // 2, "inf")],
        "clean": [],
    }


@pytest.mark.parametrize("m,n,ld", [(1000, 777, 1003), (4096, 8192, 4096)])
@pytest.mark.parametrize("case", list(_plants(1000, 777)))
def test_device_checker_negative_control(torch_cuda, m, n, ld, case):
    """my_dgemm_diff_report (the checker every full-matrix GPU parity test
    relies on) against oracle.max_abs_diff (matrix.py:210-232) on planted
    mismatches: same max (NaN included), same first offender in column-major
    order under the strict > tol rule, same offender values and the same
    reference failure line (bench.py:84-86); verify_device raises with that
    line, or on a NaN max.  A checker stubbed to 'clean' fails every
    case but 'clean' and 'only_at'."""
    torch = torch_cuda
    want = dev_matrix(torch, m, n, ld, 5, canary=-777.25)
    got = want.clone()
    for i, j, kind in _plants(m, n)[case]:
        t = j * ld + i
        want[t] = 0.5
        got[t] = {"at": 0.5 + TOL, "above": 0.5 + TOL + 2.0**-53, "big": 3.0,
                  "nan": float("nan"), "inf": float("inf")}[kind]
    dev = engine.diff_report_device(m, n, got.data_ptr(), ld, want.data_ptr(), ld, TOL)
    host = _host_report(got, want, m, n, ld, TOL)
    _same_report(dev, host)
    expect_bad = [(i, j) for i, j, kind in _plants(m, n)[case] if kind in ("above", "big", "inf")]
    if expect_bad:
        first = min(expect_bad, key=lambda p: p[1] * m + p[0])
        assert (dev.first_bad_i, dev.first_bad_j) == first
        with pytest.raises(engine.VerificationError) as ei:
            engine.verify_device(m, n, 7, got.data_ptr(), ld, want.data_ptr(), ld, TOL)
        assert ei.value.diagnostic == oracle.failure_line(host.first_bad_i, host.first_bad_j, host.value_got,
                                                          host.value_expected)
        assert ei.value.diagnostic.startswith(f"C[ {first[0]} ][ {first[1]} ] != C_ref, ")
    else:
        assert dev.clean
        if case.startswith("nan"):
            assert dev.max_abs_diff != dev.max_abs_diff
            with pytest.raises(engine.VerificationError, match="NaN"):
                engine.verify_device(m, n, 7, got.data_ptr(), ld, want.data_ptr(), ld, TOL)
        else:
            engine.verify_device(m, n, 7, got.data_ptr(), ld, want.data_ptr(), ld, TOL)
    # the canaries in the padding rows never enter the comparison
    if ld > m:
        got.view(n, ld)[:, m:] = 1e300
        again = engine.diff_report_device(m, n, got.data_ptr(), ld, want.data_ptr(), ld, TOL)
        assert (again.first_bad_i, again.first_bad_j) == (dev.first_bad_i, dev.first_bad_j)


def test_device_checker_tolerance_zero_finds_first_difference(torch_cuda):
    """tol = 0 (the reference default): the first differing element."""
    torch = torch_cuda
    m, n = 300, 200
    want = dev_matrix(torch, m, n, m, 6)
    got = want.clone()
    got[77 * m + 150] = float(got[77 * m + 150]) * (1 + 2.0**-50)
    got[150 * m + 3] += 1.0
    dev = engine.diff_report_device(m, n, got.data_ptr(), m, want.data_ptr(), m, 0.0)
    assert (dev.first_bad_i, dev.first_bad_j) == (150, 77)
    _same_report(dev, _host_report(got, want, m, n, m, 0.0))


# ------------------------------ every timed point of the cfg2 sweep, full matrix

CFG2_SIZES = list(range(256, 8192 + 1, 256))


@pytest.mark.parametrize("s", CFG2_SIZES)
def test_cfg2_sweep_point_exact_kat_and_fast_full(torch_cuda, golden, s):
    """Every size the sweep times (BASELINE configs[1]; the reference's
    run_sweep verifies every timed shape, bench.py:140-156): the exact kernel
    reproduces the reference's C bit for bit (SHA-256 of C from
    gemm_goto_parallel, tests/golden/make_golden.py), and every element of
    the fast result lies within the headline bound (c = 2, magnitude on the
    device) of it."""
    torch = torch_cuda
    kat = golden["kat"]["cfg1" if s == 512 else f"cfg2_{s}"]
    assert (kat["m"], kat["n"], kat["k"]) == (s, s, s)
    a, b, c, _ = dev_operands(torch, s, s, s)
    bound = device_bound(torch, s, s, s, a, s, b, s, c, s)
    fast, exact = c.clone(), c
    run_dev(torch, s, s, s, a, s, b, s, fast, s)
    run_dev(torch, s, s, s, a, s, b, s, exact, s, exact=True)
    assert oracle.sha256_valid(exact.cpu().numpy(), s, s, s) == kat["sha256"]
    check_dev(torch, s, s, s, fast, exact, s, bound)


def test_tile_grid_tuner_pins_a_verified_winner(torch_cuda):
    """tune_grid (the reference's tune, bench.py:238-311): every timed point is
    verified against the exact kernel, blocks larger than the probe are
    skipped with a warning, the winner is pinned for the probe shape
    (my_dgemm_tune_set) and later calls of the shape are bitwise what the
    heuristic plan gives."""
    import io

    from paper_1609_00076_b200 import tuning

    _capi.load().my_dgemm_tune_clear()
    log = io.StringIO()
    try:
        res = tuning.tune_grid({}, probe_size=96, reps=2, log=log)
        assert res.table and res.rate > 0 and res.best in res.table
        assert res.rate == max(res.table.values())
        assert all(p.bm <= 96 and p.bn <= 96 for p in res.table)
        assert "block sizes exceed probe size 96" in log.getvalue()  # the 128-row units
        m = n = k = 96
        a, b, c, _ = dev_operands(torch_cuda, m, n, k)
        tuned = c.clone()
        run_dev(torch_cuda, m, n, k, a, m, b, k, tuned, m)  # uses the pinned plan
        _capi.load().my_dgemm_tune_clear()
        heur = c.clone()
        run_dev(torch_cuda, m, n, k, a, m, b, k, heur, m)
        assert torch_cuda.equal(tuned, heur)
    finally:
        _capi.load().my_dgemm_tune_clear()
