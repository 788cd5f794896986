"""The drop-in boundary without a GPU: the library builds, loads, exports every
symbol include/my_dgemm.h declares, and rejects bad arguments before touching
any memory (reference ValueError semantics, kernels.py:41-49,
matrix.py:50-53, goto.py:196-204).  No compute is launched here."""

import ctypes
import os
import re
import sys

import numpy as np
import pytest

from paper_1609_00076_b200 import _capi, build, engine

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "my_dgemm.h")


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _capi.load()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"MY_DGEMM_API\s+[\w\s\*]+?\b(\w+)\s*\(", text)))


def test_header_declares_the_baseline_signature():
    text = open(HEADER).read()
    assert re.search(r"void my_dgemm\(int m, int n, int k, const double \*A, int lda, "
                     r"const double \*B, int ldb, double \*C, int ldc\);", text)


def test_library_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert "my_dgemm" in syms and len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _capi.SIGNATURES, f"{s} not typed in _capi.SIGNATURES"
    # nothing beyond the ABI is exported
    out = os.popen(f"nm -D --defined-only {_capi.LIB_PATH}").read()
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert exported == set(syms)


def test_library_is_sm100a(lib):
    out = os.popen(f"cuobjdump --list-elf {_capi.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    sass = os.popen(f"cuobjdump -sass {_capi.LIB_PATH} 2>&1 | grep -c DMMA").read().strip()
    assert int(sass or 0) > 0, "fast kernel must issue DMMA (FP64 tensor pipe)"


def test_version_and_counters(lib):
    assert b"sm_100a" in lib.my_dgemm_version()
    assert lib.my_dgemm_kernel_launches() >= 0


BAD = [
    # (m, n, k, lda, ldb, ldc, null index, expected status)
    (0, 4, 4, 4, 4, 4, None, -1),
    (4, 0, 4, 4, 4, 4, None, -2),
    (4, 4, 0, 4, 4, 4, None, -3),
    (4, 4, 4, 4, 4, 4, 0, -4),
    (4, 4, 4, 3, 4, 4, None, -5),
    (4, 4, 4, 4, 4, 4, 1, -6),
    (4, 4, 4, 4, 3, 4, None, -7),
    (4, 4, 4, 4, 4, 4, 2, -8),
    (4, 4, 4, 4, 4, 3, None, -9),
]


@pytest.mark.parametrize("m,n,k,lda,ldb,ldc,null,status", BAD)
def test_invalid_arguments_status_and_untouched_c(lib, m, n, k, lda, ldb, ldc, null, status):
    bufs = [np.full(64, 1.5), np.full(64, 2.5), np.full(64, 3.5)]
    ptrs = [b.ctypes.data for b in bufs]
    if null is not None:
        ptrs[null] = None
    got = lib.my_dgemm_ex(m, n, k, ptrs[0], lda, ptrs[1], ldb, ptrs[2], ldc, 0, None)
    assert got == status
    assert lib.my_dgemm_last_status() == status
    assert np.all(bufs[2] == 3.5) and np.all(bufs[0] == 1.5)
    # void entry point records the same status
    lib.my_dgemm(m, n, k, ptrs[0], lda, ptrs[1], ldb, ptrs[2], ldc)
    assert lib.my_dgemm_last_status() == status


def test_unknown_flags_rejected(lib):
    a = np.zeros(16)
    assert lib.my_dgemm_ex(4, 4, 4, a.ctypes.data, 4, a.ctypes.data, 4, a.ctypes.data, 4,
                           0x1000, None) == -10


def test_python_boundary_raises_reference_valueerrors(lib):
    a = engine.alloc_matrix(3, 4)
    b = engine.alloc_matrix(5, 2)
    c = engine.alloc_matrix(3, 2)
    with pytest.raises(ValueError, match="inner dims differ: A is 3x4, B is 5x2"):
        engine.gemm_b200(a, b, c)
    b = engine.alloc_matrix(4, 2)
    with pytest.raises(ValueError, match="C is 3x3, expected 3x2"):
        engine.gemm_b200(a, b, engine.alloc_matrix(3, 3))
    with pytest.raises(ValueError, match="leading dimension ld=2 smaller than row count m=3"):
        engine.Matrix(3, 2, 2, np.zeros(8))
    with pytest.raises(ValueError, match="buffer too small"):
        engine.Matrix(3, 2, 5, np.zeros(7))
    engine.Matrix(3, 2, 5, np.zeros(8))  # exact corner view is legal (matrix.py:58)
    with pytest.raises(ValueError, match="matrix dims must be positive"):
        engine.my_dgemm(0, 1, 1, np.zeros(1), 1, np.zeros(1), 1, np.zeros(1), 1)
    with pytest.raises(ValueError, match="buffer too small"):
        engine.my_dgemm(4, 4, 4, np.zeros(15), 4, np.zeros(16), 4, np.zeros(16), 4)


def test_operand_seed_matches_oracle(lib):
    import oracle

    for s in [(42, 1, 512, 512, 512), (42, 3, 4093, 4099, 2047), ((1 << 64) - 1, 2, 1, 1, 1)]:
        assert engine.operand_seed(*s) == oracle.operand_seed(*s)


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    monkeypatch.setattr(_capi, "_lib", None)
    with pytest.raises(_capi.NativeLibraryError):
        _capi.load(str(tmp_path / "absent.so"))


BLAS_BAD = [
    # (transa, transb, m, n, k, lda, ldb, ldc, status)
    ("X", "N", 4, 4, 4, 4, 4, 4, -1),
    ("N", "Q", 4, 4, 4, 4, 4, 4, -2),
    ("N", "N", -1, 4, 4, 4, 4, 4, -3),
    ("N", "N", 4, -1, 4, 4, 4, 4, -4),
    ("N", "N", 4, 4, -1, 4, 4, 4, -5),
    ("N", "N", 4, 4, 4, 3, 4, 4, -8),
    ("T", "N", 4, 4, 5, 4, 5, 4, -8),    # A^T: A is k x m, lda >= k
    ("N", "N", 4, 4, 4, 4, 3, 4, -10),
    ("N", "T", 4, 5, 4, 4, 4, 4, -10),   # B^T: B is n x k, ldb >= n
    ("N", "N", 4, 4, 4, 4, 4, 3, -13),
]


@pytest.mark.parametrize("ta,tb,m,n,k,lda,ldb,ldc,status", BLAS_BAD)
def test_blas_argument_checks_reference_order(lib, ta, tb, m, n, k, lda, ldb, ldc, status):
    c = np.full(64, 3.5)
    a = np.ones(64)
    got = lib.my_dgemm_blas(ta.encode(), tb.encode(), m, n, k, 1.0, a.ctypes.data, lda, a.ctypes.data, ldb, 1.0,
                            c.ctypes.data, ldc, 0, None)
    assert got == status
    assert np.all(c == 3.5)


def test_blas_quick_returns_touch_nothing(lib):
    c = np.full(16, 3.5)
    # m == 0, n == 0, or (alpha == 0 or k == 0) with beta == 1: no memory touched, no device needed
    assert lib.my_dgemm_blas(b"N", b"N", 0, 4, 4, 1.0, None, 1, None, 4, 1.0, None, 1, 0, None) == 0
    assert lib.my_dgemm_blas(b"N", b"N", 4, 0, 4, 1.0, None, 4, None, 4, 1.0, None, 4, 0, None) == 0
    assert lib.my_dgemm_blas(b"N", b"N", 4, 4, 4, 0.0, None, 4, None, 4, 1.0, c.ctypes.data, 4, 0, None) == 0
    assert lib.my_dgemm_blas(b"N", b"N", 4, 4, 0, 2.0, None, 4, None, 1, 1.0, c.ctypes.data, 4, 0, None) == 0
    assert np.all(c == 3.5)
    with pytest.raises(ValueError, match="EXACT"):
        engine.dgemm("N", "N", 2, 2, 2, 2.0, np.ones(4), 2, np.ones(4), 2, 1.0, np.ones(4), 2, exact=True)


def test_multi_argument_checks_shifted_indices(lib):
    """my_dgemm_multi(ngpu, ...) / my_dgemm_multi_ex(devices, ndev, ...):
    status -i names the first bad argument, C untouched (no GPU here, so a
    structurally valid call fails on device visibility)."""
    import ctypes

    c = np.full(16, 3.5)
    a = np.ones(16)
    p = a.ctypes.data
    assert lib.my_dgemm_multi(0, 4, 4, 4, p, 4, p, 4, c.ctypes.data, 4) == -1
    assert lib.my_dgemm_multi(1, 0, 4, 4, p, 4, p, 4, c.ctypes.data, 4) == -2
    assert lib.my_dgemm_multi(1, 4, 4, 4, p, 3, p, 4, c.ctypes.data, 4) == -6
    assert lib.my_dgemm_multi(1, 4, 4, 4, p, 4, p, 4, None, 4) == -9
    devs = (ctypes.c_int * 2)(0, 0)
    assert lib.my_dgemm_multi_ex(None, 2, 4, 4, 4, p, 4, p, 4, c.ctypes.data, 4, 0) == -1
    assert lib.my_dgemm_multi_ex(devs, 0, 4, 4, 4, p, 4, p, 4, c.ctypes.data, 4, 0) == -2
    assert lib.my_dgemm_multi_ex(devs, 2, 4, 4, 0, p, 4, p, 4, c.ctypes.data, 4, 0) == -5
    assert lib.my_dgemm_multi_ex(devs, 2, 4, 4, 4, p, 4, p, 4, c.ctypes.data, 3, 0) == -11
    assert lib.my_dgemm_multi_ex(devs, 2, 4, 4, 4, p, 4, p, 4, c.ctypes.data, 4, 0x4) == -12
    import torch

    if not torch.cuda.is_available():
        assert lib.my_dgemm_multi(1, 4, 4, 4, p, 4, p, 4, c.ctypes.data, 4) == -1
        assert lib.my_dgemm_multi_ex(devs, 2, 4, 4, 4, p, 4, p, 4, c.ctypes.data, 4, 0) == -2
        assert "not visible" in lib.my_dgemm_last_error().decode()
    assert np.all(c == 3.5)


def test_set_max_ctas_roundtrip(lib):
    """my_dgemm_set_max_ctas: returns the previous cap, rejects n < 0."""
    prev = lib.my_dgemm_set_max_ctas(100)
    assert prev == 0
    assert lib.my_dgemm_set_max_ctas(0) == 100
    assert lib.my_dgemm_set_max_ctas(-3) == -1
    assert "max_ctas" in lib.my_dgemm_last_error().decode()
    assert lib.my_dgemm_set_max_ctas(0) == 0


FP = [(p + 1) << 8 for p in range(7)]  # MY_DGEMM_FORCE_PATH(p)


@pytest.mark.parametrize("m,n,flags,want", [
    (8192, 8192, 0, 0), (8192, 1, 0, 1), (1, 8192, 0, 2), (1, 1, 0, 2), (8192, 16, 0, 3), (4095, 16, 0, 0),
    (8192, 17, 0, 0), (4, 65536, 0, 4), (4, 65537, 0, 0), (5, 4096, 0, 6), (8, 4097, 0, 6), (2, 3, 0, 4),
    (9, 8192, 0, 6), (16, 100000, 0, 6), (17, 8192, 0, 0), (8, 1, 0, 1), (4, 1, 0, 4), (100, 1, 0, 1),
    (8192, 1, 0x4, 0), (4, 4, 0x4, 0), (4, 4, 0x2, 5),
    (8192, 1, FP[0], 0), (100, 1, FP[1], 1), (1, 50, FP[2], 2), (9000, 12, FP[3], 3), (16, 99999, FP[4], 4),
    (32, 7, FP[6], 6), (2, 9999, FP[6], 6),
    (100, 2, FP[1], -3), (2, 100, FP[2], -3), (100, 17, FP[3], -3), (17, 100, FP[4], -3), (33, 100, FP[6], -3),
])
def test_path_kind_rules(lib, m, n, flags, want):
    """my_dgemm_path: which kernel family a shape runs on (0 tiled, 1 n == 1,
    2 m == 1, 3 few columns, 4 few rows (FMA), 5 exact, 6 few rows (DMMA); FORCE_TILED = 0x4;
    MY_DGEMM_FORCE_PATH(p) forces a family that suits the shape, else -3)."""
    assert lib.my_dgemm_path(m, n, flags) == want
    assert lib.my_dgemm_path(0, n, flags) == -1


def test_forced_path_must_suit_the_shape(lib):
    a = np.zeros(64)
    p = a.ctypes.data
    assert lib.my_dgemm_ex(4, 4, 4, p, 4, p, 4, p, 4, FP[1], None) == -10
    assert "FORCE_PATH" in lib.my_dgemm_last_error().decode()


def test_diagnostics_mirror_the_reference():
    """engine.failure_line / DiffReport / VerificationError restate
    bench.py:74-86 and matrix.py:90-107; checked against the reference
    package itself when oracle/_ref holds it, else against the oracle."""
    from paper_1609_00076_b200 import engine
    import oracle

    cases = [(0, 0, 1.0, 2.0), (127, 4096, -3.25e-17, float("inf")), (5, 7, float("nan"), 0.0)]
    ref_line = oracle.failure_line
    ref = os.path.join(REPO, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "gemmforge")):
        sys.path.insert(0, ref)
        try:
            from gemmforge.bench import VerificationError as RefVE, failure_line as ref_line  # noqa: F811
            assert issubclass(engine.VerificationError, RuntimeError) and issubclass(RefVE, RuntimeError)
        finally:
            sys.path.remove(ref)
    for c in cases:
        assert engine.failure_line(*c) == ref_line(*c)
    rep = engine.DiffReport(0.5)
    assert rep.clean and rep.first_bad_i is None
    rep = engine.DiffReport(0.5, 3, 4, 1.0, 0.5)
    assert not rep.clean
    e = engine.VerificationError("C[ 1 ][ 2 ] != C_ref, 1E0, 2E0", m=3, n=4, k=5, algorithm="b200")
    assert (e.diagnostic, e.m, e.n, e.k, e.algorithm) == ("C[ 1 ][ 2 ] != C_ref, 1E0, 2E0", 3, 4, 5, "b200")


def test_plan_geometry_is_the_compiled_tile_table(lib):
    """my_dgemm_plan_geometry reports every launch plan's blocking parameters
    (no GPU needed): the persistent kernel's unit shapes and the small-block
    kernel's variant table; unknown plans are -1."""
    from paper_1609_00076_b200 import tuning

    full_long = tuning.plan_geometry(1, 8192)
    assert (full_long.bm, full_long.bn, full_long.bk) == (128, 128, 32) and full_long.stages >= 3
    assert tuning.plan_geometry(1, 256).bk == 16  # short K: 16-deep slabs
    assert tuning.plan_geometry(1, 8192, vec2=False).bk == 16
    assert tuning.plan_geometry(36, 512).key[:2] == (128, 32)  # stream-K over 128x32 units
    assert tuning.plan_geometry(16, 512).key[:2] == (16, 128)
    assert tuning.plan_geometry(48, 512) is None and tuning.plan_geometry(75, 512) is None
    small = [tuning.plan_geometry(p, 512) for p in range(65, 75)]
    assert all(p is not None for p in small)
    assert (small[0].bm, small[0].bn, small[0].bk, small[0].stages) == (16, 16, 32, 4)
    for p in small + [full_long]:  # every ring fits the 227 KB opt-in shared memory
        assert p.footprint * 8 <= 232448


def test_tile_grid_expansion_and_tie_break(lib):
    """tune_grid's validation (bench.py:258-272 analogue): a fully specified
    grid point no instantiation carries is skipped with a reason, a partial
    grid keeps every compiled plan on its axes, and exact rate ties prefer
    the smaller footprint (bench.py:304-311)."""
    from paper_1609_00076_b200 import tuning

    pts, skipped = tuning.grid_points({"bm": [16, 32], "bn": [16], "bk": [32, 48], "stages": [4]}, 512)
    assert {p.key for p in pts} == {(16, 16, 32, 4), (32, 16, 32, 4)}
    assert {s[0] for s in skipped} == {(16, 16, 48, 4), (32, 16, 48, 4)}
    assert all("no compiled instantiation" in s[1] for s in skipped)
    pts, skipped = tuning.grid_points({"bm": [128]}, 4096)
    assert pts and all(p.bm == 128 for p in pts) and not skipped
    assert {p.plan for p in pts} >= {1, 2, 4, 32, 34, 36}
    with pytest.raises(ValueError):
        tuning.grid_points({"mc": [64]}, 512)
    a = tuning.TilePoint(64, 64, 16, 6, 69)
    b = tuning.TilePoint(32, 32, 32, 4, 67)
    assert tuning._beats(10.0, b, 10.0, a)  # smaller footprint wins the tie
    assert not tuning._beats(10.0, a, 10.0, b)
    assert tuning._beats(10.5, a, 10.0, b)


# ------------------------------------------------------------------ the planner, as data (no GPU)

def test_planner_picks_the_measured_plans_for_the_baseline_shapes(lib):
    """my_dgemm_plan_describe runs the planner (host code) without launching:
    the picks the B200 measurements back (DESIGN 4c, profiles/r02/) are pinned
    here so a change to the cost model that flips one is seen on CPU.  The
    reference's make_plan (parallel.py:60-105) is likewise tested as data."""
    from paper_1609_00076_b200 import tuning

    d = tuning.describe_plan
    # cfg4 (16384^2 x 256): whole-tile rounds -- every tile in the stream-K phase measured 4.05 ms vs 3.93
    p = d(16384, 16384, 256)
    assert p["kind"] == "units" and p["split"] == 1 or (p["kind"] == "stream-K" and p["sk_dp_rounds"] >= 100)
    # cfg5 and cfg2@8192: whole-tile rounds, the last one to two waves as a stream-K tail
    p = d(32768, 32768, 32768)
    assert p["kind"] == "stream-K" and p["sk_split"] == 1 and p["sk_dp_rounds"] == 32768 // 128 * (32768 // 128) // 148 - 1
    p = d(8192, 8192, 8192)
    assert p["kind"] == "stream-K" and p["sk_split"] == 1 and p["sk_dp_rounds"] == 26
    assert abs(p["model_us"] / 30050.0 - 1.0) < 0.02  # the model's absolute level (measured 30.0-30.1 ms)
    # below one wave: stream-K over 128x32 units at 1024^3 (72.7 us vs 77.1 as 128x64 units)
    p = d(1024, 1024, 1024)
    assert (p["kind"], p["sk_split"]) == ("stream-K", 4) and abs(p["model_us"] / 72.0 - 1.0) < 0.05
    # 2.2 waves, long K: every tile in the stream-K phase (696 us vs 715 after a whole-tile round)
    p = d(2304, 2304, 2304)
    assert (p["kind"], p["sk_split"], p["sk_dp_rounds"]) == ("stream-K", 1, 0)
    # several waves at K = 128: 128x64 units (78.3 us), not full tiles (93.8 us)
    p = d(5376, 1536, 128)
    assert (p["kind"], p["split"]) == ("units", 2)
    # cfg1: one round of 64x32 units; the sub-wave cfg2 point and cfg3d: the small-block kernel
    p = d(512, 512, 512)
    assert (p["kind"], p["split"]) == ("units", 8)
    assert d(256, 256, 256)["kind"] == "small" and d(37, 53, 71, 44, 76, 40)["kind"] == "small"
    # cfg3a: whole-tile rounds with the ragged last tile column run as strips in the tail launch
    p = d(4093, 4099, 2047, 4100, 2052, 4096)
    assert p["kind"] == "units" and p["edge"] >= 1 and p["q"] == 6


def test_planner_never_picks_the_k_split_plan_unasked(lib):
    """The K-split plan is the one plan that is not plan-invariant: the
    heuristic (plan 0) must never choose it unless MY_DGEMM_KSPLIT=1, the
    plan-invariant heuristic (-1, what shards run) is the same choice, and
    pinning it (48) works only where the shape allows."""
    from paper_1609_00076_b200 import tuning

    assert os.environ.get("MY_DGEMM_KSPLIT", "0") in ("", "0")
    for s in range(256, 4097, 128):
        for (m, n, k) in ((s, s, s), (s, 2 * s, 640), (s + 5, s, 2047)):
            a, b = tuning.describe_plan(m, n, k), tuning.describe_plan(m, n, k, plan=-1)
            assert a["kind"] != "K-split" and a["text"] == b["text"], (m, n, k)
    assert tuning.describe_plan(1024, 1024, 1024, plan=48)["kind"] == "K-split"
    assert tuning.describe_plan(8192, 8192, 8192, plan=48)["kind"] != "K-split"  # more tiles than SMs
    assert tuning.describe_plan(768, 640, 96, plan=48)["kind"] != "K-split"      # fewer than two slabs per CTA
    with pytest.raises(ValueError):
        tuning.describe_plan(0, 4, 4)
