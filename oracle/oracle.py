"""ctypes front end of oracle/liboracle.so plus the reference's host-side
measurement helpers, restated.  TEST INFRASTRUCTURE ONLY (see __init__.py).

Citations are relative to /root/reference/pkg/src/gemmforge/.

Parity pin: tests/test_oracle.py checks every function here against the
reference tests' golden values (tests/test_matrix.py:42-52) and against the
fixtures in tests/golden/, which tests/golden/make_golden.py produced by
importing and running the reference package itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

__all__ = [
    "lib",
    "mix64",
    "random_values",
    "values_at",
    "operand_seed",
    "fill",
    "alloc",
    "make_operands",
    "make_padded_operands",
    "naive",
    "naive_par",
    "goto",
    "pack_a",
    "pack_b",
    "tolerance",
    "headline_tolerance",
    "DiffReport",
    "max_abs_diff",
    "failure_line",
    "valid_region",
    "sha256_valid",
    "sampled_reference",
    "host_threads",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_P = ctypes.c_void_p
_I = ctypes.c_int64
_U = ctypes.c_uint64


def _load():
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
        os.path.join(_HERE, "oracle.c")
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    L = ctypes.CDLL(_SO)  # CDLL: the GIL is released during calls
    L.oracle_mix64.argtypes = [_U]
    L.oracle_mix64.restype = _U
    L.oracle_random_values.argtypes = [_U, _I, _I, _P]
    L.oracle_values_at.argtypes = [_U, _P, _I, _P]
    L.oracle_fill.argtypes = [_P, _I, _I, _I, _U]
    L.oracle_operand_seed.argtypes = [_U, _U, _I, _I, _I]
    L.oracle_operand_seed.restype = _U
    L.oracle_naive.argtypes = [_I, _I, _I, _P, _I, _P, _I, _P, _I]
    L.oracle_naive_par.argtypes = [_I, _I, _I, _P, _I, _P, _I, _P, _I, ctypes.c_int]
    L.oracle_pack_a.argtypes = [_P, _I, _I, _I, _I, _P]
    L.oracle_pack_b.argtypes = [_P, _I, _I, _I, _I, _P]
    L.oracle_goto.argtypes = [_I, _I, _I, _P, _I, _P, _I, _P, _I, _I, _I, _I, _I, _I, ctypes.c_int]
    L.oracle_goto.restype = ctypes.c_int
    return L


lib = _load()


def _ptr(a: np.ndarray):
    assert a.dtype in (np.float64, np.int64) and a.flags.c_contiguous
    return a.ctypes.data


def host_threads() -> int:
    return len(os.sched_getaffinity(0))


# -- generator (matrix.py:172-207, bench.py:89-106) ------------------------


def mix64(z: int) -> int:
    return int(lib.oracle_mix64(z & 0xFFFFFFFFFFFFFFFF))


def random_values(seed: int, count: int, start: int = 0) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    if count:
        lib.oracle_random_values(seed & 0xFFFFFFFFFFFFFFFF, count, start, _ptr(out))
    return out


def values_at(seed: int, positions) -> np.ndarray:
    pos = np.ascontiguousarray(positions, dtype=np.int64)
    out = np.empty(pos.size, dtype=np.float64)
    if pos.size:
        lib.oracle_values_at(seed & 0xFFFFFFFFFFFFFFFF, _ptr(pos), pos.size, _ptr(out))
    return out


def operand_seed(seed: int, role: int, m: int, n: int, k: int) -> int:
    return int(lib.oracle_operand_seed(seed & 0xFFFFFFFFFFFFFFFF, role, m, n, k))


def alloc(m: int, n: int, ld: int | None = None, canary: float | None = None) -> np.ndarray:
    """Flat column-major buffer of ld*n doubles (matrix.py:120-128); padding
    rows hold `canary` when given, else zero."""
    ld = m if ld is None else ld
    if m < 1 or n < 1 or ld < m:
        raise ValueError(f"bad matrix dims m={m} n={n} ld={ld}")
    buf = np.zeros(ld * n, dtype=np.float64)
    if canary is not None and ld > m:
        buf.reshape(n, ld)[:, m:] = canary
    return buf


def fill(buf: np.ndarray, m: int, n: int, ld: int, seed: int) -> np.ndarray:
    """fill_random (matrix.py:197-207): element (i,j) <- stream position j*m+i."""
    if buf.size < ld * (n - 1) + m:
        raise ValueError("buffer too small")
    lib.oracle_fill(_ptr(buf), m, n, ld, seed & 0xFFFFFFFFFFFFFFFF)
    return buf


def make_operands(seed: int, m: int, n: int, k: int):
    """bench.py:101-106 `make_operands`: tight leading dimensions."""
    a = fill(alloc(m, k), m, k, m, operand_seed(seed, 1, m, n, k))
    b = fill(alloc(k, n), k, n, k, operand_seed(seed, 2, m, n, k))
    c = fill(alloc(m, n), m, n, m, operand_seed(seed, 3, m, n, k))
    return a, b, c


def make_padded_operands(seed: int, m: int, n: int, k: int, lda: int, ldb: int, ldc: int,
                         canary: float | None = -777.25):
    """cfg-3 operands: same values as make_operands (values are ld-independent,
    reference tests/test_matrix.py:123-130), stored with padded ld and
    canaries in the padding rows."""
    a = fill(alloc(m, k, lda, canary), m, k, lda, operand_seed(seed, 1, m, n, k))
    b = fill(alloc(k, n, ldb, canary), k, n, ldb, operand_seed(seed, 2, m, n, k))
    c = fill(alloc(m, n, ldc, canary), m, n, ldc, operand_seed(seed, 3, m, n, k))
    return a, b, c


# -- GEMM oracles -----------------------------------------------------------


def naive(m, n, k, a, lda, b, ldb, c, ldc):
    """_ckernels.pyx:48-59: the reference oracle (single thread)."""
    lib.oracle_naive(m, n, k, _ptr(a), lda, _ptr(b), ldb, _ptr(c), ldc)
    return c


def naive_par(m, n, k, a, lda, b, ldb, c, ldc, threads: int | None = None):
    """Bitwise equal to naive (same per-element op sequence), threaded."""
    lib.oracle_naive_par(m, n, k, _ptr(a), lda, _ptr(b), ldb, _ptr(c), ldc,
                         threads or host_threads())
    return c


def goto(m, n, k, a, lda, b, ldb, c, ldc, mr=4, nr=4, mc=64, kc=256, nc=4096,
         threads: int = 1):
    """goto.py:187-239 / parallel.py:108-243 (loop ic) restated in C."""
    rc = lib.oracle_goto(m, n, k, _ptr(a), lda, _ptr(b), ldb, _ptr(c), ldc,
                         mr, nr, mc, kc, nc, threads)
    if rc != 0:
        raise ValueError(f"oracle_goto rejected parameters (rc={rc})")
    return c


def pack_a(src: np.ndarray, ld: int, mc: int, kc: int, mr: int) -> np.ndarray:
    buf = np.full(-(-mc // mr) * mr * kc, np.nan)
    lib.oracle_pack_a(_ptr(src), ld, mc, kc, mr, _ptr(buf))
    return buf


def pack_b(src: np.ndarray, ld: int, kc: int, nc: int, nr: int) -> np.ndarray:
    buf = np.full(-(-nc // nr) * nr * kc, np.nan)
    lib.oracle_pack_b(_ptr(src), ld, kc, nc, nr, _ptr(buf))
    return buf


# -- parity metric (kernels.py:31-38, matrix.py:90-107,210-232, bench.py:84-86)


def tolerance(k: int, a_max: float, b_max: float) -> float:
    """The reference's reorder gate: 2^-50 * k * max|A| * max|B|."""
    return 2.0**-50 * k * a_max * b_max


def headline_tolerance(k: int, ab_plus_c_max: float, c: float = 2.0) -> float:
    """BASELINE north_star bound: c * k * eps * (|A||B| + |C|)_max, eps = 2^-52,
    c = 2."""
    return c * k * 2.0**-52 * ab_plus_c_max


def valid_region(buf: np.ndarray, m: int, n: int, ld: int) -> np.ndarray:
    """The m x n valid region as an (n, m) view: row j is column j of the matrix."""
    return np.lib.stride_tricks.as_strided(buf, shape=(n, m), strides=(ld * 8, 8))


@dataclass
class DiffReport:
    max_abs_diff: float
    first_bad_i: int | None = None
    first_bad_j: int | None = None
    value_got: float | None = None
    value_expected: float | None = None

    @property
    def clean(self) -> bool:
        return self.first_bad_i is None


def max_abs_diff(got, want, m, n, ld_got, ld_want=None, tol: float = 0.0) -> DiffReport:
    """matrix.py:210-232: max |got-want| over the valid region, first offender
    (strict > tol) in column-major scan order."""
    g = valid_region(got, m, n, ld_got)
    w = valid_region(want, m, n, ld_want or ld_got)
    d = np.abs(g - w)
    rep = DiffReport(float(d.max()) if d.size else 0.0)
    bad = np.nonzero(d.ravel() > tol)[0]
    if bad.size:
        t = int(bad[0])
        j, i = divmod(t, m)
        rep.first_bad_i, rep.first_bad_j = i, j
        rep.value_got, rep.value_expected = float(g[j, i]), float(w[j, i])
    return rep


def failure_line(i: int, j: int, got: float, want: float) -> str:
    """bench.py:84-86 diagnostic."""
    return f"C[ {i} ][ {j} ] != C_ref, {got:.6E}, {want:.6E}"


def sha256_valid(buf: np.ndarray, m: int, n: int, ld: int) -> str:
    """SHA-256 of the valid region, column-major little-endian f64 (SURVEY 8c KATs)."""
    import hashlib

    h = hashlib.sha256()
    v = valid_region(buf, m, n, ld)
    for j in range(n):
        h.update(np.ascontiguousarray(v[j]).astype("<f8").tobytes())
    return h.hexdigest()


def sampled_reference(seed: int, m: int, n: int, k: int, rows, cols):
    """Oracle values of C_ref(i, j) for the sampled (i, j) grid of a
    make_operands problem, without materialising A, B or C.

    Each element is gemm_naive on the 1 x k row of A and the k x 1 column of
    B plus c_ij -- bitwise the full-GEMM element, since the per-element order
    is p-ascending (_ckernels.pyx:48-59).  Also returns (|A||B|+|C|)(i, j)
    for the headline tolerance.
    """
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    sa, sb, sc = (operand_seed(seed, r, m, n, k) for r in (1, 2, 3))
    p = np.arange(k, dtype=np.int64)
    a_rows = np.stack([values_at(sa, p * m + i) for i in rows])          # (R, k)
    b_cols = np.stack([values_at(sb, j * k + p) for j in cols])          # (Cn, k)
    c0 = np.stack([values_at(sc, j * m + rows) for j in cols], axis=1)   # (R, Cn)
    out = np.empty((rows.size, cols.size))
    mag = np.empty_like(out)
    for r in range(rows.size):
        arow = np.ascontiguousarray(a_rows[r])
        for q in range(cols.size):
            cc = np.array([c0[r, q]])
            lib.oracle_naive(1, 1, k, _ptr(arow), 1, _ptr(np.ascontiguousarray(b_cols[q])), k,
                             _ptr(cc), 1)
            out[r, q] = cc[0]
            mag[r, q] = float(np.abs(arow) @ np.abs(b_cols[q])) + abs(c0[r, q])
    return out, mag
