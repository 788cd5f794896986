"""Host-side mirror of the reference's engine / plugin interface for the
my_dgemm path, over the sm_100a C ABI.

The reference (Python package `gemmforge`, /root/reference/pkg) selects GEMM
engines by name through `KernelRegistry.register_variant(name, factory)`
(pkg/src/gemmforge/registry.py:113-125); a factory maps a config to
`engine(a, b, c, backend=None, stats=None, **kw) -> c` (the shape of
`_goto_factory`, registry.py:185-198) over column-major `Matrix` objects
(matrix.py:39-87).  This module provides exactly that surface:

  * `Matrix`, `check_conformal`  -- same attributes, same ValueError wording;
  * `gemm_b200(a, b, c)`         -- the engine (the drop-in for gemm_goto /
                                    gemm_goto_parallel, goto.py:187,
                                    parallel.py:108);
  * `b200_factory(cfg)`          -- the registry factory;
  * `register(registry)`         -- `registry.register_variant("b200", ...)`,
                                    which runs the reference's own validation
                                    gate (registry.py:127-137) when given the
                                    reference registry;
  * `my_dgemm(...)`              -- the flat-buffer BASELINE signature.

Any object with `.m .n .ld .data` (a float64 1-D numpy array) is accepted as a
matrix, so the reference's own Matrix instances work unchanged.  Device
operands (torch CUDA tensors as `.data`) run asynchronously on the current
stream; host operands stage through the library's device workspace.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _capi

__all__ = [
    "Matrix",
    "alloc_matrix",
    "check_conformal",
    "gemm_b200",
    "b200_factory",
    "register",
    "my_dgemm",
    "my_dgemm_multi",
    "set_max_ctas",
    "dsyrk",
    "dtrmm",
    "dtrsm",
    "path",
    "dgemm_device",
    "fill_random_device",
    "operand_seed",
    "max_abs_diff_device",
    "DiffReport",
    "diff_report_device",
    "failure_line",
    "VerificationError",
    "verify_device",
    "kernel_launches",
    "dgemm",
    "tune",
]


class Matrix:
    """Column-major float64 matrix over an explicit leading dimension.

    Mirrors gemmforge.matrix.Matrix (matrix.py:39-87): element (i, j) at
    data[j*ld + i]; data must hold at least ld*(n-1)+m elements.
    """

    __slots__ = ("m", "n", "ld", "data")

    def __init__(self, m: int, n: int, ld: int, data):
        if m < 1 or n < 1:
            raise ValueError(f"matrix dims must be positive, got m={m} n={n}")
        if ld < m:
            raise ValueError(f"leading dimension ld={ld} smaller than row count m={m}")
        _check_buffer(data, ld * (n - 1) + m)
        self.m, self.n, self.ld, self.data = m, n, ld, data

    @property
    def shape(self) -> tuple[int, int]:
        return (self.m, self.n)

    def __repr__(self) -> str:
        return f"Matrix(m={self.m}, n={self.n}, ld={self.ld})"


def alloc_matrix(m: int, n: int, ld: int | None = None) -> Matrix:
    """Zeroed host matrix (matrix.py:120-128)."""
    ld = m if ld is None else ld
    if m < 1 or n < 1:
        raise ValueError(f"matrix dims must be positive, got m={m} n={n}")
    if ld < m:
        raise ValueError(f"leading dimension ld={ld} smaller than row count m={m}")
    return Matrix(m, n, ld, np.zeros(ld * n, dtype=np.float64))


def _is_device(data) -> bool:
    return hasattr(data, "__cuda_array_interface__") or (
        hasattr(data, "is_cuda") and bool(getattr(data, "is_cuda"))
    )


def _check_buffer(data, need: int) -> None:
    if _is_device(data):
        import torch

        if data.dtype != torch.float64 or data.dim() != 1 or not data.is_contiguous():
            raise ValueError("data must be a 1-D float64 ndarray")
        size = data.numel()
    else:
        if not isinstance(data, np.ndarray) or data.dtype != np.float64 or data.ndim != 1:
            raise ValueError("data must be a 1-D float64 ndarray")
        if not data.flags.c_contiguous:
            raise ValueError("data must be contiguous")
        size = data.size
    if size < need:
        raise ValueError(f"buffer too small: need {need} elements, got {size}")


def _ptr(data) -> int:
    if isinstance(data, np.ndarray):
        return data.ctypes.data
    return int(data.data_ptr())


def check_conformal(a, b, c) -> tuple[int, int, int]:
    """Validate C(m,n) := A(m,k) * B(k,n) + C (kernels.py:41-49, same messages)."""
    if a.n != b.m:
        raise ValueError(f"inner dims differ: A is {a.m}x{a.n}, B is {b.m}x{b.n}")
    if c.m != a.m or c.n != b.n:
        raise ValueError(
            f"C is {c.m}x{c.n}, expected {a.m}x{b.n} from A {a.m}x{a.n} * B {b.m}x{b.n}"
        )
    return a.m, b.n, a.n


# launch-plan pins of `strips` (dgemm_device) -> flag bits, built once
_STRIPS_FLAGS = {0: 0, 1: _capi.FORCE_TILES, 2: _capi.FORCE_STRIPS2, 4: _capi.FORCE_STRIPS4, 8: _capi.FORCE_UNITS8,
                 16: _capi.FORCE_ROWS16, 32: _capi.FORCE_STREAMK, 34: _capi.FORCE_STREAMK | _capi.FORCE_STRIPS2,
                 36: _capi.FORCE_STREAMK | _capi.FORCE_STRIPS4, 40: _capi.FORCE_STREAMK | _capi.FORCE_UNITS8,
                 48: _capi.FORCE_KSPLIT, -1: _capi.PLAN_INVARIANT,
                 **{64 + v: _capi.FORCE_SMALL | _capi.SMALL_VARIANT(v) for v in range(16)}}


def _flags(exact: bool, force_tiled: bool = False, force_vec1: bool = False, strips: int = 0,
           path: int | None = None) -> int:
    f = _capi.EXACT if exact else 0
    f |= _capi.FORCE_PATH(path) if path is not None else 0
    f |= _capi.FORCE_TILED if force_tiled else 0
    f |= _capi.FORCE_VEC1 if force_vec1 else 0
    f |= _STRIPS_FLAGS[strips]
    return f


def gemm_b200(a, b, c, backend=None, stats=None, exact: bool = False, stream=None, **kw):
    """C := A*B + C on the B200.  Reference engine signature (registry.py:190).

    `backend` is accepted and ignored (the reference's CPU backend switch,
    backends.py:93-100, has no meaning for the GPU engine).  `stats`, when a
    dict, counts launches under "gpu_calls".  exact=True selects the bitwise
    oracle twin.  Host operands: synchronous.  Device operands (torch CUDA
    tensors, all three): asynchronous on `stream` (default: torch's current
    stream).
    """
    m, n, k = check_conformal(a, b, c)
    for mat, rows in ((a, m), (b, k), (c, m)):
        _check_buffer(mat.data, mat.ld * (mat.n - 1) + rows)
    dev = [_is_device(x.data) for x in (a, b, c)]
    lib = _capi.load()
    flags = _flags(exact, kw.get("force_tiled", False), kw.get("force_vec1", False))
    if all(dev):
        if stream is None:
            import torch

            stream = torch.cuda.current_stream(c.data.device).cuda_stream
        st = lib.my_dgemm_ex(m, n, k, _ptr(a.data), a.ld, _ptr(b.data), b.ld, _ptr(c.data), c.ld,
                             flags | _capi.DEVICE_PTRS, ctypes.c_void_p(stream))
    elif not any(dev):
        st = lib.my_dgemm_ex(m, n, k, _ptr(a.data), a.ld, _ptr(b.data), b.ld, _ptr(c.data), c.ld,
                             flags, None)
    else:
        raise ValueError("operands must be all host or all device buffers")
    _capi.check(st)
    if stats is not None:
        stats["gpu_calls"] = stats.get("gpu_calls", 0) + 1
    return c


def b200_factory(cfg=None):
    """Registry factory (registry.py:185-198 shape).  The CPU blocking
    parameters in cfg.goto / cfg.threads do not apply to the GPU engine and
    are ignored; `cfg.exact` (optional) selects the bitwise twin."""
    exact = bool(getattr(cfg, "exact", False)) if cfg is not None else False

    def run(a, b, c, backend=None, stats=None, **kw):
        return gemm_b200(a, b, c, backend=backend, stats=stats, exact=kw.pop("exact", exact), **kw)

    return run


def register(registry=None, name: str = "b200", validate: bool = True):
    """Register the engine as a named variant.  With the reference registry
    (gemmforge.registry.default_registry()) this passes through its own
    validation gate (registry.py:127-137) before it becomes selectable."""
    if registry is None:
        from gemmforge.registry import default_registry  # the reference package

        registry = default_registry()
    if name in registry.variant_names():
        return registry.variant(name)
    return registry.register_variant(name, b200_factory, validate=validate)


def my_dgemm(m: int, n: int, k: int, A: np.ndarray, lda: int, B: np.ndarray, ldb: int,
             C: np.ndarray, ldc: int, exact: bool = False) -> np.ndarray:
    """The BASELINE signature on flat host buffers.  Checks the
    buffer lengths the C ABI cannot see, then calls my_dgemm_ex."""
    if m < 1 or n < 1 or k < 1:
        raise ValueError(f"matrix dims must be positive, got m={m} n={n} k={k}")
    Matrix(m, k, lda, A), Matrix(k, n, ldb, B), Matrix(m, n, ldc, C)
    lib = _capi.load()
    _capi.check(lib.my_dgemm_ex(m, n, k, _ptr(A), lda, _ptr(B), ldb, _ptr(C), ldc,
                                _flags(exact), None))
    return C


def my_dgemm_multi(devices, m: int, n: int, k: int, A: np.ndarray, lda: int, B: np.ndarray, ldb: int,
                   C: np.ndarray, ldc: int, exact: bool = False) -> np.ndarray:
    """my_dgemm over several GPUs of this process (C ABI my_dgemm_multi[_ex]).
    `devices`: a device count (GPUs 0..n-1) or an explicit list of device ids
    (entries may repeat: each is its own column shard).  Host buffers;
    synchronous; C is bitwise the single-device my_dgemm result."""
    if m < 1 or n < 1 or k < 1:
        raise ValueError(f"matrix dims must be positive, got m={m} n={n} k={k}")
    Matrix(m, k, lda, A), Matrix(k, n, ldb, B), Matrix(m, n, ldc, C)
    lib = _capi.load()
    if isinstance(devices, int) and not exact:
        _capi.check(lib.my_dgemm_multi(devices, m, n, k, _ptr(A), lda, _ptr(B), ldb, _ptr(C), ldc))
        return C
    ids = list(range(devices)) if isinstance(devices, int) else [int(d) for d in devices]
    arr = (ctypes.c_int * max(1, len(ids)))(*ids)
    _capi.check(lib.my_dgemm_multi_ex(arr, len(ids), m, n, k, _ptr(A), lda, _ptr(B), ldb, _ptr(C), ldc,
                                      _flags(exact)))
    return C


def dgemm_device(m, n, k, a_ptr: int, lda: int, b_ptr: int, ldb: int, c_ptr: int, ldc: int,
                 stream: int = 0, exact: bool = False, force_tiled: bool = False,
                 force_vec1: bool = False, strips: int = 0, path: int | None = None) -> None:
    """Raw device-pointer call (asynchronous on `stream`).  `strips` pins
    the launch plan (tests, tuning): 1 full tiles only, 2 / 4 / 8 / 16 every tile as 128x64 /
    128x32 / 64x32 / 16x128 units, 32 / 34 / 36 / 40 the stream-K schedule
    over full tiles / those units, 64 + v the small-block kernel's variant v
    (1..10; 64: the planner's pick); `path` forces a kernel family
    (_capi.PATH_*, what sharded drivers pass to every shard).  Every one of
    these plans gives bitwise the same C.  48 is the opt-in K-split plan
    (MY_DGEMM_FORCE_KSPLIT: deterministic and within the tolerance, but not
    that same chain), -1 the heuristic kept to the plan-invariant plans
    (MY_DGEMM_PLAN_INVARIANT; the default unless MY_DGEMM_KSPLIT=1)."""
    lib = _capi._lib or _capi.load()
    if exact or force_tiled or force_vec1 or strips or path is not None:
        flags = _flags(exact, force_tiled, force_vec1, strips, path) | _capi.DEVICE_PTRS
    else:  # (the common call: no Python work beyond the ctypes call)
        flags = _capi.DEVICE_PTRS
    status = lib.my_dgemm_ex(m, n, k, a_ptr, lda, b_ptr, ldb, c_ptr, ldc, flags, stream)
    if status:
        _capi.check(status)


def fill_random_device(ptr: int, m: int, n: int, ld: int, seed: int, col0: int = 0,
                       stream: int = 0) -> None:
    """splitmix64-v1 fill on the device, bit-exact with fill_random (matrix.py:197-207)."""
    lib = _capi.load()
    _capi.check(lib.my_dgemm_fill_random(ptr, m, n, ld, seed & 0xFFFFFFFFFFFFFFFF, col0,
                                         ctypes.c_void_p(stream)))


def operand_seed(seed: int, role: int, m: int, n: int, k: int) -> int:
    """bench.py:89-98 `_operand_seed`."""
    return int(_capi.load().my_dgemm_operand_seed(seed & 0xFFFFFFFFFFFFFFFF, role, m, n, k))


def max_abs_diff_device(m: int, n: int, x_ptr: int, ldx: int, y_ptr: int, ldy: int,
                        tol: float = 0.0, stream: int = 0) -> tuple[float, int | None, int | None]:
    """matrix.py:210-232 on the device: (max |X-Y|, first_bad_i, first_bad_j)."""
    lib = _capi.load()
    mx = ctypes.c_double()
    first = ctypes.c_int64()
    _capi.check(lib.my_dgemm_max_abs_diff(m, n, x_ptr, ldx, y_ptr, ldy, tol, ctypes.byref(mx),
                                          ctypes.byref(first), ctypes.c_void_p(stream)))
    if first.value < 0:
        return mx.value, None, None
    j, i = divmod(first.value, m)
    return mx.value, i, j


class DiffReport:
    """matrix.py:90-107 `DiffReport`: the largest |got - want| and, iff some
    difference exceeds the tolerance, the first offender in column-major scan
    order with its two values."""

    __slots__ = ("max_abs_diff", "first_bad_i", "first_bad_j", "value_got", "value_expected")

    def __init__(self, max_abs_diff, first_bad_i=None, first_bad_j=None, value_got=None, value_expected=None):
        self.max_abs_diff = max_abs_diff
        self.first_bad_i = first_bad_i
        self.first_bad_j = first_bad_j
        self.value_got = value_got
        self.value_expected = value_expected

    @property
    def clean(self) -> bool:
        return self.first_bad_i is None

    def __repr__(self) -> str:
        return (f"DiffReport(max_abs_diff={self.max_abs_diff!r}, first_bad_i={self.first_bad_i!r}, "
                f"first_bad_j={self.first_bad_j!r}, value_got={self.value_got!r}, "
                f"value_expected={self.value_expected!r})")


def failure_line(i: int, j: int, got: float, want: float) -> str:
    """bench.py:84-86: the mismatch diagnostic in the classic test-driver form."""
    return f"C[ {i} ][ {j} ] != C_ref, {got:.6E}, {want:.6E}"


class VerificationError(RuntimeError):
    """bench.py:74-81: a result outside tolerance of the oracle; `diagnostic`
    is the failure line."""

    def __init__(self, diagnostic: str, m=None, n=None, k=None, algorithm=None):
        super().__init__(diagnostic)
        self.diagnostic = diagnostic
        self.m, self.n, self.k = m, n, k
        self.algorithm = algorithm


def diff_report_device(m: int, n: int, got_ptr: int, ld_got: int, want_ptr: int, ld_want: int,
                       tol: float = 0.0, stream: int = 0) -> DiffReport:
    """matrix.py:210-232 `max_abs_diff` on device-resident matrices: the
    reference's DiffReport (strict > tol offender rule, column-major first
    offender, NaN max when a difference is NaN)."""
    lib = _capi.load()
    mx, first, got, want = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    _capi.check(lib.my_dgemm_diff_report(m, n, got_ptr, ld_got, want_ptr, ld_want, tol, ctypes.byref(mx),
                                         ctypes.byref(first), ctypes.byref(got), ctypes.byref(want),
                                         ctypes.c_void_p(stream)))
    if first.value < 0:
        return DiffReport(mx.value)
    j, i = divmod(first.value, m)
    return DiffReport(mx.value, i, j, got.value, want.value)


def verify_device(m: int, n: int, k: int, got_ptr: int, ld_got: int, want_ptr: int, ld_want: int, tol: float,
                  algorithm: str = "b200", stream: int = 0) -> DiffReport:
    """run_sweep's check (bench.py:140-156) on the device: raise
    VerificationError carrying the reference's failure line at the first
    offender; also raise when the max difference is NaN (which the strict
    offender rule alone would let through)."""
    rep = diff_report_device(m, n, got_ptr, ld_got, want_ptr, ld_want, tol, stream)
    if not rep.clean:
        raise VerificationError(failure_line(rep.first_bad_i, rep.first_bad_j, rep.value_got, rep.value_expected),
                                m=m, n=n, k=k, algorithm=algorithm)
    if rep.max_abs_diff != rep.max_abs_diff:
        raise VerificationError(f"max |C - C_ref| is NaN over {m}x{n}", m=m, n=n, k=k, algorithm=algorithm)
    return rep


def path(m: int, n: int, exact: bool = False) -> int:
    """Kernel family of an (m, n) call (my_dgemm_path): _capi.PATH_TILED or
    one of the bandwidth kernels.  Sharded drivers force the tiled kernel on
    every shard exactly when the whole problem is tiled."""
    k = int(_capi.load().my_dgemm_path(m, n, _flags(exact)))
    if k < 0:
        raise ValueError(_capi.last_error())
    return k


def set_max_ctas(n: int) -> int:
    """Cap the tiled kernel at n SMs (0 = all); returns the previous cap.
    Results are bitwise independent of the cap (my_dgemm_set_max_ctas)."""
    prev = int(_capi.load().my_dgemm_set_max_ctas(int(n)))
    if prev < 0:
        raise ValueError(_capi.last_error())
    return prev


def kernel_launches() -> int:
    return int(_capi.load().my_dgemm_kernel_launches())


def dgemm(transa: str, transb: str, m: int, n: int, k: int, alpha: float, A, lda: int, B, ldb: int,
          beta: float, C, ldc: int, exact: bool = False, stream: int | None = None, epilogue: bool = False,
          plan: int = 0):
    """BLAS dgemm: C := alpha op(A) op(B) + beta C.

    Host numpy buffers (synchronous) or torch CUDA tensors (asynchronous on
    `stream`, default torch's current stream).  Argument errors raise
    ValueError naming the BLAS parameter.  `epilogue` (tests) forces alpha /
    beta into the kernel epilogue instead of the reference-BLAS order; `plan`
    pins the launch plan of the tiled kernel (dgemm_device's `strips`).
    """
    lib = _capi.load()
    flags = _flags(exact, strips=plan) | (_capi.BLAS_EPILOGUE if epilogue else 0)
    dev = _is_device(C)
    if dev:
        if stream is None:
            import torch

            stream = torch.cuda.current_stream(C.device).cuda_stream
        flags |= _capi.DEVICE_PTRS
    ptr = lambda x: None if x is None else _ptr(x)  # noqa: E731
    st = lib.my_dgemm_blas(transa.encode()[:1], transb.encode()[:1], m, n, k, float(alpha), ptr(A), lda,
                           ptr(B), ldb, float(beta), ptr(C), ldc, flags,
                           ctypes.c_void_p(stream) if dev else None)
    _capi.check(st)
    return C


def _level3_stream(t, stream):
    if not _is_device(t):
        raise ValueError("level-3 routines take CUDA tensors (device pointers)")
    if stream is None:
        import torch

        stream = torch.cuda.current_stream(t.device).cuda_stream
    return ctypes.c_void_p(stream)


def dsyrk(uplo: str, trans: str, n: int, k: int, alpha: float, A, lda: int, beta: float, C, ldc: int,
          stream: int | None = None):
    """C := alpha op(A) op(A)^T + beta C on the `uplo` triangle (my_dsyrk; GEMM-based
    level-3 BLAS).  CUDA tensors, asynchronous on `stream`."""
    st = _level3_stream(C, stream)
    _capi.check(_capi.load().my_dsyrk(uplo.encode()[:1], trans.encode()[:1], n, k, float(alpha),
                                      None if A is None else _ptr(A), lda, float(beta), _ptr(C), ldc,
                                      _capi.DEVICE_PTRS, st))
    return C


def _tri(fn, side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, stream):
    st = _level3_stream(B, stream)
    _capi.check(getattr(_capi.load(), fn)(side.encode()[:1], uplo.encode()[:1], transa.encode()[:1],
                                          diag.encode()[:1], m, n, float(alpha), None if A is None else _ptr(A),
                                          lda, _ptr(B), ldb, _capi.DEVICE_PTRS, st))
    return B


def dtrmm(side: str, uplo: str, transa: str, diag: str, m: int, n: int, alpha: float, A, lda: int, B, ldb: int,
          stream: int | None = None):
    """B := alpha op(A) B (side 'L') or alpha B op(A) (side 'R'), A triangular (my_dtrmm)."""
    return _tri("my_dtrmm", side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, stream)


def dtrsm(side: str, uplo: str, transa: str, diag: str, m: int, n: int, alpha: float, A, lda: int, B, ldb: int,
          stream: int | None = None):
    """Solve op(A) X = alpha B (side 'L') or X op(A) = alpha B (side 'R'); X overwrites B (my_dtrsm)."""
    return _tri("my_dtrsm", side, uplo, transa, diag, m, n, alpha, A, lda, B, ldb, stream)


def tune(m: int, n: int, k: int, lda: int | None = None, ldb: int | None = None, ldc: int | None = None,
         reps: int = 3) -> tuple[int, float]:
    """Pick the fastest launch plan for this shape (my_dgemm_tune); later calls
    of the shape use it.  Returns (plan, ms).  Results are unaffected."""
    lib = _capi.load()
    plan = ctypes.c_int()
    ms = ctypes.c_double()
    _capi.check(lib.my_dgemm_tune(m, n, k, lda or m, ldb or k, ldc or m, reps, ctypes.byref(plan),
                                  ctypes.byref(ms)))
    return plan.value, ms.value
