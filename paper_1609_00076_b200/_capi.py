"""ctypes binding of libmy_dgemm_b200.so (the C ABI in include/my_dgemm.h).

ctypes.CDLL releases the GIL for the duration of every call, as the
reference's Cython kernels do with `nogil` (_ckernels.pyx:7-8).  There is no
fallback: if the library is missing or fails to load, every entry point
raises, so a GPU test can never pass on a silent CPU path.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MY_DGEMM_LIB") or os.path.join(HERE, "libmy_dgemm_b200.so")

# Flags (include/my_dgemm.h)
DEVICE_PTRS = 0x1
EXACT = 0x2
FORCE_TILED = 0x4
FORCE_VEC1 = 0x8
FORCE_STRIPS2 = 0x10
FORCE_STRIPS4 = 0x20
FORCE_UNITS8 = 0x40
FORCE_ROWS16 = 0x80
FORCE_STREAMK = 0x800
BLAS_EPILOGUE = 0x1000
FORCE_SMALL = 0x2000
FORCE_TILES = 0x40000
PLAN_INVARIANT = 0x80000
FORCE_KSPLIT = 0x100000


def SMALL_VARIANT(v: int) -> int:  # noqa: N802 - mirrors the C macro
    return v << 14


IPC_HANDLE_BYTES = 64
PATH_TILED, PATH_GEMV_N1, PATH_GEMV_M1, PATH_FEW_COLS, PATH_FEW_ROWS, PATH_EXACT, PATH_ROWS_DMMA = range(7)


def FORCE_PATH(p: int) -> int:  # noqa: N802 - mirrors the C macro
    return (p + 1) << 8

# Every symbol the header declares, with (restype, argtypes).
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64
_D = ctypes.c_double
SIGNATURES = {
    "my_dgemm": (None, [_I, _I, _I, _P, _I, _P, _I, _P, _I]),
    "bl_dgemm": (None, [_I, _I, _I, _P, _I, _P, _I, _P, _I]),
    "my_dgemm_ex": (_I, [_I, _I, _I, _P, _I, _P, _I, _P, _I, ctypes.c_uint, _P]),
    "my_dgemm_shard": (_I, [_I, _I, _I, _P, _I, _P, _I, _P, _I, _P]),
    "my_dgemm_blas": (_I, [ctypes.c_char, ctypes.c_char, _I, _I, _I, _D, _P, _I, _P, _I, _D, _P, _I,
                           ctypes.c_uint, _P]),
    "my_dsyrk": (_I, [ctypes.c_char, ctypes.c_char, _I, _I, _D, _P, _I, _D, _P, _I, ctypes.c_uint, _P]),
    "my_dtrmm": (_I, [ctypes.c_char, ctypes.c_char, ctypes.c_char, ctypes.c_char, _I, _I, _D, _P, _I, _P, _I,
                      ctypes.c_uint, _P]),
    "my_dtrsm": (_I, [ctypes.c_char, ctypes.c_char, ctypes.c_char, ctypes.c_char, _I, _I, _D, _P, _I, _P, _I,
                      ctypes.c_uint, _P]),
    "my_dgemm_multi": (_I, [_I, _I, _I, _I, _P, _I, _P, _I, _P, _I]),
    "my_dgemm_multi_ex": (_I, [ctypes.POINTER(_I), _I, _I, _I, _I, _P, _I, _P, _I, _P, _I, ctypes.c_uint]),
    "my_dgemm_fill_random": (_I, [_P, _I64, _I64, _I64, _U64, _I64, _P]),
    "my_dgemm_operand_seed": (_U64, [_U64, _U64, _I64, _I64, _I64]),
    "my_dgemm_max_abs_diff": (_I, [_I64, _I64, _P, _I64, _P, _I64, _D, ctypes.POINTER(_D),
                                   ctypes.POINTER(_I64), _P]),
    "my_dgemm_diff_report": (_I, [_I64, _I64, _P, _I64, _P, _I64, _D, ctypes.POINTER(_D),
                                  ctypes.POINTER(_I64), ctypes.POINTER(_D), ctypes.POINTER(_D), _P]),
    "my_dgemm_tune": (_I, [_I, _I, _I, _I, _I, _I, _I, ctypes.POINTER(_I), ctypes.POINTER(_D)]),
    "my_dgemm_tune_clear": (None, []),
    "my_dgemm_plan_geometry": (_I, [_I, _I, _I, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_I),
                                    ctypes.POINTER(_I)]),
    "my_dgemm_tune_set": (_I, [_I, _I, _I, _I, _I, _I]),
    "my_dgemm_plan_describe": (_I, [_I, _I, _I, _I, _I, _I, _I, ctypes.c_char_p, _I]),
    "my_dgemm_set_max_ctas": (_I, [_I]),
    "my_dgemm_path": (_I, [_I, _I, ctypes.c_uint]),
    "my_dgemm_ipc_export": (_I, [_P, ctypes.c_char_p, ctypes.POINTER(_U64)]),
    "my_dgemm_ipc_open": (_I, [ctypes.c_char_p, _U64, ctypes.POINTER(_P)]),
    "my_dgemm_ipc_close": (_I, [_P, _U64]),
    "my_dgemm_signal_write": (_I, [_P, _P, ctypes.c_uint32]),
    "my_dgemm_signal_wait_geq": (_I, [_P, _P, ctypes.c_uint32]),
    "my_dgemm_copy_async": (_I, [_P, _P, _U64, _P]),
    "my_dgemm_last_error": (ctypes.c_char_p, []),
    "my_dgemm_last_status": (_I, []),
    "my_dgemm_version": (ctypes.c_char_p, []),
    "my_dgemm_kernel_launches": (_U64, []),
    "my_dgemm_release_workspace": (None, []),
}


class NativeLibraryError(RuntimeError):
    """The sm_100a library is missing or failed to load."""


class CudaError(RuntimeError):
    """A CUDA runtime failure inside the library (status >= 1000)."""

    def __init__(self, status: int, message: str):
        super().__init__(f"[status {status}] {message}")
        self.status = status


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the library.  Raises NativeLibraryError."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} not built; run `python -m paper_1609_00076_b200.build` "
            "(there is no CPU fallback)"
        )
    try:
        lib = ctypes.CDLL(path)
    except OSError as e:  # pragma: no cover - environment specific
        raise NativeLibraryError(f"cannot load {path}: {e}") from e
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().my_dgemm_last_error().decode()


def check(status: int) -> None:
    """Map a C-ABI status to the reference's exception types: negative
    statuses are argument errors (ValueError, as kernels.py:41-49 /
    matrix.py:50-53 raise), >= 1000 are CUDA failures."""
    if status == 0:
        return
    msg = last_error()
    if status < 0:
        raise ValueError(msg)
    raise CudaError(status, msg)
