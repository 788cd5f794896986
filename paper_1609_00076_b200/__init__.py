"""paper_1609_00076_b200 -- B200-native (sm_100a) FP64 GEMM behind the
reference's `my_dgemm` path (BLISlab, arXiv:1609.00076; reference package
`gemmforge`).

The hot path is hand-written CUDA in csrc/ compiled to libmy_dgemm_b200.so,
whose C ABI is include/my_dgemm.h.  This package is the host-side mirror of
the reference's engine/registry interface (engine.py), the jc-sharded
multi-GPU driver (multi.py) and its copy-engine exchange of A over NVLink
peer memory (peer.py).  There is no CPU fallback: calls raise when the
library is absent.
"""

from .engine import (  # noqa: F401
    Matrix,
    alloc_matrix,
    b200_factory,
    check_conformal,
    dgemm,
    dgemm_device,
    fill_random_device,
    gemm_b200,
    kernel_launches,
    DiffReport,
    VerificationError,
    diff_report_device,
    failure_line,
    max_abs_diff_device,
    verify_device,
    my_dgemm,
    operand_seed,
    register,
    tune,
)
from .tuning import TilePoint, TileTuneResult, tune_grid  # noqa: F401

__version__ = "0.1.0"
