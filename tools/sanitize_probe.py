"""Small ragged shapes through every kernel and path, for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
from paper_1609_00076_b200 import engine

st = torch.cuda.current_stream().cuda_stream
for (m, n, k, pa, pb, pc) in [(37, 53, 71, 7, 5, 3), (1, 70, 33, 7, 5, 3), (70, 1, 33, 7, 5, 3),
                              (129, 130, 47, 1, 1, 1), (200, 260, 300, 0, 0, 0), (65, 33, 17, 2, 2, 2),
                              (6, 300, 90, 1, 2, 3), (4100, 7, 60, 2, 1, 1), (1300, 1500, 100, 2, 2, 2)]:
    lda, ldb, ldc = m + pa, k + pb, m + pc
    a, b, c = oracle.make_padded_operands(42, m, n, k, lda, ldb, ldc)
    want = oracle.naive(m, n, k, a, lda, b, ldb, c.copy(), ldc)
    for kw in ({}, {"exact": True}):
        got = engine.my_dgemm(m, n, k, a, lda, b, ldb, c.copy(), ldc, **kw)
        assert np.abs(got - want).max() <= oracle.tolerance(k, 1, 1), (m, n, k, kw)
    # device path, exact-size buffers (no slack past (n-1)*ld+m), every unit shape
    for strips in (0, 2, 4, 8, 16, 32, 34, 36, 40):
        da = torch.from_numpy(a[: (k - 1) * lda + m].copy()).cuda()
        db = torch.from_numpy(b[: (n - 1) * ldb + k].copy()).cuda()
        dc = torch.from_numpy(c[: (n - 1) * ldc + m].copy()).cuda()
        engine.dgemm_device(m, n, k, da.data_ptr(), lda, db.data_ptr(), ldb, dc.data_ptr(), ldc, st,
                            strips=strips, force_tiled=strips > 0)
        torch.cuda.synchronize()
        got = dc.cpu().numpy()
        assert np.abs(got - want[: (n - 1) * ldc + m]).max() <= oracle.tolerance(k, 1, 1), (m, n, k, strips)
d = torch.empty(40 * 7, dtype=torch.float64, device="cuda")
engine.fill_random_device(d.data_ptr(), 37, 7, 40, 5, 0, st)
mx, i, j = engine.max_abs_diff_device(37, 7, d.data_ptr(), 40, d.data_ptr(), 40, 0.0, st)
assert mx == 0.0 and i is None
torch.cuda.synchronize()
print("sanitize probe ok")
