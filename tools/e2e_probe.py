"""End-to-end my_dgemm_ex timing from pinned vs pageable host buffers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1609_00076_b200 import _capi
lib = _capi.load()
m = n = k = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
for kind in ("pinned", "pageable"):
    if kind == "pinned":
        A = torch.rand(m * k, dtype=torch.float64).pin_memory(); B = torch.rand(k * n, dtype=torch.float64).pin_memory()
        C = torch.rand(m * n, dtype=torch.float64).pin_memory()
        pa, pb, pc = A.data_ptr(), B.data_ptr(), C.data_ptr()
    else:
        A = np.random.rand(m * k); B = np.random.rand(k * n); C = np.random.rand(m * n)
        pa, pb, pc = A.ctypes.data, B.ctypes.data, C.ctypes.data
    call = lambda: _capi.check(lib.my_dgemm_ex(m, n, k, pa, m, pb, k, pc, m, 0, None))
    call(); call()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); call(); ts.append(time.perf_counter() - t0)
    t = min(ts)
    print(f"{kind}: {t*1e3:.1f} ms  {2*m*n*k/t/1e12:.2f} TF", flush=True)
