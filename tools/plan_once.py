"""One call of the given launch plan on device-resident operands, after a
warm-up call (ncu target): python tools/plan_once.py M N K PLAN [PLAN ...]
(LDC_PAD=p: ldc = m + p)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import engine

m, n, k = (int(v) for v in sys.argv[1:4])
plans = [int(p) for p in sys.argv[4:]] or [0]
st = torch.cuda.current_stream().cuda_stream
a = torch.empty(m * k, dtype=torch.float64, device="cuda")
b = torch.empty(k * n, dtype=torch.float64, device="cuda")
ldc = m + int(os.environ.get("LDC_PAD", "0"))
c = torch.empty(ldc * n, dtype=torch.float64, device="cuda")
for t, (buf, r, cc, ld) in enumerate(((a, m, k, m), (b, k, n, k), (c, m, n, ldc))):
    engine.fill_random_device(buf.data_ptr(), r, cc, ld, 1000 + t, 0, st)
for p in plans:
    for _ in range(2):
        engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), ldc, st, strips=p)
torch.cuda.synchronize()
print("ok")
