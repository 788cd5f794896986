"""Run the fast kernel on device-resident operands a few times (ncu target).

  python tools/profile_one.py [m n k] [--launches L]
"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

argv = sys.argv[1:]
launches = 3
if "--launches" in argv:
    i = argv.index("--launches")
    launches = int(argv[i + 1])
    del argv[i:i + 2]
args = [a for a in argv if not a.startswith("--")]
m, n, k = (int(x) for x in (args or [8192, 8192, 8192]))
st = torch.cuda.current_stream().cuda_stream
a = torch.empty(m * k, dtype=torch.float64, device="cuda")
b = torch.empty(k * n, dtype=torch.float64, device="cuda")
c = torch.empty(m * n, dtype=torch.float64, device="cuda")
for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c, m, n))):
    engine.fill_random_device(buf.data_ptr(), r, cc, r, 7 + t, 0, st)
for _ in range(launches):
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st)
torch.cuda.synchronize()
print("ok", m, n, k, launches)
