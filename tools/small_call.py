"""Run one shape a few times through the C ABI (target for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import engine

m, n, k = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
st = torch.cuda.current_stream().cuda_stream
a = torch.rand(m * k, dtype=torch.float64, device="cuda")
b = torch.rand(k * n, dtype=torch.float64, device="cuda")
c = torch.rand(m * n, dtype=torch.float64, device="cuda")
for _ in range(reps):
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st)
torch.cuda.synchronize()
print("ok", m, n, k)
