"""Print the planner's choice (MY_DGEMM_PLAN_TRACE) for shapes given as MxNxK (development aid)."""
import os
import sys
os.environ["MY_DGEMM_PLAN_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

for spec in sys.argv[1:]:
    m, n, k = (int(x) for x in spec.split("x"))
    a = torch.zeros(m * k, dtype=torch.float64, device="cuda")
    b = torch.zeros(k * n, dtype=torch.float64, device="cuda")
    c = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
