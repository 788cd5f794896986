"""Time the m==1 / n==1 kernels (cfg3b / cfg3c) against the HBM roofline."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine
for name, (m, n, k, lda, ldb, ldc) in {"cfg3b": (1, 8192, 8192, 8, 8197, 4),
                                       "cfg3c": (8192, 1, 8192, 8199, 8197, 8195),
                                       "n1_aligned": (8192, 1, 8192, 8192, 8192, 8192),
                                       "m1_aligned": (1, 8192, 8192, 1, 8192, 1)}.items():
    st = torch.cuda.current_stream().cuda_stream
    a = torch.rand(lda * k, dtype=torch.float64, device="cuda")
    b = torch.rand(ldb * n, dtype=torch.float64, device="cuda")
    c = torch.rand(ldc * n, dtype=torch.float64, device="cuda")
    go = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), ldc, st)
    for _ in range(3): go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): go()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 50 * 1e-3
    byts = 8.0 * (m * k + k * n + 2 * m * n)
    print(f"{name}: {t*1e6:.1f} us  {byts/t/1e9:.0f} GB/s ({byts/t/1e9/6550.7*100:.1f}% of 6550.7)", flush=True)
