"""16x128-unit throughput (few-row and ragged-row shapes) for A/B of staging variants (development aid)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

label = sys.argv[1] if len(sys.argv) > 1 else "product"
CASES = [(16, 8192, 8192, 0), (12, 9000, 4096, 0), (16, 65536, 2048, 0), (32, 8192, 8192, 0), (32, 8192, 8192, 8),
         (32, 8192, 8192, 16), (64, 8192, 8192, 0), (64, 8192, 8192, 8), (64, 8192, 8192, 16), (2048, 2048, 2048, 16),
         (4100, 3000, 2000, 0), (4100, 3000, 2000, 8), (4100, 3000, 2000, 16), (8, 8192, 8192, 0), (8, 8192, 8192, 16),
         (4, 65536, 4096, 0), (4, 65536, 4096, 16), (100, 8192, 8192, 0), (100, 8192, 8192, 8)]
for (m, n, k, strips) in CASES:
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c = torch.empty(m * n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, strips=strips)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    t = min(ts) * 1e-3
    gbs = 8.0 * (m * k + k * n + 2 * m * n) / t / 1e9
    tf = 2.0 * m * n * k / t / 1e12
    print(f"{label:8s} {m}x{n}x{k} strips={strips}: {t*1e6:9.1f} us  {tf:6.2f} TF  {gbs:7.1f} GB/s", flush=True)
