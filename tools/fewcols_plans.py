"""Few-column / few-row shapes just above the bandwidth kernels' range (17..64):
time per launch plan (development aid)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

PLANS = {0: "heuristic", 2: "128x64", 4: "128x32", 8: "64x32", 16: "16x128", 34: "SK 128x64", 36: "SK 128x32",
         40: "SK 64x32"}
shapes = [(8192, 17, 8192), (8192, 32, 8192), (8192, 48, 8192), (8192, 64, 8192), (16384, 32, 8192),
          (32, 8192, 8192), (48, 8192, 8192), (17, 8192, 8192), (8192, 96, 8192), (8192, 128, 8192)]
for (m, n, k) in shapes:
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c = torch.empty(m * n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    row = []
    for p, name in PLANS.items():
        run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, strips=p)
        try:
            run(); run(); torch.cuda.synchronize()
        except Exception:
            row.append(f"{name}: n/a")
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
        row.append(f"{name}: {min(ts):.0f}")
    gb = 8.0 * (m * k + k * n + 2 * m * n) / 1e9
    print(f"{m}x{n}x{k} ({gb:.2f} GB, {2.0*m*n*k/1e9:.1f} GFLOP) us | " + " | ".join(row), flush=True)
