"""Ragged-K shapes (K mod 16 small) for the zero-k-step skip A/B (development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine
label = sys.argv[1] if len(sys.argv) > 1 else "product"
for (m, n, k) in [(12000, 12000, 100), (12000, 12000, 96), (16384, 16384, 260), (16384, 16384, 256), (8192, 8192, 1028),
                  (8192, 8192, 8196), (8192, 8192, 8192), (4093, 4099, 2047), (2048, 2048, 2050), (16384, 16384, 129)]:
    a = torch.empty(m * k, dtype=torch.float64, device="cuda"); b = torch.empty(k * n, dtype=torch.float64, device="cuda"); c = torch.empty(m * n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st)
    run(); run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(4):
        e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    t = min(ts)
    print(f"{label:8s} {m}x{n}x{k}: {t:9.1f} us  {2.0*m*n*k/t/1e6/37.22*100:5.1f}%", flush=True)
    del a, b, c
