"""Short-K shapes with odd / even ldc (development aid; profiles/oddc_short_k_r01.log)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine
label = sys.argv[1] if len(sys.argv) > 1 else "product"
for (m, n, k, ldc_pad) in [(12000, 12000, 100, 0), (12001, 12001, 100, 0), (12001, 12001, 100, 1), (12000, 12000, 96, 0),
                            (12001, 12001, 128, 0), (12001, 12001, 128, 1), (16384, 16384, 256, 0), (16384, 16384, 256, 1),
                            (8192, 8192, 8192, 1), (4093, 4099, 2047, 0)]:
    lda, ldb, ldc = m, k, m + ldc_pad
    a = torch.empty(lda * k, dtype=torch.float64, device="cuda"); b = torch.empty(ldb * n, dtype=torch.float64, device="cuda"); c = torch.empty(ldc * n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for t, (buf, r, cc, ld) in enumerate(((a, m, k, lda), (b, k, n, ldb), (c, m, n, ldc))):
        engine.fill_random_device(buf.data_ptr(), r, cc, ld, 1000 + t, 0, st)
    run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), ldc, st)
    run(); run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(4):
        e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3)
    t = min(ts)
    print(f"{label:8s} {m}x{n}x{k} lda {lda} ldb {ldb} ldc {ldc}: {t:9.1f} us  {2.0*m*n*k/t/1e6/37.22*100:5.1f}%", flush=True)
    del a, b, c
