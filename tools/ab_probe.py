"""A/B timing of library variants (MY_DGEMM_LIB=...) on device-resident
operands: python tools/ab_probe.py [label] (development aid)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

SHAPES = [(16384, 16384, 256), (8192, 8192, 256), (16384, 16384, 128), (16384, 16384, 512), (1024, 1024, 1024),
          (2048, 2048, 2048), (4096, 4096, 4096), (8192, 8192, 8192), (4093, 4099, 2047)]
label = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("MY_DGEMM_LIB", "product")
for (m, n, k) in SHAPES:
    lda, ldb, ldc = (m + 7, k + 5, m + 3) if m == 4093 else (m, k, m)
    a = torch.empty(lda * k, dtype=torch.float64, device="cuda")
    b = torch.empty(ldb * n, dtype=torch.float64, device="cuda")
    c = torch.empty(ldc * n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for t, (buf, r, cc, ld) in enumerate(((a, m, k, lda), (b, k, n, ldb), (c, m, n, ldc))):
        engine.fill_random_device(buf.data_ptr(), r, cc, ld, 1000 + t, 0, st)
    run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), ldc, st)
    reps = 3 if m * n * k >= 8192 ** 3 else 10
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts.sort()
    tf = 2.0 * m * n * k / ts[0] / 1e9
    print(f"{label:10s} {m}x{n}x{k}: best {ts[0]*1e3:9.1f} us  median {ts[len(ts)//2]*1e3:9.1f} us  "
          f"{tf:6.2f} TF ({tf / 37.22 * 100:5.1f}%)", flush=True)
    del a, b, c
