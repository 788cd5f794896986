"""Roofline scan over a grid of shapes (development aid): for each (m, n, k)
the default call's time against max(2mnk / 37.22 TF, 8(mk+kn+2mn) / 6.55 TB/s)
plus a fixed 5 us launch floor; prints the worst fractions first."""
import itertools
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

MS = [int(x) for x in os.environ.get("SCAN_MS", "17,64,100,200,300,600,1000,2000,4000,8000").split(",")]
KS = [int(x) for x in os.environ.get("SCAN_KS", "64,512,4096").split(",")]
res = []
st = torch.cuda.current_stream().cuda_stream
for m, n, k in itertools.product(MS, MS, KS):
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st)
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    inner = max(1, min(50, int(2e9 / (2.0 * m * n * k))))
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(inner):
            run()
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / inner)
    floor = max(2.0 * m * n * k / 37.22e6, 8.0 * (m * k + k * n + 2 * m * n) / 6.55e6) + 5.0
    res.append((floor / best, m, n, k, best, floor, engine.path(m, n)))
    del a, b, c
res.sort()
for frac, m, n, k, t, f, p in res:
    print(f"{m:5d}x{n:5d}x{k:5d} path {p}: {t:9.1f} us  floor {f:8.1f} us  {frac*100:5.1f}%", flush=True)
