"""Whole-call time of every launch plan for given shapes (development aid):
python tools/plans_for.py 1500x3000x100 700x700x100 ..."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

PLANS = {0: "heuristic", 2: "128x64", 4: "128x32", 8: "64x32", 16: "16x128", 32: "SK tiles", 34: "SK 128x64",
         36: "SK 128x32", 40: "SK 64x32"}
for spec in sys.argv[1:]:
    m, n, k = (int(x) for x in spec.split("x"))
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c = torch.empty(m * n, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    row = []
    for p, name in list(PLANS.items()) + [(0, "heuristic again")]:
        run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, strips=p)
        try:
            run(); run(); torch.cuda.synchronize()
        except Exception:
            row.append(f"{name}: n/a")
            continue
        inner = max(1, min(50, int(2e9 / (2.0 * m * n * k))))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(3):
            e0.record()
            for _ in range(inner):
                run()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / inner)
        row.append(f"{name}: {best:.1f}")
    print(f"{spec} us | " + " | ".join(row), flush=True)
