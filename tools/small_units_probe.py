"""Sub-wave problems: per-plan time of the small unit shapes (32x32 = 17,
16x32 = 18) against 64x32 units (8), 128x32 (4), 128x64 (2) and the
heuristic (0), back-to-back calls (as tools/sweep.py times them) and single
calls; every plan's C must be bitwise the 64x32 plan's (development aid,
profiles/small_units_r02*.log)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import engine

PLANS = {0: "heur", 8: "64x32", 17: "32x32", 18: "16x32", 4: "128x32", 2: "128x64"}
shapes = [(s, s, s) for s in (256, 384, 512, 640, 768, 1024)] + [
    (128, 128, 2048), (256, 256, 4096), (64, 64, 512), (100, 300, 1000), (200, 200, 200), (512, 256, 1024)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
st = torch.cuda.current_stream().cuda_stream
for (m, n, k) in shapes:
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c0 = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c0, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    ref = c0.clone()
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, ref.data_ptr(), m, st, strips=8)
    row = []
    for p, name in PLANS.items():
        cc = c0.clone()
        engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, cc.data_ptr(), m, st, strips=p)
        torch.cuda.synchronize()
        same = torch.equal(cc, ref)
        c = c0.clone()
        run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st,  # noqa: E731
                                          strips=p)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        reps = max(20, int(3e6 / (m * n * k / 1e3)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b2b = 1e9
        for _ in range(3):
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            b2b = min(b2b, e0.elapsed_time(e1) * 1e3 / reps)
        single = 1e9
        for _ in range(20):
            e0.record()
            run()
            e1.record()
            torch.cuda.synchronize()
            single = min(single, e0.elapsed_time(e1) * 1e3)
        tf = 2.0 * m * n * k / b2b / 1e6
        row.append(f"{name}: {b2b:.2f}/{single:.2f} us {tf / 37.22 * 100:.1f}%{'' if same else ' MISMATCH'}")
    print(f"{m}x{n}x{k} | " + " | ".join(row), flush=True)
