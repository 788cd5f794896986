"""Device time of my_dgemm on device-resident operands for the given shapes
(development aid): best and median of back-to-back calls.

  python tools/shape_time.py 16384x16384x256 8192x8192x8192 [--reps N] [--ldc-odd]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import engine

args = [a for a in sys.argv[1:] if not a.startswith("--")]
reps = int(next((a.split("=")[1] for a in sys.argv[1:] if a.startswith("--reps=")), 5))
odd = "--ldc-odd" in sys.argv
tag = os.environ.get("SHAPE_TAG", "")
st = torch.cuda.current_stream().cuda_stream
for spec in args:
    m, n, k = (int(v) for v in spec.split("x"))
    ldc = m + 1 if odd else m
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c = torch.empty(ldc * n, dtype=torch.float64, device="cuda")
    for t, (buf, r, cc, ld) in enumerate(((a, m, k, m), (b, k, n, k), (c, m, n, ldc))):
        engine.fill_random_device(buf.data_ptr(), r, cc, ld, 1000 + t, 0, st)
    run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), ldc, st)  # noqa: E731
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    inner = max(1, int(2e11 / (2.0 * m * n * k)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        for _ in range(inner):
            run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / inner)
    ts.sort()
    best, med = ts[0], ts[len(ts) // 2]
    tf = 2.0 * m * n * k / best / 1e9
    print(f"{tag} {m}x{n}x{k}{' ldc-odd' if odd else ''}: best {best * 1e3:.1f} us median {med * 1e3:.1f} us "
          f"{tf:.2f} TF {tf / 37.22 * 100:.2f}%", flush=True)
