"""Few-row shapes: the 2 <= m <= 16 bandwidth kernel vs the tiled kernel
(FORCE_TILED), device time and GB/s over 8(mk + kn + 2mn) (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import engine

st = torch.cuda.current_stream().cuda_stream


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    return best


shapes = [(2, 8192, 8192), (4, 8192, 8192), (8, 8192, 8192), (16, 8192, 8192), (4, 100000, 2000),
          (16, 4096, 4096), (8, 32768, 8192), (3, 5000, 777), (16, 512, 4096), (8, 256, 8192), (4, 1000, 1000),
          (16, 2048, 2048), (12, 1024, 300)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
for m, n, k in shapes:
    a = torch.rand(m * k, dtype=torch.float64, device="cuda")
    b = torch.rand(k * n, dtype=torch.float64, device="cuda")
    c = torch.rand(m * n, dtype=torch.float64, device="cuda")
    byts = 8.0 * (m * k + k * n + 2 * m * n)
    res = {}
    for tiled in (False, True):
        cc = c.clone()
        res[tiled] = timed(lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, cc.data_ptr(), m,  # noqa: B023
                                                       st, force_tiled=tiled))
    ce, cf = c.clone(), c.clone()
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, ce.data_ptr(), m, st, exact=True)
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, cf.data_ptr(), m, st)
    torch.cuda.synchronize()
    err = float((ce - cf).abs().max())
    print(f"{m}x{n}x{k}: msmall {res[False]:.1f} us ({byts / res[False] / 1e3:.0f} GB/s) | tiled {res[True]:.1f} us "
          f"({byts / res[True] / 1e3:.0f} GB/s) | max|fast-exact| {err:.2e}", flush=True)
