"""BLAS epilogue cost by (alpha, beta) at short and long K (development aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import engine


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


n = 8192
A = torch.rand(n * n, dtype=torch.float64, device="cuda")
B = torch.rand(n * n, dtype=torch.float64, device="cuda")
C = torch.rand(n * n, dtype=torch.float64, device="cuda")
for (m, nn, k) in [(8192, 8192, 512), (8192, 8192, 256), (8192, 8192, 2048)]:
    for a, b in [(1.0, 1.0), (-1.0, 1.0), (1.0, 0.5), (1.0, 0.0), (2.0, 0.0)]:
        ms = timed(lambda: engine.dgemm("N", "N", m, nn, k, a, A, n, B, n, b, C, n))
        print(f"{m}x{nn}x{k} alpha={a} beta={b}: {ms * 1e3:9.1f} us  {2 * m * nn * k / ms / 1e9:6.2f} TF/s", flush=True)
