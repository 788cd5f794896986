"""GEMM-based level-3 BLAS throughput on one GPU (development aid): my_dsyrk,
my_dtrsm, my_dtrmm at square sizes, device-resident, best of 5 (CUDA events),
flop counts n^2 k (syrk) and m^2 n / m n^2 (trsm, trmm), beside cuBLAS through
torch (solve_triangular = dtrsm; A @ A^T = a full dgemm for syrk)."""
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


sizes = [int(a) for a in sys.argv[1:]] or [2048, 4096, 8192]
for n in sizes:
    A = torch.rand(n, n, dtype=torch.float64, device="cuda") * 2 - 1
    T = torch.tril(A) / n ** 0.5 + torch.eye(n, dtype=torch.float64, device="cuda") * 2
    B = torch.rand(n, n, dtype=torch.float64, device="cuda") * 2 - 1
    C = torch.rand(n, n, dtype=torch.float64, device="cuda")
    # column-major views: a torch row-major (n, n) tensor is the transpose; fine for timing
    f3 = 1.0 * n ** 3
    ms = timed(lambda: engine.dsyrk("L", "N", n, n, -1.0, A, n, 1.0, C, n))
    msg = timed(lambda: torch.mm(A, A.t()))
    print(f"dsyrk  n={n}: {ms:8.3f} ms  {f3 / ms / 1e9:6.2f} TF/s (n^2 k) | cuBLAS full A A^T {msg:8.3f} ms", flush=True)
    Bw = B.clone()
    for side in "LR":
        ms = timed(lambda: engine.dtrsm(side, "L", "N", "N", n, n, 1.0, T, n, Bw, n))
        msc = timed(lambda: torch.linalg.solve_triangular(T, B, upper=False, left=(side == "L")))
        print(f"dtrsm  {side} n={n}: {ms:8.3f} ms  {f3 / ms / 1e9:6.2f} TF/s | cuBLAS dtrsm {msc:8.3f} ms "
              f"({f3 / msc / 1e9:6.2f} TF/s)", flush=True)
        Bw.copy_(B)
        ms = timed(lambda: engine.dtrmm(side, "L", "N", "N", n, n, 1.0, T, n, Bw, n))
        print(f"dtrmm  {side} n={n}: {ms:8.3f} ms  {f3 / ms / 1e9:6.2f} TF/s", flush=True)
        Bw.copy_(B)
