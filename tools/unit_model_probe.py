"""Per-round and per-launch cost of every unit shape of the persistent kernel (planner model
refit, round 2): forced plan s on shapes with exactly r * 148 units, K from 64 to 4096,
back-to-back calls.  Prints time per call and the least-squares (fixed, per-round) pair per
(s, K) -> profiles/r02/unit_model_r02a.log."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1609_00076_b200 import engine

st = torch.cuda.current_stream().cuda_stream
M = 37 * 128
Ks = [64, 128, 256, 512, 1024, 2048, 4096]
ROUNDS = [1, 2, 3, 4, 6, 8]
for s, ncol in ((1, 512), (2, 256), (4, 128), (8, 64)):
    for K in Ks:
        ts = []
        for r in ROUNDS:
            N = ncol * r
            if s == 8 and N % 128:
                N += 64  # (a half tile column: its units exist but one strip pair is empty)
                continue
            a = torch.empty(M * K, dtype=torch.float64, device="cuda")
            b = torch.empty(K * N, dtype=torch.float64, device="cuda")
            c = torch.empty(M * N, dtype=torch.float64, device="cuda")
            for t, (buf, rr, cc) in enumerate(((a, M, K), (b, K, N), (c, M, N))):
                engine.fill_random_device(buf.data_ptr(), rr, cc, rr, 1000 + t, 0, st)
            run = lambda: engine.dgemm_device(M, N, K, a.data_ptr(), M, b.data_ptr(), K, c.data_ptr(), M, st, strips=s)  # noqa: E731
            run(); run(); torch.cuda.synchronize()
            inner = max(3, min(100, int(1e9 / (2.0 * M * N * K))))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            best = 1e9
            for _ in range(3):
                e0.record()
                for _ in range(inner):
                    run()
                e1.record()
                torch.cuda.synchronize()
                best = min(best, e0.elapsed_time(e1) * 1e3 / inner)
            ts.append((r, best))
        ideal = 2.0 * 128 * 128 / s * K / 251.5e3
        A = np.array([[1.0, r] for r, _ in ts])
        y = np.array([t for _, t in ts])
        sol = np.linalg.lstsq(A, y, rcond=None)[0]
        print(f"s={s} K={K}: ideal/round {ideal:.2f} us | " + " ".join(f"r{r}:{t:.1f}" for r, t in ts) +
              f" | fit fixed {sol[0]:.2f} per-round {sol[1]:.2f} (= ideal/{ideal / sol[1]:.3f}; ideal/0.99 + {sol[1] - ideal / 0.99:.2f})",
              flush=True)
