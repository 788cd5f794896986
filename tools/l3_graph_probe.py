"""Is the GEMM-based dtrsm / dtrmm at 1024-4096 host-launch bound?  Time of
back-to-back calls vs the same calls replayed from a CUDA graph (development
aid, profiles/r02/l3_graph_probe_r02a.log)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1609_00076_b200 import engine, kernel_launches

for n in [int(a) for a in sys.argv[1:]] or [1024, 2048, 4096]:
    A = torch.rand(n, n, dtype=torch.float64, device="cuda") * 2 - 1
    A = A + n * torch.eye(n, dtype=torch.float64, device="cuda")
    B = torch.rand(n, n, dtype=torch.float64, device="cuda")
    for name, fn in (("dtrsm", engine.dtrsm), ("dtrmm", engine.dtrmm)):
        X = B.clone()
        call = lambda s=None: fn("L", "L", "N", "N", n, n, 1.0, A, n, X, n, stream=s)  # noqa: E731
        call()
        torch.cuda.synchronize()
        l0 = kernel_launches()
        call()
        torch.cuda.synchronize()
        launches = kernel_launches() - l0
        reps = 20
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        direct = e0.elapsed_time(e1) / reps
        g = torch.cuda.CUDAGraph()
        s2 = torch.cuda.Stream()
        with torch.cuda.stream(s2):
            call(s2.cuda_stream)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s2):
                call(s2.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        graph = e0.elapsed_time(e1) / reps
        print(f"{name} L n={n}: {launches} launches; back-to-back {direct * 1e3:.0f} us, graph replay {graph * 1e3:.0f} us",
              flush=True)
