"""K-split plan (strips=48) against the plan-invariant heuristic (strips=-1) and the default
heuristic (strips=0) on mid-size problems: time (back-to-back calls, as tools/sweep.py times
them), max |C - C_exact| against the exact kernel with the c = 2 bound, run-to-run bitwise
determinism.  Evidence for the planner's K-split cost (profiles/r02/ksplit_r02*.log).

    python tools/ksplit_probe.py [m,n,k | s] ...
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine

EPS = 2.0 ** -52
shapes = []
for arg in sys.argv[1:]:
    p = [int(x) for x in arg.split(",")]
    shapes.append(tuple(p) if len(p) == 3 else (p[0], p[0], p[0]))
if not shapes:
    shapes = [(s, s, s) for s in (512, 640, 768, 896, 1024, 1152, 1280, 1408, 1536)] + \
             [(1024, 1024, 4096), (2048, 512, 2048), (1000, 1100, 1200), (896, 1664, 300), (4096, 256, 1024)]
st = torch.cuda.current_stream().cuda_stream
for (m, n, k) in shapes:
    a = torch.empty(m * k, dtype=torch.float64, device="cuda")
    b = torch.empty(k * n, dtype=torch.float64, device="cuda")
    c0 = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for t, (buf, r, cc) in enumerate(((a, m, k), (b, k, n), (c0, m, n))):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, 1000 + t, 0, st)
    ref = c0.clone()
    engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, ref.data_ptr(), m, st, exact=True)
    tol = 2 * k * EPS * (k / 3 + 1)  # loose a-priori stand-in for (|A||B|+|C|)max; the tests use the true bound
    row = []
    for p, name in ((-1, "invariant"), (48, "K-split"), (0, "default")):
        outs = []
        for _ in range(2):
            c = c0.clone()
            engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, strips=p)
            outs.append(c)
        torch.cuda.synchronize()
        det = bool(torch.equal(outs[0], outs[1]))
        err = float((outs[0] - ref).abs().max())
        c = c0.clone()
        run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st, strips=p)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        reps = max(5, int(2e6 / (m * n * k / 1e3)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(3):
            e0.record()
            for _ in range(reps):
                run()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
        tf = 2.0 * m * n * k / best / 1e6
        row.append(f"{name}: {best:.1f} us {tf / 37.22 * 100:.1f}% err {err:.2e}{'' if det else ' NONDETERMINISTIC'}"
                   f"{'' if err <= tol else ' OVER-TOL'}")
    print(f"{m}x{n}x{k} | " + " | ".join(row), flush=True)
