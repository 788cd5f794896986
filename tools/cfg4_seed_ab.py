"""cfg4 (16384^2 x 256) with three operand sets in one process -- the shape_time.py seeds, the reference generator seeds, A = 0 -- best of 20 single calls each, three rounds (development aid: the time does not depend on the values; the 2-3 % cfg4 difference between runs that day was a code regression, profiles/r02/cfg4_box_variation_r02a.log)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine
m, n, k = 16384, 16384, 256
st = torch.cuda.current_stream().cuda_stream
def mk(seeds):
    a = torch.empty(m * k, dtype=torch.float64, device="cuda"); b = torch.empty(k * n, dtype=torch.float64, device="cuda"); c = torch.empty(m * n, dtype=torch.float64, device="cuda")
    for buf, r, cc, s in ((a, m, k, seeds[0]), (b, k, n, seeds[1]), (c, m, n, seeds[2])):
        engine.fill_random_device(buf.data_ptr(), r, cc, r, s, 0, st)
    return a, b, c
def t(ops, reps=20):
    a, b, c = ops
    for _ in range(2): engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st)
    torch.cuda.synchronize(); best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    return best
A = mk((1000, 1001, 1002))
B = mk(tuple(engine.operand_seed(42, r, m, n, k) for r in (1, 2, 3)))
Z = mk((5, 6, 7)); Z[0].zero_()
for rnd in range(3):
    print(f"round {rnd}: shape_time seeds {t(A):.1f} us | reference seeds {t(B):.1f} us | A = 0 {t(Z):.1f} us", flush=True)
