import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1609_00076_b200 import engine
st = torch.cuda.current_stream().cuda_stream
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize(); best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
n = 8192
A = torch.rand(n * n, dtype=torch.float64, device="cuda"); B = torch.rand(n * n, dtype=torch.float64, device="cuda")
C = torch.rand(n * n, dtype=torch.float64, device="cuda")
for (m, nn, k) in [(7680, 8192, 512), (4096, 8192, 512), (512, 8192, 512), (512, 8192, 7680), (512, 8192, 4096), (384, 8192, 128), (96, 8192, 32), (32, 8192, 32)]:
    for s in (1.0, -1.0):
        ms = timed(lambda: engine.dgemm("N", "N", m, nn, k, s, A, n, B, n, 1.0, C, n))
        print(f"{m}x{nn}x{k} alpha={s}: {ms*1e3:9.1f} us  {2*m*nn*k/ms/1e9:6.2f} TF/s", flush=True)
