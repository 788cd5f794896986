import torch, sys
sys.path.insert(0, "/root/repo")
from paper_1609_00076_b200 import engine
m = n = 16384; k = 256
a = torch.rand(m, k, dtype=torch.float64, device="cuda"); b = torch.rand(k, n, dtype=torch.float64, device="cuda"); c = torch.rand(m, n, dtype=torch.float64, device="cuda")
def t(fn):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    return best
cb = t(lambda: c.addmm_(a, b))
print(f"cfg4 cuBLAS (torch addmm_): {cb:.3f} ms {2*m*n*k/cb/1e9:.1f} TF")
