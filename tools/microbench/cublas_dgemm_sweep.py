"""cuBLAS DGEMM (torch addmm_, C += A B) vs this engine over the sweep sizes
(a comparison reference only; cuBLAS is never on the product path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

from paper_1609_00076_b200 import engine

sizes = [int(x) for x in sys.argv[1:]] or [256, 512, 768, 1024, 1280, 1536, 1792, 2048, 2560, 2816, 3072, 4096,
                                           6144, 8192]
st = torch.cuda.current_stream().cuda_stream


def timed(fn, inner):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(inner):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / inner)
    return best


for n in sizes:
    a = torch.rand(n, n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, n, dtype=torch.float64, device="cuda")
    c = torch.rand(n, n, dtype=torch.float64, device="cuda")
    inner = max(1, int(2e10 / (2.0 * n ** 3)))
    t_cb = timed(lambda: c.addmm_(a, b), inner)
    t_me = timed(lambda: engine.dgemm_device(n, n, n, a.data_ptr(), n, b.data_ptr(), n, c.data_ptr(), n, st), inner)
    f = 2.0 * n ** 3 / 1e6
    print(f"n={n}: cuBLAS {t_cb:.1f} us {f / t_cb:.2f} TF | b200 {t_me:.1f} us {f / t_me:.2f} TF | ratio {t_cb / t_me:.2f}x",
          flush=True)
