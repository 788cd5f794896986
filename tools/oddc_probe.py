import os, sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine
def probe(m, n, k, lda, ldb, ldc, reps=5):
    st = torch.cuda.current_stream().cuda_stream
    a = torch.empty(lda * k, dtype=torch.float64, device="cuda")
    b = torch.empty(ldb * n, dtype=torch.float64, device="cuda")
    c0 = torch.empty(ldc * n, dtype=torch.float64, device="cuda")
    for t, (buf, r, cc, ld) in enumerate(((a, m, k, lda), (b, k, n, ldb), (c0, m, n, ldc))):
        engine.fill_random_device(buf.data_ptr(), r, cc, ld, 1000 + t, 0, st)
    c = c0.clone()
    run = lambda: engine.dgemm_device(m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, c.data_ptr(), ldc, st)
    run(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); run(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    cc = c0.clone()
    engine.dgemm_device(m, n, k, a.data_ptr(), lda, b.data_ptr(), ldb, cc.data_ptr(), ldc, st)
    torch.cuda.synchronize()
    h = float(cc.view(n, ldc)[:, :m].double().sum())
    best = min(ts)
    print(f"{os.environ.get('MYD_C_INPLACE','copy')} {m}x{n}x{k} ld {lda},{ldb},{ldc}: {best:.3f} ms {2*m*n*k/best/1e9:.2f} TF  sum {h!r}", flush=True)
for s in [(4093, 4099, 257, 4093, 257, 4093), (4096, 4096, 256, 4096, 256, 4097), (8191, 8191, 8191, 8191, 8191, 8191),
          (8192, 8192, 8192, 8192, 8192, 8193), (16384, 16384, 256, 16384, 256, 16385), (2047, 2047, 2047, 2047, 2047, 2047),
          (1000, 1000, 1000, 1001, 1001, 1001)]:
    probe(*s)
