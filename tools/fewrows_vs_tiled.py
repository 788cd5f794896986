import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import engine, _capi
st = torch.cuda.current_stream().cuda_stream
def t(fn):
    fn(); torch.cuda.synchronize(); best=1e9
    for _ in range(10):
        e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); e0.record(); fn(); e1.record(); torch.cuda.synchronize(); best=min(best,e0.elapsed_time(e1)*1e3)
    return best
SHAPES = [(m, n, 8192) for m in (2, 3, 4, 5, 6, 8) for n in (2048, 4096, 8192, 16384, 32768)] + \
    [(4, 65536, 4096), (4, 131072, 2048), (2, 131072, 2048), (8, 65536, 2048), (6, 50000, 3000)]
for m,n,k in SHAPES:
    a=torch.rand(m*k,dtype=torch.float64,device="cuda"); b=torch.rand(k*n,dtype=torch.float64,device="cuda"); c=torch.rand(m*n,dtype=torch.float64,device="cuda")
    r={}
    for p in (_capi.PATH_FEW_ROWS, _capi.PATH_TILED):
        r[p]=t(lambda: engine.dgemm_device(m,n,k,a.data_ptr(),m,b.data_ptr(),k,c.data_ptr(),m,st,path=p))
    byts=8.0*(m*k+k*n+2*m*n)
    print(f"{m}x{n}x{k}: few-rows {r[4]:.1f} us ({byts/r[4]/1e3:.0f} GB/s) | tiled {r[0]:.1f} us ({byts/r[0]/1e3:.0f} GB/s) | default path {engine.path(m,n)}", flush=True)
