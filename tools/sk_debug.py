import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch, numpy as np
from paper_1609_00076_b200 import engine
import oracle
def run(m,n,k,lda,ldb,ldc,strips):
    s=[oracle.operand_seed(42, r, m, n, k) for r in (1,2,3)]
    st=torch.cuda.current_stream().cuda_stream
    def mk(r,c,ld,seed):
        b=torch.full((ld*c,), -777.25, dtype=torch.float64, device="cuda"); engine.fill_random_device(b.data_ptr(), r, c, ld, seed, 0, st); return b
    a=mk(m,k,lda,s[0]); b=mk(k,n,ldb,s[1]); c=mk(m,n,ldc,s[2])
    outs={}
    for sp in strips:
        cc=c.clone(); engine.dgemm_device(m,n,k,a.data_ptr(),lda,b.data_ptr(),ldb,cc.data_ptr(),ldc,st,strips=sp); torch.cuda.synchronize(); outs[sp]=cc.cpu().numpy().reshape(n,ldc)
    for sp in strips[1:]:
        d=np.argwhere(outs[sp]!=outs[strips[0]])
        print(m,n,k,"strips",sp,"mismatches",len(d), "first (col,row)", d[:3].tolist() if len(d) else None, "cols range", (d[:,0].min(), d[:,0].max()) if len(d) else None, "rows", (d[:,1].min(), d[:,1].max()) if len(d) else None)
run(4093,4099,200,4100,202,4096,[0,34,36,40,32])
run(4096,4096,200,4096,200,4096,[0,34,36,40])
run(4093,4096,200,4094,200,4094,[0,34,36,40])
run(4096,4099,200,4096,200,4096,[0,34,36,40])
