"""Read the MYD_FAST_PROFILE counters of an instrumented build (per consumer warp-unit)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import _capi, engine
lib = _capi.load()
fn = lib.my_dgemm_fast_profile
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
m, n, k = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else [8192, 8192, 8192]))
st = torch.cuda.current_stream().cuda_stream
a = torch.rand(m * k, dtype=torch.float64, device="cuda")
b = torch.rand(k * n, dtype=torch.float64, device="cuda")
c = torch.rand(m * n, dtype=torch.float64, device="cuda")
engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
fn(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); engine.dgemm_device(m, n, k, a.data_ptr(), m, b.data_ptr(), k, c.data_ptr(), m, st); e1.record()
torch.cuda.synchronize()
fn(buf, 1)
v = list(buf)
wu = max(1, v[7])  # consumer warp-units
ms = e0.elapsed_time(e1)
print(f"{m}x{n}x{k}: {ms:.3f} ms ({2*m*n*k/ms/1e9:.2f} TF); per consumer warp-unit: C-load {v[6]/wu:.0f} cyc, "
      f"first-slab wait {v[4]/wu:.0f}, main loop {v[5]/wu:.0f} (slow waits {v[1]/wu:.2f}, {v[0]/wu:.0f} cyc); "
      f"producer empty-wait {v[2]/max(1,v[3]):.0f} cyc/wait")
