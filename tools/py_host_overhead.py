"""Host cost of one device-pointer call from Python: engine.dgemm_device vs a raw ctypes my_dgemm_ex (development aid)."""
import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1609_00076_b200 import engine, _capi
mn = k = 256
st = torch.cuda.current_stream().cuda_stream
a = torch.rand(mn*k, dtype=torch.float64, device="cuda"); b = torch.rand(mn*k, dtype=torch.float64, device="cuda"); c = torch.rand(mn*mn, dtype=torch.float64, device="cuda")
for _ in range(10): engine.dgemm_device(mn, mn, k, a.data_ptr(), mn, b.data_ptr(), k, c.data_ptr(), mn, st)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000): engine.dgemm_device(mn, mn, k, a.data_ptr(), mn, b.data_ptr(), k, c.data_ptr(), mn, st)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"python engine.dgemm_device host {((t1-t0)/2000)*1e6:.2f} us/call")
lib = _capi.load(); import ctypes
f = lib.my_dgemm_ex; vp = ctypes.c_void_p(st); pa, pb, pc = a.data_ptr(), b.data_ptr(), c.data_ptr()
t0 = time.perf_counter()
for _ in range(2000): f(mn, mn, k, pa, mn, pb, k, pc, mn, 1, vp)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"python raw ctypes my_dgemm_ex host {((t1-t0)/2000)*1e6:.2f} us/call")
