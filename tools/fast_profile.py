"""Read the MYD_FAST_PROFILE counters of an instrumented variant build."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1609_00076_b200 import _capi, engine
lib = _capi.load()
fn = lib.my_dgemm_fast_profile
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
m = n = k = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
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
tiles = ((m + 127) // 128) * ((n + 127) // 128)
cw = tiles * 8
print(f"time {e0.elapsed_time(e1):.3f} ms  ({2*m*n*k/e0.elapsed_time(e1)/1e9:.2f} TF)")
print(f"consumer loop cycles/warp-tile {v[5]/cw:.0f}; slow waits {v[1]} ({v[1]/cw:.1f}/warp-tile), "
      f"cycles in slow waits/warp-tile {v[0]/cw:.0f}; first-slab wait/warp-tile {v[4]/cw:.0f}")
print(f"producer empty waits {v[3]} cycles/producer-tile {v[2]/(tiles*4):.0f}")
