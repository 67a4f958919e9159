import time, numpy as np, torch, sys, ctypes as C
sys.path.insert(0, ".")
import paper_1610_03525_b200 as pt
from paper_1610_03525_b200 import _abi
lib = _abi.load()
n = 4096 * 4096
a = np.ones(n * 2, dtype=np.float64); b = np.empty_like(a)
for _ in range(2): np.copyto(b, a)
t0 = time.perf_counter(); 
for _ in range(5): np.copyto(b, a)
cp = (time.perf_counter() - t0) / 5
d = torch.empty(n, dtype=torch.float32, device="cuda"); h = torch.empty(n, dtype=torch.float32).pin_memory()
for _ in range(3): h.copy_(d)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10): h.copy_(d)
torch.cuda.synchronize(); d2h = (time.perf_counter() - t0) / 10
cfg = pt.FbmConfig(seed=1, smoothstep=5, resolution=4096, base_frequency=8, octaves=12).to_c()
hd = torch.empty(n, dtype=torch.float64).pin_memory()
for _ in range(3): lib.tg_fbm_generate_f64_host(C.byref(cfg), 0, 0, 4096, hd.data_ptr(), n, None)
ts = []
for _ in range(15):
    t0 = time.perf_counter(); lib.tg_fbm_generate_f64_host(C.byref(cfg), 0, 0, 4096, hd.data_ptr(), n, None); ts.append(time.perf_counter() - t0)
print(f"numpy copy 256MiB {2*8*n/cp/1e9:6.1f} GB/s (r+w)   d2h fp32 {4*n/d2h/1e9:5.1f} GB/s   e2e {1e3*sorted(ts)[7]:.3f} ms")
