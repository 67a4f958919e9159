import ctypes as C, sys
sys.path.insert(0, '/root/repo')
import torch, paper_1610_03525_b200 as pt
from paper_1610_03525_b200 import _abi
lib = _abi.load(); R = 32768
cfg = pt.FbmConfig(seed=1, smoothstep=5, resolution=R, base_frequency=32, octaves=14)
m = torch.empty((R, R), dtype=torch.float32, device='cuda'); pt.generate_into_device(cfg, (0, 0), R, m)
sizes = (C.c_int32 * 6)(2, 4, 8, 16, 32, 64); cnt = (C.c_int64 * 6)(); a, b = C.c_int64(), C.c_int64()
for _ in range(2): lib.tg_coastline_boxcount(m.data_ptr(), R, 0.0, sizes, 6, cnt, C.byref(a), C.byref(b), None)
torch.cuda.synchronize()
