"""tg_coastline_boxcount_band on the config-5 map (32768^2), sea = 0, sizes
2..64: wall time of the synchronous call (REPS times) for an ncu launch list."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1610_03525_b200 as pt  # noqa: E402
from paper_1610_03525_b200 import _abi  # noqa: E402

T = int(os.environ.get("TG_R", "32768"))
lib = _abi.load()
c = pt.FbmConfig(seed=1, smoothstep=5, resolution=32768, base_frequency=32, octaves=16).to_c()
m = torch.empty((T, T), dtype=torch.float32, device="cuda")
assert lib.tg_fbm_generate_rect_f32(C.byref(c), 0, 0, T, T, m.data_ptr(), T, None) == 0
sz = (C.c_int32 * 6)(2, 4, 8, 16, 32, 64)
cnt = (C.c_int64 * 6)()
a, b = C.c_int64(), C.c_int64()
for i in range(int(os.environ.get("REPS", "3"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    assert lib.tg_coastline_boxcount_band(m.data_ptr(), T, T, T, 0, 0, -0.02631, sz, 6, cnt, C.byref(a), C.byref(b),
                                          None) == 0
    print(f"coast+box {1e3 * (time.perf_counter() - t0):.3f} ms  counts {list(cnt)} coast {a.value} land {b.value}")
