"""One tg_median_f32 call on the config-5 map (32768^2) for an ncu launch list."""
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
out = C.c_float()
for i in range(int(os.environ.get("REPS", "3"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    assert lib.tg_median_f32(m.data_ptr(), m.numel(), C.byref(out), None) == 0
    print(f"median {out.value:.9f}  {1e3 * (time.perf_counter() - t0):.3f} ms")
import numpy as np  # noqa: E402

h = np.zeros(2048, dtype=np.uint64)
for i in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    assert lib.tg_histogram_f32(m.data_ptr(), T, T, T, 0, 0, 21, 11, h.ctypes.data, None) == 0
    print(f"full histogram pass {1e3 * (time.perf_counter() - t0):.3f} ms")
