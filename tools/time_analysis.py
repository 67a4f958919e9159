"""Time the analysis pass pieces on a config-2 map (wall clock around the
synchronous C-ABI calls, and CUDA events for the device time)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1610_03525_b200 as pt  # noqa: E402
from paper_1610_03525_b200 import _abi  # noqa: E402

R = int(os.environ.get("TG_R", "4096"))
cfg = pt.FbmConfig(seed=1, smoothstep=5, resolution=R, base_frequency=8, octaves=12)
m = torch.empty((R, R), dtype=torch.float32, device="cuda")
pt.generate_into_device(cfg, (0, 0), R, m)
torch.cuda.synchronize()
lib = _abi.load()


def bench(name, fn, n=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    print(f"{name:28s} {(time.perf_counter() - t0) / n * 1e3:8.3f} ms")


out = C.c_float()
bench("median (3-pass radix)", lambda: lib.tg_median_f32(m.data_ptr(), m.numel(), C.byref(out), None))
sea = out.value
sizes = (C.c_int32 * 6)(2, 4, 8, 16, 32, 64)
cnt = (C.c_int64 * 6)()
a, b = C.c_int64(), C.c_int64()
bench("coastline+boxcount", lambda: lib.tg_coastline_boxcount(m.data_ptr(), R, sea, sizes, 6, cnt, C.byref(a),
                                                             C.byref(b), None))
mask = torch.empty((R, R), dtype=torch.uint8, device="cuda")
bench("coastline mask u8", lambda: lib.tg_coastline_mask(m.data_ptr(), R, sea, mask.data_ptr(), C.byref(a), None))
hist = np.zeros(2048, dtype=np.uint64)
bench("histogram pass", lambda: lib.tg_histogram_f32(m.data_ptr(), R, R, R, 0, 0, 21, 11, hist.ctypes.data, None))
lags = (C.c_int32 * 12)(*[1 << i for i in range(12)])
ss = (C.c_double * 24)()
pr = (C.c_int64 * 24)()
bench("variogram 12 lags x 2 axes", lambda: lib.tg_variogram_f32(m.data_ptr(), R, R, R, lags, 12, ss, pr, None))
lo, hi = C.c_double(), C.c_double()
bench("minmax", lambda: lib.tg_minmax_f32(m.data_ptr(), m.numel(), C.byref(lo), C.byref(hi), None))
bench("generate (for scale)", lambda: pt.generate_into_device(cfg, (0, 0), R, m))
print("counts", list(cnt), "sea", sea)
