"""Variogram debugging / timing: per-lag, per-axis sums against the oracle on
a small map, then device time of each pass at 32768^2 (TG_VG_AXES)."""
import ctypes as C
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1610_03525_b200 as pt  # noqa: E402
from paper_1610_03525_b200 import _abi  # noqa: E402

lib = _abi.load()


def vg(m, W, H, lags):
    lg = (C.c_int32 * len(lags))(*lags)
    ss = (C.c_double * (2 * len(lags)))()
    pr = (C.c_int64 * (2 * len(lags)))()
    assert lib.tg_variogram_f32(m.data_ptr(), W, H, W, lg, len(lags), ss, pr, None) == 0, _abi.last_error()
    return np.array(ss[:]).reshape(-1, 2)


if "--time" not in sys.argv:
    from oracle.pyoracle import Oracle
    o = Oracle()
    for (W, H) in [(1000, 700), (4096, 300), (9000, 40)]:
        cfg = pt.FbmConfig(seed=3, smoothstep=5, resolution=8192, base_frequency=8, octaves=10)
        m = torch.empty((H, W), dtype=torch.float32, device="cuda")
        pt.generate_rect_device(cfg, (0, 0), W, H, m)
        lags = [1, 2, 4, 8, 16, 32, 64, 128, 3, 5, 600]
        got = vg(m, W, H, lags)
        ref, _ = o.variogram(m.cpu().numpy().astype(np.float64), lags)
        rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
        print(W, H)
        for i, h in enumerate(lags):
            print(f"  lag {h:5d}  x {got[i,0]:.6e} / {ref[i,0]:.6e} ({rel[i,0]:.1e})   y {got[i,1]:.6e} / {ref[i,1]:.6e} ({rel[i,1]:.1e})")
else:
    R = 32768
    cfg = pt.FbmConfig(seed=1, smoothstep=5, resolution=R, base_frequency=32, octaves=16)
    m = torch.empty((R, R), dtype=torch.float32, device="cuda")
    pt.generate_into_device(cfg, (0, 0), R, m)
    torch.cuda.synchronize()
    lags = [1 << i for i in range(13)]
    for axes in ("1", "2", "3"):
        r = subprocess.run([sys.executable, "-c", f"""
import os, sys, time, ctypes as C
os.environ['TG_VG_AXES'] = '{axes}'
sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
import torch, paper_1610_03525_b200 as pt
from paper_1610_03525_b200 import _abi
lib = _abi.load()
R = {R}
cfg = pt.FbmConfig(seed=1, smoothstep=5, resolution=R, base_frequency=32, octaves=16)
m = torch.empty((R, R), dtype=torch.float32, device='cuda')
pt.generate_into_device(cfg, (0, 0), R, m)
lags = {lags}
lg = (C.c_int32 * len(lags))(*lags); ss = (C.c_double * 26)(); pr = (C.c_int64 * 26)()
lib.tg_variogram_f32(m.data_ptr(), R, R, R, lg, 13, ss, pr, None)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(3): lib.tg_variogram_f32(m.data_ptr(), R, R, R, lg, 13, ss, pr, None)
print('axes {axes}: %.3f ms' % ((time.perf_counter() - t) / 3 * 1e3))
"""], capture_output=True, text=True)
        print(r.stdout.strip(), r.stderr.strip()[-300:])
