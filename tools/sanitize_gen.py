"""Small config-2-shaped workload for compute-sanitizer (racecheck /
synccheck / memcheck): the fused 2D kernel on a 1024 x 512 window of the
config-2 map (the same tiles, octave plan, shared-memory staging and TMA
store as the full map), launched twice back to back on one stream (the
programmatic-dependent-launch path), plus one config-4-shaped 3D block, the
permutation-table Perlin and OpenSimplex kernels, and the analysis kernels
on the map.

    compute-sanitizer --tool racecheck python tools/sanitize_gen.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1610_03525_b200 as pt  # noqa: E402
from paper_1610_03525_b200 import _abi  # noqa: E402

lib = _abi.load()
s = torch.cuda.current_stream().cuda_stream
cfg = pt.FbmConfig(seed=1, smoothstep=5, resolution=4096, base_frequency=8, octaves=12).to_c()
a = torch.empty((512, 1024), dtype=torch.float32, device="cuda")
b = torch.empty((512, 1024), dtype=torch.float32, device="cuda")
assert lib.tg_fbm_generate_rect_f32(C.byref(cfg), 0, 0, 1024, 512, a.data_ptr(), 1024, s) == 0, _abi.last_error()
assert lib.tg_fbm_generate_rect_f32(C.byref(cfg), 0, 0, 1024, 512, b.data_ptr(), 1024, s) == 0, _abi.last_error()
torch.cuda.synchronize()
assert torch.equal(a, b)
v = torch.empty((64, 64, 128), dtype=torch.float32, device="cuda")
pt.generate3d_device(pt.FbmConfig(method=1, seed=1, resolution=512, base_frequency=8, octaves=8), (0, 0, 0),
                     (64, 64, 128), v)
for m in (pt.Method.perlin_perm, pt.Method.opensimplex, pt.Method.perlin5, pt.Method.generic):
    c = pt.FbmConfig(method=m, seed=1, resolution=4096, base_frequency=8, octaves=12).to_c()
    assert lib.tg_fbm_generate_rect_f32(C.byref(c), 0, 0, 256, 128, b.data_ptr(), 1024, s) == 0, _abi.last_error()
med = C.c_float()
assert lib.tg_median_f32(a.data_ptr(), a.numel(), C.byref(med), s) == 0
sz = (C.c_int32 * 6)(2, 4, 8, 16, 32, 64)
cnt = (C.c_int64 * 6)()
x, y = C.c_int64(), C.c_int64()
assert lib.tg_coastline_boxcount_band(a.data_ptr(), 1024, 512, 1024, 0, 0, med.value, sz, 6, cnt, C.byref(x),
                                      C.byref(y), s) == 0
lg = (C.c_int32 * 4)(1, 2, 64, 4096)
ss, pr = (C.c_double * 8)(), (C.c_int64 * 8)()
assert lib.tg_variogram_f32(a.data_ptr(), 1024, 512, 1024, lg, 4, ss, pr, s) == 0
torch.cuda.synchronize()
print("sanitize workload ok", float(a.abs().max()), list(cnt))
