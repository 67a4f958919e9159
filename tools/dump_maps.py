"""Dump maps of the timing configs with the library in TG_LIB_PATH, or compare two dumps.

    python tools/dump_maps.py dump TAG      -> /tmp/tg_maps_TAG.npz
    python tools/dump_maps.py cmp TAG_A TAG_B
Used to check that a kernel variant reproduces the previous bits.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

if sys.argv[1] == "cmp":
    a = np.load(f"/tmp/tg_maps_{sys.argv[2]}.npz")
    b = np.load(f"/tmp/tg_maps_{sys.argv[3]}.npz")
    for k in a.files:
        d = np.abs(a[k].astype(np.float64) - b[k].astype(np.float64))
        print(f"{k:8s} identical={np.array_equal(a[k], b[k])} max|d|={d.max():.3e} amp={np.abs(a[k]).max():.3f}")
    sys.exit(0)

import torch  # noqa: E402

import paper_1610_03525_b200 as pt  # noqa: E402
CONFIGS = {
    "cfg1": (dict(seed=1, resolution=1024, base_frequency=8, octaves=8), 1024, 1024),
    "cfg2": (dict(seed=1, smoothstep=5, resolution=4096, base_frequency=8, octaves=12), 4096, 4096),
    "cfg2sep": (dict(seed=1, method=pt.Method.zg_separable, smoothstep=5, resolution=4096, base_frequency=8,
                     octaves=12), 4096, 4096),
    "cfg3p": (dict(seed=1, method=pt.Method.perlin3, resolution=4096, base_frequency=8, octaves=12), 4096, 4096),
    "cfg3g": (dict(seed=1, method=pt.Method.generic, resolution=4096, base_frequency=8, octaves=12), 4096, 4096),
    "cfg5": (dict(seed=1, smoothstep=5, resolution=32768, base_frequency=32, octaves=16), 4096, 4096),
}

out = {}
for name in ("cfg1", "cfg2", "cfg2sep", "cfg3p", "cfg3g", "cfg5"):
    kw, w, h = CONFIGS[name]
    buf = torch.empty((h, w), dtype=torch.float32, device="cuda")
    pt.generate_rect_device(pt.FbmConfig(**kw), (0, 0), w, h, buf)
    out[name] = buf.cpu().numpy()
c4 = pt.FbmConfig(seed=1, method=pt.Method.zg_separable, resolution=512, base_frequency=8, octaves=8)
for name, org, ext in (("cfg4", (0, 0, 0), (256, 256, 256)), ("cfg4odd", (64, 0, 128), (40, 72, 100))):
    v = torch.empty(ext, dtype=torch.float32, device="cuda")  # (nz, ny, nx)
    pt.generate3d_device(c4, org, ext, v)
    out[name] = v.cpu().numpy()
np.savez(f"/tmp/tg_maps_{sys.argv[2]}.npz", **out)
print("dumped", sys.argv[2])
