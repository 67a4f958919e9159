"""Bit-exactness of library variants: maps from TG_LIB_PATH variants compared word for word.

    python tools/bitcmp.py base.so other.so [...]   (paths to .so files)
Runs each variant in a child process (one library per process), dumps the
config-1/2/3/5-chunk maps and reports max |diff| and the count of differing words.
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_1610_03525_b200 as pt
out = {}
cfgs = {
  "cfg1": (dict(seed=7, resolution=1024, base_frequency=8, octaves=8), (0, 0), 1024),
  "cfg2": (dict(seed=1, smoothstep=5, resolution=4096, base_frequency=8, octaves=12), (0, 0), 4096),
  "cfg2sep": (dict(seed=3, method=pt.Method.zg_separable, smoothstep=5, resolution=4096, base_frequency=8, octaves=12), (0, 0), 4096),
  "cfg3g": (dict(seed=1, method=pt.Method.generic, resolution=4096, base_frequency=8, octaves=12), (0, 0), 2048),
  "cfg3p": (dict(seed=1, method=pt.Method.perlin3, resolution=4096, base_frequency=8, octaves=12), (0, 0), 2048),
  "cfg5": (dict(seed=5, smoothstep=5, resolution=32768, base_frequency=32, octaves=16), (31744, 8192), 1024),
}
for k, (kw, org, n) in cfgs.items():
    cfg = pt.FbmConfig(**kw)
    o = torch.empty((n, n), dtype=torch.float32, device="cuda")
    pt.generate_rect_device(cfg, org, n, n, o)
    torch.cuda.synchronize()
    out[k] = o.cpu().numpy()
np.savez(sys.argv[1], **out)
"""
res = []
for i, lib in enumerate(sys.argv[1:]):
    f = f"/tmp/bitcmp_{i}.npz"
    env = dict(os.environ, TG_LIB_PATH=lib)
    subprocess.run([sys.executable, "-c", CHILD % ROOT, f], env=env, check=True)
    res.append(np.load(f))
for i in range(1, len(res)):
    for k in res[0].files:
        a, b = res[0][k].view(np.uint32), res[i][k].view(np.uint32)
        nd = int((a != b).sum())
        md = float(np.abs(res[0][k] - res[i][k]).max())
        print(f"{os.path.basename(sys.argv[1 + i])} {k}: differing words {nd}, max |diff| {md:.3g}")
