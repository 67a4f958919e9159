"""Small, repeatable generation run for ncu captures (one process, one GPU).

    python tools/prof_gen.py [--config cfg2|cfg1|cfg3p|cfg5|cfg4] [--iters 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1610_03525_b200 as pt  # noqa: E402

CONFIGS = {
    "cfg1": (dict(seed=1, resolution=1024, base_frequency=8, octaves=8), 1024),
    "cfg2": (dict(seed=1, smoothstep=5, resolution=4096, base_frequency=8, octaves=12), 4096),
    "cfg3p": (dict(seed=1, method=pt.Method.perlin3, resolution=4096, base_frequency=8, octaves=12), 4096),
    "cfg3s": (dict(seed=1, method=pt.Method.opensimplex, resolution=4096, base_frequency=8, octaves=12), 4096),
    "cfg3g": (dict(seed=1, method=pt.Method.generic, resolution=4096, base_frequency=8, octaves=12), 4096),
    "cfg5": (dict(seed=1, smoothstep=5, resolution=32768, base_frequency=32, octaves=16), 4096),
}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--rotate", type=int, default=1, help="output buffers written in rotation (3: the bench's)")
a = ap.parse_args()
if a.config == "cfg4":
    cfg = pt.FbmConfig(seed=1, method=pt.Method.zg_separable, resolution=512, base_frequency=8, octaves=8)
    out = torch.empty((512, 512, 512), dtype=torch.float32, device="cuda")
    for _ in range(a.iters):
        pt.generate3d_device(cfg, (0, 0, 0), (512, 512, 512), out)
else:
    kw, ext = CONFIGS[a.config]
    cfg = pt.FbmConfig(**kw)
    outs = [torch.empty((ext, ext), dtype=torch.float32, device="cuda") for _ in range(a.rotate)]
    for i in range(a.iters):
        pt.generate_into_device(cfg, (0, 0), ext, outs[i % a.rotate])
    out = outs[0]
torch.cuda.synchronize()
print("ok", a.config, float(out.abs().max()))
