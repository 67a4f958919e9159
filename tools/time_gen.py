"""Quick device timing of generation launches (CUDA events, rotating outputs).

    python tools/time_gen.py [--configs cfg1,cfg2,cfg3p,cfg5] [--iters 50]
Prints one line per config: mean us per launch and G sample-octaves/s.
Set TG_LIB_PATH to time a library variant.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1610_03525_b200 as pt  # noqa: E402

CONFIGS = {
    "cfg1": (dict(seed=1, resolution=1024, base_frequency=8, octaves=8), 1024, 1024),
    "cfg2": (dict(seed=1, smoothstep=5, resolution=4096, base_frequency=8, octaves=12), 4096, 4096),
    "cfg2sep": (dict(seed=1, method=pt.Method.zg_separable, smoothstep=5, resolution=4096, base_frequency=8,
                     octaves=12), 4096, 4096),
    "cfg3p": (dict(seed=1, method=pt.Method.perlin3, resolution=4096, base_frequency=8, octaves=12), 4096, 4096),
    "cfg3p5": (dict(seed=1, method=pt.Method.perlin5, resolution=4096, base_frequency=8, octaves=12), 4096, 4096),
    "cfg3g": (dict(seed=1, method=pt.Method.generic, resolution=4096, base_frequency=8, octaves=12), 4096, 4096),
    "cfg3s": (dict(seed=1, method=pt.Method.opensimplex, resolution=4096, base_frequency=8, octaves=12), 4096,
              4096),
    "cfg3pp": (dict(seed=1, method=pt.Method.perlin_perm, resolution=4096, base_frequency=8, octaves=12), 4096,
               4096),
    "cfg5": (dict(seed=1, smoothstep=5, resolution=32768, base_frequency=32, octaves=16), 4096, 4096),
}

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="cfg1,cfg2,cfg3p,cfg5")
ap.add_argument("--iters", type=int, default=50)
a = ap.parse_args()
for name in a.configs.split(","):
    kw, w, h = CONFIGS[name]
    cfg = pt.FbmConfig(**kw)
    bufs = [torch.empty((h, w), dtype=torch.float32, device="cuda") for _ in range(3)]
    for i in range(5):
        pt.generate_rect_device(cfg, (0, 0), w, h, bufs[i % 3])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.iters):
        pt.generate_rect_device(cfg, (0, 0), w, h, bufs[i % 3])
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.iters
    so = w * h * cfg.octaves
    print(f"{name:8s} {us:9.1f} us  {so / us / 1e3:8.1f} G sample-oct/s  ({w}x{h}x{cfg.octaves})", flush=True)


def time_batch(n_maps=64, iters=20):
    cfg = pt.FbmConfig(seed=1, resolution=1024, base_frequency=8, octaves=8)
    out = torch.empty((n_maps, 1024, 1024), dtype=torch.float32, device="cuda")
    seeds = list(range(1, n_maps + 1))
    for _ in range(3):
        pt.generate_batch_device(cfg, seeds, (0, 0), 1024, 1024, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        pt.generate_batch_device(cfg, seeds, (0, 0), 1024, 1024, out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    so = n_maps * 1024 * 1024 * 8
    print(f"cfg1x{n_maps} {us:9.1f} us  {so / us / 1e3:8.1f} G sample-oct/s  (batch of {n_maps} 1024^2x8 maps)")


def time_3d(iters=5):
    cfg = pt.FbmConfig(seed=1, method=pt.Method.zg_separable, resolution=512, base_frequency=8, octaves=8)
    out = torch.empty((512, 512, 512), dtype=torch.float32, device="cuda")
    for _ in range(2):
        pt.generate3d_device(cfg, (0, 0, 0), (512, 512, 512), out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        pt.generate3d_device(cfg, (0, 0, 0), (512, 512, 512), out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    so = 512 ** 3 * 8
    print(f"cfg4     {us:9.1f} us  {so / us / 1e3:8.1f} G sample-oct/s  (512^3x8 volume)")


if "--batch" in sys.argv[0:0] or os.environ.get("TG_TIME_EXTRA"):
    time_batch()
    time_3d()
