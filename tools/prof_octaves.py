"""One generation launch of the config-2 grid with N octaves (ncu target).

    python tools/prof_octaves.py N [--iters 3]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1610_03525_b200 as pt  # noqa: E402

n = int(sys.argv[1])
iters = int(sys.argv[sys.argv.index("--iters") + 1]) if "--iters" in sys.argv else 3
cfg = pt.FbmConfig(seed=1, smoothstep=5, resolution=4096, base_frequency=8, octaves=n)
out = torch.empty((4096, 4096), dtype=torch.float32, device="cuda")
for _ in range(iters):
    pt.generate_into_device(cfg, (0, 0), 4096, out)
torch.cuda.synchronize()
print("ok", n)
