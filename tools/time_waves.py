"""Wave-quantisation probe: config-2 octaves over maps of growing height.
Prints us per launch and us per 64-row tile row; a step at a wave boundary
(444 resident CTAs = 13.9 tile rows of 32 CTAs) means a tail effect."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1610_03525_b200 as pt  # noqa: E402

cfg = pt.FbmConfig(seed=1, smoothstep=5, resolution=4096, base_frequency=8, octaves=12)
out = torch.empty((8192, 4096), dtype=torch.float32, device="cuda")
for rows in range(3072, 5376, 128):
    for _ in range(3):
        pt.generate_rect_device(cfg, (0, 0), 4096, rows, out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        pt.generate_rect_device(cfg, (0, 0), 4096, rows, out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    print(f"rows {rows:5d}  ctas {32 * rows // 64:5d}  waves {32 * rows / 64 / 444:5.2f}  {us:7.1f} us  "
          f"{us / (rows / 64):6.3f} us/tile-row", flush=True)
