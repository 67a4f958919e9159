"""Config 5: the 32768^2 terrain, 16 octaves, zg_paper S5, base cell 1024 px
(f0 = 32), as row bands (one per rank) followed by the fractal statistics of
the whole terrain (median sea level, coastline + box count eps 2..64,
variogram over lags 1..4096) through the C-ABI driver tg_terrain_stats_band,
reduced across ranks by the native NCCL communicator.

    python tools/terrain_run.py                      # 1 GPU
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/terrain_run.py

Prints one JSON line (rank 0): bench.cfg5_terrain's numbers plus a per-phase
breakdown of the analysis on rank 0 (the same C-ABI calls the driver makes,
timed one by one with syncs).
"""
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_1610_03525_b200 as pt  # noqa: E402
from paper_1610_03525_b200 import _abi  # noqa: E402
from paper_1610_03525_b200.shard import plan_band  # noqa: E402


def phases(lib, world, rank):
    """Rank 0's band: generation of band + halo + lookahead, the three median
    histogram passes, coastline + box count, variogram — each synchronised."""
    T = bench.T5
    cfg = pt.FbmConfig(seed=1, method=pt.Method.zg_paper, smoothstep=5, resolution=T, base_frequency=bench.F05,
                       octaves=bench.OCT5)
    c = cfg.to_c()
    band = plan_band(T, T, world, rank, align=1024, max_lag=4096)
    buf = torch.empty((band.gen_rows, T), dtype=torch.float32, device="cuda")
    own = buf.data_ptr() + 4 * band.halo_top * T
    out = {}

    def t(name, fn, reps=2):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        out[name] = round((time.perf_counter() - t0) / reps * 1e3, 3)

    t("regenerate_band_ms", lambda: lib.tg_fbm_generate_rect_f32(C.byref(c), 0, band.gen_y0, T, band.gen_rows,
                                                                 buf.data_ptr(), T, None))
    med = C.c_float()
    # the band's own upper median (the radix select with the sampled candidate window)
    t("median_ms", lambda: lib.tg_median_f32(own, T * band.rows, C.byref(med), None))
    sz = (C.c_int32 * 6)(2, 4, 8, 16, 32, 64)
    cnt = (C.c_int64 * 6)()
    a, b = C.c_int64(), C.c_int64()
    t("coastline_boxcount_ms", lambda: lib.tg_coastline_boxcount_band(own, T, band.rows, T, band.halo_top,
                                                                      0 if band.is_last else 1, 0.0, sz, 6, cnt,
                                                                      C.byref(a), C.byref(b), None))
    lg = (C.c_int32 * 13)(*[1 << i for i in range(13)])
    ss = (C.c_double * 26)()
    pr = (C.c_int64 * 26)()
    t("variogram_ms", lambda: lib.tg_variogram_band_f32(own, T, band.rows + band.below, T, band.rows, lg, 13, ss,
                                                        pr, None))
    return out


def main():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = _abi.load()
    res = bench.cfg5_terrain(lib, world, rank, steps=3, analysis=True)
    torch.cuda.empty_cache()
    ph = phases(lib, world, rank) if rank == 0 else None
    if rank == 0:
        res["analysis_phases_ms_rank0"] = ph
        print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
