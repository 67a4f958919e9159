"""Config 5: a 32768^2 terrain, 16 octaves, zg_paper S5, base cell 1024 px
(f0 = 32), generated as row bands (one per rank) followed by the fractal
analysis (median sea level, coastline + box count eps 2..64, variogram over
lags 1..4096), statistics all-reduced across ranks.

    python tools/terrain_run.py                      # 1 GPU
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/terrain_run.py

Prints one JSON line (rank 0): generation time (max over ranks), sample-
octaves/s, analysis time, box-count and variogram dimensions.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1610_03525_b200 as pt  # noqa: E402
from paper_1610_03525_b200.shard import Comm, DeviceBackend, plan_band, terrain_stats  # noqa: E402

T = int(os.environ.get("TG_T", "32768"))
OCT = 16


def main():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = pt.FbmConfig(seed=1, method=pt.Method.zg_paper, smoothstep=5, resolution=T, base_frequency=T // 1024,
                       octaves=OCT)
    sizes = [2, 4, 8, 16, 32, 64]
    lags = [1 << i for i in range(13)]
    band = plan_band(T, T, world, rank, align=1024, max_lag=max(lags))
    be = DeviceBackend(cfg)
    comm = Comm(device=torch.device("cuda", local))
    # warm-up generation of the band (allocations, LUTs)
    be.generate(band)
    torch.cuda.synchronize()
    # timed generation of the owned rows only (the throughput number)
    out = torch.empty((band.rows, T), dtype=torch.float32, device="cuda")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    pt.generate_rect_device(cfg, (0, band.y0), T, band.rows, out)
    e1.record()
    torch.cuda.synchronize()
    gen_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(gen_ms, op=dist.ReduceOp.MAX)
    del out
    # analysis: regenerates the band + halo/lookahead rows, all-reduces
    # statistics; one untimed warm-up pass (module loading, pool growth)
    terrain_stats(band, be, comm, sizes, lags)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    phases = {}

    def timed(name, fn):
        def w(*a, **k):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = fn(*a, **k)
            torch.cuda.synchronize()
            phases[name] = phases.get(name, 0.0) + (time.perf_counter() - t) * 1e3
            return r
        return w

    be.generate = timed("regenerate_band_ms", be.generate)
    be.histogram = timed("median_histograms_ms", be.histogram)
    be.boxcount = timed("coastline_boxcount_ms", be.boxcount)
    be.variogram = timed("variogram_ms", be.variogram)
    t0 = time.perf_counter()
    st = terrain_stats(band, be, comm, sizes, lags)
    torch.cuda.synchronize()
    an_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(an_s, op=dist.ReduceOp.MAX)
    if rank == 0:
        so = T * T * OCT
        print(json.dumps({
            "workload": f"config 5: {T}^2 zg_paper S5, {OCT} octaves, base cell 1024 px, {world} row bands",
            "n_gpus": world, "gen_ms": float(gen_ms.item()), "sample_octaves_per_s": so / (gen_ms.item() * 1e-3),
            "analysis_s": float(an_s.item()), "analysis_phases_ms_rank0": {k: round(v, 3) for k, v in phases.items()},
            "sea_level": st.sea_level, "land_fraction": st.land_fraction,
            "box_counts": st.counts, "d_box": st.d_box, "r2_box": st.r2_box,
            "variogram_gamma": [float(g) for g in st.gamma], "hurst": st.hurst, "d_variogram": st.d_variogram,
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
