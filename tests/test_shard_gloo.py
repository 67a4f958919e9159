"""Multi-rank terrain sharding on CPU (gloo, world size 2): generation needs
no exchange; the analysis statistics (median sea level via histogram
all-reduce, box counts, land/coast counts, variogram) reduced across ranks
must equal the single-rank result exactly (counts) / to rounding (sums)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import make_cfg

W, H = 256, 256
SIZES = [2, 4, 8, 16, 32, 64]
LAGS = [1, 2, 4, 8, 16, 32, 64, 128]


def cfg():
    return make_cfg(method=0, smoothstep=5, seed=11, resolution=256, base_frequency=4, octaves=9)


def run(world, rank):
    from paper_1610_03525_b200.shard import Comm, plan_band, terrain_stats
    from shard_oracle import OracleBackend

    band = plan_band(W, H, world, rank, align=64, max_lag=max(LAGS))
    return terrain_stats(band, OracleBackend(cfg()), Comm(), SIZES, LAGS)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        st = run(world, rank)
        q.put((rank, st.sea_level, st.counts, st.coast_pixels, st.land_fraction, st.sum_sq, st.pairs))
    finally:
        dist.destroy_process_group()


def test_band_plan_covers_terrain_once():
    from paper_1610_03525_b200.shard import plan_band

    for world in (1, 2, 3, 8):
        rows = []
        for r in range(world):
            b = plan_band(4096, 32768, world, r, align=1024, max_lag=4096)
            assert b.y0 % 1024 == 0 and b.gen_y0 >= 0 and b.gen_y0 + b.gen_rows <= 32768
            rows.extend(range(b.y0, b.y0 + b.rows))
        assert rows == list(range(32768))


def test_single_rank_matches_reference_semantics(oracle):
    st = run(1, 0)
    m = oracle.sample(cfg(), *[a.ravel() for a in np.meshgrid(np.arange(W), np.arange(H))]).reshape(H, W)
    m = m.astype(np.float32).astype(np.float64)
    sea = oracle.upper_median(m)
    assert st.sea_level == sea
    s, mask, land = oracle.coastline_mask(m, sea)
    s, counts, d, k, r2 = oracle.box_count(mask, SIZES)
    assert st.counts == list(counts) and st.coast_pixels == int(mask.sum())
    ss, pr = oracle.variogram(m, LAGS)
    assert np.array_equal(st.pairs, pr) and np.allclose(st.sum_sq, ss, rtol=1e-12)


def test_two_ranks_gloo_equal_single_rank():
    single = run(1, 0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, sea, counts, coast, lf, ss, pr in res:
        assert sea == single.sea_level
        assert counts == single.counts and coast == single.coast_pixels and lf == single.land_fraction
        assert np.array_equal(pr, single.pairs)
        assert np.allclose(ss, single.sum_sq, rtol=1e-12, atol=0)
