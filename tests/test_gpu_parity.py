"""GPU parity: the sm_100a path through the C-ABI against the oracle.

Bars (BASELINE.json north_star): lattice hashes bit-exact (u64), fp32 corner
heights equal float(reference double) exactly, heights within
max|dh| <= 1e-5 * A (A = max |h_ref| over the window, helpers.height_tolerance),
region/tiling/batch/shard invariance bit-exact, integer analysis results exact.
"""
import ctypes as C

import numpy as np
import pytest

from helpers import amplitude_sum, cfg_from_dict, height_tolerance, keys_from_golden, make_cfg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1610_03525_b200 as pt  # noqa: E402
from paper_1610_03525_b200 import _abi  # noqa: E402

LANES = {"height": 0, "angle": 0xA0761D6478BD642F, "magnitude": 0xE7037ED1A0B428DB}


def gen(c, ox, oy, w, h=None):
    h = w if h is None else h
    out = torch.empty((h, w), dtype=torch.float32, device="cuda")
    st = _abi.load().tg_fbm_generate_rect_f32(C.byref(c), ox, oy, w, h, out.data_ptr(), w,
                                              torch.cuda.current_stream().cuda_stream)
    assert st == 0, _abi.last_error()
    return out


def check_close(got, ref, c, what=""):
    tol = height_tolerance(ref, c)
    err = float(np.max(np.abs(got.astype(np.float64) - ref)))
    assert err <= tol, f"{what}: max|dh|={err:.3e} > tol={tol:.3e}"
    return err


# ---- lattice --------------------------------------------------------------------

def _dev_keys(lat):
    k = keys_from_golden(lat)
    return torch.from_numpy(k.view(np.uint8).copy()).cuda(), len(k)


def test_lattice_hash_bit_exact(golden):
    lat = golden["lattice"]
    dk, n = _dev_keys(lat)
    for name, lane in LANES.items():
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        assert _abi.load().tg_lattice_hash(dk.data_ptr(), n, lane, out.data_ptr(), None) == 0
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, lat[f"hash_{name}"]), name


def test_lattice_height_is_rounded_reference(golden):
    lat = golden["lattice"]
    dk, n = _dev_keys(lat)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    assert _abi.load().tg_lattice_height_f32(dk.data_ptr(), n, out.data_ptr(), None) == 0
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), lat["height"].astype(np.float32))


def test_lattice_unit_gradient_within_tolerance(golden):
    lat = golden["lattice"]
    dk, n = _dev_keys(lat)
    out = torch.empty(2 * n, dtype=torch.float32, device="cuda")
    assert _abi.load().tg_lattice_unit_gradient_f32(dk.data_ptr(), n, out.data_ptr(), None) == 0
    torch.cuda.synchronize()
    g = out.cpu().numpy().reshape(-1, 2).astype(np.float64)
    assert np.max(np.abs(g - lat["unit_gradient"])) < 1e-6


# ---- maps against the reference's golden outputs --------------------------------

def test_golden_maps(golden):
    worst = {}
    for name, meta in golden["maps_meta"].items():
        ref = golden["maps"][name]
        c = cfg_from_dict(meta["cfg"])
        ox, oy = meta["origin"]
        ext = meta["extent"]
        if meta["cfg"]["normalize"]:
            hm = pt.generate_region(pt.FbmConfig(seed=c.seed, octaves=c.octaves, resolution=c.resolution,
                                                 base_frequency=c.base_frequency, normalize=True),
                                    (ox, oy), ext)
            assert hm.normalized and hm.data.min() == -1.0 and hm.data.max() == 1.0
            got = hm.data
        else:
            got = gen(c, ox, oy, ext).cpu().numpy()
        if meta["cfg"]["zero_lattice"]:
            assert np.all(got == 0.0)
            continue
        worst[name] = check_close(got, ref, c, name)


# ---- full-size BASELINE configs against the restated oracle ----------------------

def _sample_check(oracle, c, dev_map, ox, oy, n=4096, seed=0):
    h, w = dev_map.shape
    rng = np.random.default_rng(seed)
    ys = rng.integers(0, h, n)
    xs = rng.integers(0, w, n)
    ref = oracle.sample(c, xs + ox, ys + oy)
    got = dev_map.cpu().numpy()[ys, xs].astype(np.float64)
    tol = 1e-5 * max(float(np.max(np.abs(ref))), 1e-12)
    err = float(np.max(np.abs(got - ref)))
    assert err <= tol, f"sampled max|dh|={err:.3e} > {tol:.3e}"


def test_config1_full_map(oracle):
    c = make_cfg(method=0, seed=1, resolution=1024, base_frequency=8, octaves=8)
    m = gen(c, 0, 0, 1024).cpu().numpy()
    check_close(m, oracle.generate(c, 0, 0, 1024), c, "cfg1")


# config 2, 3 and 5 at their full shapes: tests/test_gpu_fullshape.py


def test_config5_proxy_equals_golden(golden):
    # (R=1024, f0=1) is the top-left chunk of (32768, f0=32).
    ref = golden["maps"]["cfg5_proxy_S5"]
    c = make_cfg(method=0, smoothstep=5, seed=1, resolution=32768, base_frequency=32, octaves=16)
    got = gen(c, 0, 0, 64).cpu().numpy()
    check_close(got, ref, c, "cfg5 proxy")


# ---- bit-exact invariants (test_fbm.cpp:256-300, acceptance C6) ------------------

@pytest.mark.parametrize("method", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("ratio", [2.0, 1.7])
def test_region_equals_submap(method, ratio):
    c = make_cfg(method=method, seed=909, resolution=64, octaves=3, frequency_ratio=ratio)
    full = gen(c, 0, 0, 64)
    region = gen(c, 32, 32, 32)
    assert torch.equal(region, full[32:, 32:])


@pytest.mark.parametrize("method", [0, 1, 2, 3, 4])
def test_four_way_tiling_bit_exact(method):
    c = make_cfg(method=method, seed=2024, resolution=512, octaves=4)
    full = gen(c, 0, 0, 512)
    for oy in (0, 256):
        for ox in (0, 256):
            assert torch.equal(gen(c, ox, oy, 256), full[oy:oy + 256, ox:ox + 256])


def test_unaligned_windows_and_shards_bit_exact():
    # cfg2-like map cut at odd (but octave-0 aligned) origins and shapes.
    c = make_cfg(method=0, smoothstep=5, seed=7, resolution=2048, base_frequency=64, octaves=13)
    full = gen(c, 0, 0, 2048)
    for ox, oy, w, h in [(32, 96, 96, 160), (1024, 0, 1024, 37), (1984, 2016, 64, 32)]:
        assert torch.equal(gen(c, ox, oy, w, h), full[oy:oy + h, ox:ox + w])
    # row-band shards of any count reassemble the map (multi-GPU sharding unit)
    for n in (2, 3, 8):
        bands = []
        rows = [2048 * i // n // 32 * 32 for i in range(n)] + [2048]
        for a, b in zip(rows[:-1], rows[1:]):
            bands.append(gen(c, 0, a, 2048, b - a))
        assert torch.equal(torch.cat(bands, 0), full)


def test_negative_origin_region():
    c = make_cfg(seed=3, resolution=64, octaves=4)
    a = gen(c, 32, -32, 16)
    b = gen(c, 0, -64, 64)
    assert torch.equal(a, b[32:48, 32:48])


def test_zero_source_gives_zero_map():
    for m in (0, 2, 3):
        c = make_cfg(method=m, resolution=16, octaves=4, zero_lattice=1)
        assert torch.count_nonzero(gen(c, 0, 0, 16)).item() == 0


def test_deterministic():
    c = make_cfg(method=2, seed=777, resolution=64, octaves=4)
    assert torch.equal(gen(c, 0, 0, 64), gen(c, 0, 0, 64))


def test_batch_equals_single_maps():
    c = make_cfg(method=0, smoothstep=5, seed=0, resolution=1024, base_frequency=8, octaves=8)
    seeds = [1, 2, 99, 2**63 + 5]
    out = torch.empty((len(seeds), 256, 256), dtype=torch.float32, device="cuda")
    pt.generate_batch_device(pt.FbmConfig(method=0, smoothstep=5, resolution=1024, base_frequency=8, octaves=8),
                             seeds, (256, 512), 256, 256, out)
    for i, s in enumerate(seeds):
        c.seed = s
        assert torch.equal(out[i], gen(c, 256, 512, 256))


def test_host_drop_in_matches_device():
    cfg = pt.FbmConfig(seed=17, resolution=512, octaves=6)
    dev = gen(cfg.to_c(), 0, 0, 512).cpu().numpy().astype(np.float64)
    buf = np.full((512, 512), 123.0)  # stale content must be overwritten (test_fbm.cpp:375-387)
    pt.generate_into(cfg, (0, 0), 512, buf)
    assert np.array_equal(buf, dev)
    hm = pt.generate_heightmap(cfg)
    assert np.array_equal(hm.data, dev) and len(hm.octave_seconds) == 6
    with pytest.raises(pt.ValidationError):
        pt.generate_into(cfg, (0, 0), 512, np.zeros((511, 511)))
    f32 = np.zeros((512, 512), np.float32)
    pt.generate_into(cfg, (0, 0), 512, f32)
    assert np.array_equal(f32.astype(np.float64), dev)


@pytest.mark.parametrize("frac", ["0", "0.5", "1"])
def test_host_pipeline_bands_pinned_pageable(frac, monkeypatch):
    """Banded host path: ragged bands through the staging ring, f64
    (device- and host-widened mixes) and f32 destinations, pinned, pageable
    and misaligned (streaming-store head) buffers."""
    monkeypatch.setenv("TG_HOST_WIDEN_FRAC", frac)
    cfg = pt.FbmConfig(seed=5, resolution=4096, base_frequency=8, octaves=12, smoothstep=5)
    E = 3000
    dev = gen(cfg.to_c(), 0, 0, E).cpu()
    for dt in (torch.float64, torch.float32):
        want = dev.to(dt)
        for pinned in (True, False):
            t = torch.full((E * E + 1,), 7.0, dtype=dt, pin_memory=pinned)
            for off in (0, 1):
                view = t[off:off + E * E]
                pt.generate_into(cfg, (0, 0), E, view.numpy())
                assert torch.equal(view.view(E, E), want), (dt, pinned, off)


def test_host_pipeline_concurrent_callers_and_schedules(monkeypatch):
    """The asynchronous pool join under contention: four host threads call the
    drop-in at once (ctypes drops the GIL) with different seeds and extents;
    every result equals the device map.  Then the band schedule knobs
    (small / large bands, shallow / deep rings) give the same bytes."""
    import threading

    cases = [(seed, E) for seed, E in ((3, 1024), (4, 1500), (5, 2048), (6, 777))]
    cfgs = {seed: pt.FbmConfig(seed=seed, resolution=4096, base_frequency=8, octaves=12, smoothstep=5)
            for seed, _ in cases}
    want = {seed: gen(cfgs[seed].to_c(), 0, 0, E).cpu().to(torch.float64) for seed, E in cases}
    outs = {seed: torch.full((E, E), -3.0, dtype=torch.float64, pin_memory=(seed % 2 == 0)) for seed, E in cases}
    errs = []

    def work(seed, E):
        try:
            for _ in range(6):
                outs[seed].fill_(-3.0)
                pt.generate_into(cfgs[seed], (0, 0), E, outs[seed].numpy())
                if not torch.equal(outs[seed], want[seed]):
                    errs.append((seed, "mismatch"))
        except Exception as e:  # pragma: no cover
            errs.append((seed, repr(e)))

    th = [threading.Thread(target=work, args=c) for c in cases]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    seed, E = 5, 2048
    for env in ({"TG_HOST_BAND_LOG2": "17"}, {"TG_HOST_BAND_LOG2": "23"}, {"TG_HOST_SLOTS": "3"},
                {"TG_HOST_SLOTS": "16", "TG_HOST_LOOK": "2"}, {"TG_HOST_SPIN": "0"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        outs[seed].fill_(-3.0)
        pt.generate_into(cfgs[seed], (0, 0), E, outs[seed].numpy())
        assert torch.equal(outs[seed], want[seed]), env
        for k in env:
            monkeypatch.delenv(k)


def test_validation_errors_on_device_path():
    cfg = pt.FbmConfig(resolution=64)
    with pytest.raises(pt.ValidationError):
        pt.generate_region(cfg, (5, 0), 16)
    with pytest.raises(pt.ValidationError):
        pt.generate_region(cfg, (0, 33), 16)
    pt.generate_region(cfg, (32, -32), 16)


def test_warnings_and_normalize():
    hm = pt.generate_heightmap(pt.FbmConfig(resolution=8, octaves=4))
    assert len(hm.warnings) == 1 and "octave 3" in hm.warnings[0]
    assert pt.generate_heightmap(pt.FbmConfig(resolution=8, octaves=3)).warnings == []
    n = pt.generate_heightmap(pt.FbmConfig(seed=21, resolution=32, octaves=3, normalize=True))
    assert n.data.min() == -1.0 and n.data.max() == 1.0 and n.normalized


def test_octave_sweep_amplitude_bound():
    # |h| <= sum of per-octave kernel bounds (test_fbm.cpp:83-110, 223-237)
    for m, per in ((0, 9.0), (3, 2.0)):
        c = make_cfg(method=m, seed=31337, resolution=64, octaves=6)
        v = gen(c, 0, 0, 64)
        assert float(v.abs().max()) <= per * amplitude_sum(c)


# ---- device normalization (fbm.hpp:638-656) ---------------------------------------

def test_device_minmax_rescale(oracle):
    c = make_cfg(seed=21, resolution=256, octaves=5)
    m = gen(c, 0, 0, 256)
    lo, hi = C.c_double(), C.c_double()
    assert _abi.load().tg_minmax_f32(m.data_ptr(), m.numel(), C.byref(lo), C.byref(hi), None) == 0
    host = m.cpu().numpy().astype(np.float64)
    assert lo.value == host.min() and hi.value == host.max()
    assert _abi.load().tg_rescale_f32(m.data_ptr(), m.numel(), lo.value, hi.value, None) == 0
    torch.cuda.synchronize()
    ref, *_ = oracle.normalize(host)
    got = m.cpu().numpy()
    assert got.min() == -1.0 and got.max() == 1.0
    assert np.array_equal(got, ref.astype(np.float32))


# ---- analysis pass --------------------------------------------------------------

def test_median_exact():
    for seed, R in ((42, 128), (5, 1000), (1, 4096)):
        c = make_cfg(seed=seed, resolution=R, octaves=6)
        m = gen(c, 0, 0, R)
        med = pt.upper_median_device(m)
        host = np.sort(m.cpu().numpy().ravel())
        assert med == host[host.size // 2]


def test_coastline_mask_matches_oracle(oracle):
    c = make_cfg(seed=42, resolution=300, octaves=6)
    m = gen(c, 0, 0, 300)
    mask, sea, lf = pt.coastline_mask_device(m, 300)
    host = m.cpu().numpy().astype(np.float64)
    st, ref_mask, land = oracle.coastline_mask(host, sea)
    assert st == 0 and np.array_equal(mask.cpu().numpy(), ref_mask)
    assert lf == land / host.size


def test_halfplane_and_all_land():
    half = torch.tensor(np.where(np.arange(8)[None, :] < 4, 1.0, -1.0) * np.ones((8, 1)),
                        dtype=torch.float32, device="cuda")
    mask, _, lf = pt.coastline_mask_device(half.contiguous(), 8, 0.0)
    expect = np.zeros((8, 8), np.uint8)
    expect[:, 3] = 1
    assert np.array_equal(mask.cpu().numpy(), expect) and lf == 0.5
    with pytest.raises(pt.ValidationError):
        pt.coastline_mask_device(torch.full((4, 4), 2.0, device="cuda"), 4, 0.0)


def test_box_count_known_answers():
    col = torch.zeros((64, 64), dtype=torch.uint8, device="cuda")
    col[:, 31] = 1
    r = pt.box_count_mask_device(col, 64, [2, 4, 8, 16])
    assert r.counts == [32, 16, 8, 4] and abs(r.d - 1.0) < 1e-12 and abs(r.k - 64.0) < 1e-9
    r = pt.box_count_mask_device(torch.ones((64, 64), dtype=torch.uint8, device="cuda"), 64, [2, 4, 8, 16])
    assert r.counts == [1024, 256, 64, 16] and abs(r.d - 2.0) < 1e-12
    with pytest.raises(pt.ValidationError):
        pt.box_count_mask_device(col, 64, [2, 4])
    with pytest.raises(pt.ValidationError):
        pt.box_count_mask_device(col, 64, [4, 2, 8])
    with pytest.raises(pt.ValidationError):
        pt.box_count_mask_device(torch.zeros((8, 8), dtype=torch.uint8, device="cuda"), 8, [2, 4, 8])


@pytest.mark.parametrize("R,sizes", [(512, [2, 4, 8, 16, 32, 64]), (1000, [3, 5, 7, 33, 100]),
                                     (4096, [2, 4, 8, 16, 32, 64]),
                                     (1000, [1, 2, 3, 4, 8, 16, 32, 64, 128, 256, 500]),
                                     (777, [2, 4, 8, 16, 32, 64, 128])])
def test_fused_boxcount_matches_oracle(oracle, R, sizes):
    c = make_cfg(method=0, smoothstep=5, seed=42, resolution=R, base_frequency=8, octaves=8)
    m = gen(c, 0, 0, R)
    rep = pt.box_count_device(m, R, sizes)
    host = m.cpu().numpy().astype(np.float64)
    assert rep.sea_level == oracle.upper_median(host)
    st, mask, land = oracle.coastline_mask(host, rep.sea_level)
    st, counts, d, k, r2 = oracle.box_count(mask, sizes)
    assert list(counts) == rep.counts
    assert rep.coast_pixels == int(mask.sum()) and rep.land_fraction == land / host.size
    assert abs(rep.d - d) < 1e-12 and abs(rep.r2 - r2) < 1e-12


def test_variogram_matches_oracle(oracle):
    c = make_cfg(method=0, smoothstep=5, seed=3, resolution=512, base_frequency=8, octaves=10)
    m = gen(c, 0, 0, 512)
    lags = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512]
    ss, pr = pt.variogram_device(m, 512, 512, lags)
    rss, rpr = oracle.variogram(m.cpu().numpy().astype(np.float64), lags)
    assert np.array_equal(pr, rpr)
    assert np.allclose(ss, rss, rtol=1e-10, atol=0)


def test_variogram_special_values(oracle):
    """Zeros, signed zeros and subnormals take the hardware fp32->fp64 path."""
    g = torch.Generator().manual_seed(4)
    m = torch.randn((64, 300), generator=g)
    m[::3, ::5] = 0.0
    m[1::7, ::3] = -0.0
    m[2::5, 1::4] = 1e-40
    m[3::9, 2::6] = -3e-42
    m[5, :] = 3.0e38
    dev = m.cuda()
    lags = [1, 2, 3, 5, 8, 13, 21, 34, 55]
    ss, pr = pt.variogram_device(dev, 300, 64, lags)
    rss, rpr = oracle.variogram(m.numpy().astype(np.float64), lags)
    assert np.array_equal(pr, rpr)
    assert np.allclose(ss, rss, rtol=1e-10, atol=0)


def test_variogram_row_offsets_beyond_32_bits(oracle):
    """h * ld >= 2^31: the y-axis of that lag is summed by the wide-offset kernel."""
    H, W, ld = 1100, 64, 1 << 21
    big = torch.empty((H, ld), dtype=torch.float32, device="cuda")  # 9.2 GB, only W columns touched
    g = torch.Generator().manual_seed(8)
    m = torch.randn((H, W), generator=g)
    big[:, :W] = m.cuda()
    lags = [1, 3, 1023, 1024, 1099, 1100]
    arr = (C.c_int32 * len(lags))(*lags)
    ss = (C.c_double * (2 * len(lags)))()
    pr = (C.c_int64 * (2 * len(lags)))()
    assert _abi.load().tg_variogram_f32(big.data_ptr(), W, H, ld, arr, len(lags), ss, pr, None) == 0
    rss, rpr = oracle.variogram(m.numpy().astype(np.float64), lags)
    assert np.array_equal(np.array(pr[:]).reshape(-1, 2), rpr)
    assert np.allclose(np.array(ss[:]).reshape(-1, 2), rss, rtol=1e-10, atol=0)
    del big


@pytest.mark.parametrize("W,H,lags", [
    (700, 300, [1, 3, 7, 100, 299, 300, 650]),                   # ragged, lags >= H, 7 -> padded to 8
    (9000, 40, [1, 2, 4096, 4097, 5000, 8999, 9000]),            # segments + apron, x-lags beyond the apron
    (257, 129, list(range(1, 21))),                              # 20 lags: two passes (16 + 4)
])
def test_variogram_segments_and_lag_sets(oracle, W, H, lags):
    c = make_cfg(method=0, smoothstep=5, seed=9, resolution=16384, base_frequency=32, octaves=12)
    m = gen(c, 0, 0, W, H)
    ss, pr = pt.variogram_device(m, W, H, lags)
    rss, rpr = oracle.variogram(m.cpu().numpy().astype(np.float64), lags)
    assert np.array_equal(pr, rpr)
    assert np.allclose(ss, rss, rtol=1e-10, atol=0)


# ---- 3D (new; property-pinned + restated oracle) ------------------------------------

def test_fbm3d_matches_restated_oracle(oracle):
    c = make_cfg(method=1, seed=5, resolution=64, base_frequency=8, octaves=5)
    out = torch.empty((64, 64, 64), dtype=torch.float32, device="cuda")
    pt.generate3d_device(pt.FbmConfig(method=1, seed=5, resolution=64, base_frequency=8, octaves=5),
                         (0, 0, 0), (64, 64, 64), out)
    ref = oracle.generate3d(c, 0, 0, 0, 64, 64, 64)
    check_close(out.cpu().numpy(), ref, c, "3d")


def test_fbm3d_subvolume_bit_exact():
    cfg = pt.FbmConfig(method=1, seed=9, resolution=128, base_frequency=4, octaves=7, smoothstep=5)
    full = torch.empty((128, 128, 128), dtype=torch.float32, device="cuda")
    pt.generate3d_device(cfg, (0, 0, 0), (128, 128, 128), full)
    sub = torch.empty((32, 64, 96), dtype=torch.float32, device="cuda")
    pt.generate3d_device(cfg, (32, 64, 96), (32, 64, 96), sub)
    assert torch.equal(sub, full[96:128, 64:128, 32:128])


# ---- row-band shards (multi-GPU unit) -----------------------------------

def test_device_band_stats_sum_to_whole_map(oracle):
    from paper_1610_03525_b200.shard import Comm, DeviceBackend, plan_band, terrain_stats

    cfgp = pt.FbmConfig(method=0, smoothstep=5, seed=3, resolution=1024, base_frequency=4, octaves=12)
    sizes, lags = [2, 4, 8, 16, 32, 64], [1, 2, 4, 8, 16, 32, 64, 128, 256, 512]
    whole = terrain_stats(plan_band(1024, 1024, 1, 0, align=256, max_lag=512), DeviceBackend(cfgp), Comm(),
                          sizes, lags)
    # the whole-map numbers against the oracle on the GPU's own map
    m = gen(cfgp.to_c(), 0, 0, 1024).cpu().numpy().astype(np.float64)
    sea = oracle.upper_median(m)
    assert whole.sea_level == sea
    st, mask, land = oracle.coastline_mask(m, sea)
    st, counts, d, k, r2 = oracle.box_count(mask, sizes)
    assert whole.counts == list(counts) and whole.coast_pixels == int(mask.sum())
    ss, pr = oracle.variogram(m, lags)
    assert np.array_equal(whole.pairs, pr) and np.allclose(whole.sum_sq, ss, rtol=1e-10)
    # 4 bands evaluated one after another on this GPU, summed on the host
    tot_c, tot_ss, tot_pr, tot_coast = np.zeros(len(sizes), np.int64), 0.0, 0, 0
    for r in range(4):
        b = plan_band(1024, 1024, 4, r, align=256, max_lag=512)
        s = terrain_stats(b, DeviceBackend(cfgp), Comm(), sizes, lags, sea_level=sea)
        tot_c += np.array(s.counts)
        tot_ss = tot_ss + s.sum_sq
        tot_pr = tot_pr + s.pairs
        tot_coast += s.coast_pixels
    assert list(tot_c) == whole.counts and tot_coast == whole.coast_pixels
    assert np.array_equal(tot_pr, whole.pairs) and np.allclose(tot_ss, whole.sum_sq, rtol=1e-10)


@pytest.mark.parametrize("R,f0,ratio,octs", [(60, 3, 2.0, 5), (48, 2, 1.7, 5), (64, 2, 2.0, 7)])
def test_fbm3d_general_paths_match_oracle(oracle, R, f0, ratio, octs):
    c = make_cfg(method=1, seed=2, resolution=R, base_frequency=f0, octaves=octs, frequency_ratio=ratio,
                 smoothstep=5)
    cfgp = pt.FbmConfig(method=1, seed=2, resolution=R, base_frequency=f0, octaves=octs, frequency_ratio=ratio,
                        smoothstep=5)
    n = min(R, 40)
    out = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
    pt.generate3d_device(cfgp, (0, 0, 0), (n, n, n), out)
    check_close(out.cpu().numpy(), oracle.generate3d(c, 0, 0, 0, n, n, n), c, f"3d R{R} f0{f0} r{ratio}")


# ---- edge cases: extreme origins / octave counts / odd resolutions -------------------

@pytest.mark.parametrize("method", [0, 2, 3])
def test_far_origin_near_limit(oracle, method):
    # |origin| up to 2^40 (fbm.hpp:552); lattice indices then need full int64 keys
    R = 1024
    for ox, oy in [((1 << 40) - 1024, -(1 << 40)), (-(1 << 39), (1 << 39) + 512)]:
        c = make_cfg(method=method, seed=2**64 - 7, resolution=R, base_frequency=2, octaves=10)
        m = gen(c, ox, oy, 96, 64)
        ys, xs = np.meshgrid(np.arange(oy, oy + 64), np.arange(ox, ox + 96), indexing="ij")
        ref = oracle.sample(c, xs.ravel(), ys.ravel()).reshape(64, 96)
        check_close(m.cpu().numpy(), ref, c, f"far origin m{method}")


def test_thirty_two_octaves(oracle):
    c = make_cfg(method=0, smoothstep=5, seed=9, resolution=1024, base_frequency=1, octaves=32, persistence=0.9)
    m = gen(c, 0, 0, 128)
    check_close(m.cpu().numpy(), oracle.generate(c, 0, 0, 128), c, "32 octaves")


@pytest.mark.parametrize("R,f0", [(1000, 8), (768, 3), (4097, 1)])
def test_odd_resolutions(oracle, R, f0):
    for method in (0, 3):
        c = make_cfg(method=method, seed=4, resolution=R, base_frequency=f0, octaves=9)
        m = gen(c, 0, 0, 256)
        check_close(m.cpu().numpy(), oracle.generate(c, 0, 0, 256), c, f"R{R} f0{f0} m{method}")


@pytest.mark.parametrize("method", [1, 2, 4])
def test_s5_other_methods(oracle, method):
    c = make_cfg(method=method, smoothstep=5, seed=12, resolution=2048, base_frequency=4, octaves=11)
    m = gen(c, 0, 0, 2048)
    check_close(m[:128, :128].cpu().numpy(), oracle.generate(c, 0, 0, 128), c, f"S5 m{method}")
    _sample_check(oracle, c, m, 0, 0, n=2048)


# ---- OpenSimplex (new baseline; parity vs the restated oracle, unpinned) ------------

@pytest.mark.parametrize("R,f0,octs,ratio", [(256, 2, 6, 2.0), (4096, 8, 12, 2.0), (100, 3, 5, 1.7)])
def test_opensimplex_matches_restated_oracle(oracle, R, f0, octs, ratio):
    c = make_cfg(method=5, seed=77, resolution=R, base_frequency=f0, octaves=octs, frequency_ratio=ratio)
    n = min(R, 256)
    m = gen(c, 0, 0, n)
    check_close(m.cpu().numpy(), oracle.generate(c, 0, 0, n), c, f"opensimplex R{R}")


@pytest.mark.parametrize("R,f0,octs,pers,ox,oy,n", [
    (512, 64, 5, 1.0, 0, 0, 256),          # persistence 1: fine octaves located per pixel (no stepping)
    (256, 8, 8, 0.5, 0, 0, 256),           # fr up to 4: hashed octaves, stepped groups
    (32768, 32, 16, 0.5, 31 * 1024, 30 * 1024, 200),  # far window (cell-aligned origin, the oracle's contract)
    (4096, 8, 12, 0.5, 3584, 3584, 500),              # config 3's last tiles, partial pixel groups
])
def test_opensimplex_modes_and_far_windows(oracle, R, f0, octs, pers, ox, oy, n):
    # fp32 lattice selection (region_case): near a region boundary the vertex that
    # changes carries attn ~ 0, so the sum matches the fp64 oracle within tolerance
    c = make_cfg(method=5, seed=31, resolution=R, base_frequency=f0, octaves=octs, persistence=pers)
    m = gen(c, ox, oy, n)
    check_close(m.cpu().numpy(), oracle.generate(c, ox, oy, n), c, f"opensimplex R{R} p{pers} @({ox},{oy})")


def test_opensimplex_region_and_zero():
    c = make_cfg(method=5, seed=909, resolution=64, octaves=3)
    assert torch.equal(gen(c, 32, 32, 32), gen(c, 0, 0, 64)[32:, 32:])
    c.zero_lattice = 1
    assert torch.count_nonzero(gen(c, 0, 0, 64)).item() == 0


# ---- PGM16 / PNG16 export of device maps --------------------------

@pytest.mark.skipif(not __import__("os").path.exists(__import__("os").path.join(
    __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))),
    "oracle", "_ref", "libtgref.so")), reason="reference build absent")
@pytest.mark.parametrize("W,H", [(257, 257), (512, 512), (1024, 96)])
def test_pgm_png_bytes_equal_reference_writers(W, H):
    from oracle.pyoracle import Reference

    ref = Reference()
    c = make_cfg(method=0, smoothstep=5, seed=5, resolution=1024, base_frequency=4, octaves=10)
    m = gen(c, 0, 0, W, H)
    host = m.cpu().numpy().astype(np.float64)
    assert pt.encode_pgm16(m, W, H) == ref.encode16(host, png=False)
    assert pt.encode_png16(m, W, H) == ref.encode16(host, png=True)


# ---- texture epilogue and gradient / Hessian norm maps -------

@pytest.mark.skipif(not __import__("os").path.exists(__import__("os").path.join(
    __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))),
    "oracle", "_ref", "libtgref.so")), reason="reference build absent")
@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("method", [0, 3])
def test_texture_matches_reference_render(kind, method):
    from oracle.pyoracle import Reference

    c = make_cfg(method=method, seed=31, resolution=512, base_frequency=4, octaves=6)
    out = torch.empty((512, 512), dtype=torch.float32, device="cuda")
    assert _abi.load().tg_texture_generate_f32(C.byref(c), kind, 2.5, 4.0, out.data_ptr(), None) == 0
    torch.cuda.synchronize()
    ref = Reference().texture(c, kind, 2.5, 4.0)
    err = float(np.max(np.abs(out.cpu().numpy().astype(np.float64) - ref)))
    assert err <= 1e-5, err  # values in [-1, 1]


def test_norm_maps_match_restated_cli_stencils(oracle):
    c = make_cfg(method=0, smoothstep=5, seed=8, resolution=512, base_frequency=4, octaves=8)
    m = gen(c, 0, 0, 320, 200)
    host = m.cpu().numpy().astype(np.float64)
    for hess in (False, True):
        out = torch.empty_like(m)
        pt.norm_map_device(m, 320, 200, out, hessian=hess)
        torch.cuda.synchronize()
        ref = oracle.norm_map(host, hess).astype(np.float32)
        assert np.array_equal(out.cpu().numpy(), ref)


# ---- programmatic dependent launch: stream order of the output writes ---------

def test_back_to_back_launches_keep_stream_order():
    """The 2D kernel starts under programmatic stream serialisation and waits
    for the previous grid before its stores: back-to-back launches into ONE
    buffer (and a preceding torch fill / a following torch read on the same
    stream) must still leave exactly the last launch's map."""
    R = 1024
    lib = _abi.load()
    s = torch.cuda.Stream()
    buf = torch.empty((R, R), dtype=torch.float32, device="cuda")
    cfgs = [make_cfg(seed=sd, smoothstep=5, resolution=R, base_frequency=2, octaves=12) for sd in (3, 4, 5)]
    refs = [gen(c, 0, 0, R).cpu() for c in cfgs]
    with torch.cuda.stream(s):
        for it in range(40):
            buf.fill_(float("nan"))
            for c in cfgs[: 1 + it % 3]:
                assert lib.tg_fbm_generate_rect_f32(C.byref(c), 0, 0, R, R, buf.data_ptr(), R, s.cuda_stream) == 0
            snap = buf.clone()  # a torch kernel reading the output right after
            assert torch.equal(snap.cpu(), refs[it % 3]), it
    torch.cuda.synchronize()


# ---- permutation-table Perlin (new; parity unpinned: restated oracle) ---------------

@pytest.mark.parametrize("R,f0,octs,ratio,order", [(256, 2, 6, 2.0, 0), (240, 3, 5, 2.0, 3), (200, 2, 5, 1.7, 5),
                                                   (512, 8, 9, 2.0, 0)])
def test_perm_perlin_matches_restated_oracle(oracle, R, f0, octs, ratio, order):
    c = make_cfg(method=6, seed=31, resolution=R, base_frequency=f0, octaves=octs, frequency_ratio=ratio,
                 smoothstep=order)
    check_close(gen(c, 0, 0, R).cpu().numpy(), oracle.generate(c, 0, 0, R), c, f"perm R{R}")
    # negative origins wrap the table like the oracle's & 255
    o = -R
    check_close(gen(c, o, o, R).cpu().numpy(), oracle.generate(c, o, o, R), c, f"perm R{R} negative origin")


def test_perm_perlin_region_batch_and_zero():
    c = make_cfg(method=6, seed=77, resolution=512, base_frequency=4, octaves=7)
    full = gen(c, 0, 0, 512)
    assert torch.equal(gen(c, 128, 256, 256), full[256:, 128:384])
    cz = make_cfg(method=6, seed=77, resolution=512, base_frequency=4, octaves=7, zero_lattice=1)
    assert torch.count_nonzero(gen(cz, 0, 0, 128)) == 0
    cfg = pt.FbmConfig(method=pt.Method.perlin_perm, resolution=256, base_frequency=4, octaves=5)
    seeds = [3, 9, 27]
    out = torch.empty((3, 256, 256), dtype=torch.float32, device="cuda")
    pt.generate_batch_device(cfg, seeds, (0, 0), 256, 256, out)
    for i, s in enumerate(seeds):
        one = torch.empty((256, 256), dtype=torch.float32, device="cuda")
        pt.generate_into_device(pt.FbmConfig(method=pt.Method.perlin_perm, seed=s, resolution=256,
                                             base_frequency=4, octaves=5), (0, 0), 256, one)
        assert torch.equal(out[i], one)


def test_native_nccl_comm_one_rank_and_terrain_stats(oracle):
    # tg_comm_init_nccl with one rank (no torch.distributed): the NCCL
    # all-reduce path runs for real; the statistics equal the host-comm ones
    from paper_1610_03525_b200.shard import Comm, DeviceBackend, plan_band, terrain_stats

    comm = Comm.nccl(device=torch.device("cuda", 0))
    a = comm.allreduce(np.array([1, 2, 3], dtype=np.int64))
    assert list(a) == [1, 2, 3]
    f = comm.allreduce(np.array([0.5, -2.0]), op="max")
    assert list(f) == [0.5, -2.0]
    cfgp = pt.FbmConfig(method=0, smoothstep=5, seed=3, resolution=1024, base_frequency=4, octaves=12)
    sizes, lags = [2, 4, 8, 16, 32, 64], [1, 2, 4, 8, 16, 32, 64, 128, 256, 512]
    band = plan_band(1024, 1024, 1, 0, align=256, max_lag=512)
    s1 = terrain_stats(band, DeviceBackend(cfgp), comm, sizes, lags)
    s2 = terrain_stats(band, DeviceBackend(cfgp), Comm(), sizes, lags)
    comm.close()
    assert s1.sea_level == s2.sea_level and s1.counts == s2.counts and s1.coast_pixels == s2.coast_pixels
    # (the variogram sums use fp64 atomics across CTAs: equal to rounding, not bit for bit)
    assert np.array_equal(s1.pairs, s2.pairs) and np.allclose(s1.sum_sq, s2.sum_sq, rtol=1e-12, atol=0)
    assert 1.0 < s1.d_box < 2.0 and 2.0 < s1.d_variogram < 3.0


def test_race_stress_back_to_back_and_concurrent_streams():
    # compute-sanitizer is closed on this GPU pool (it left GPUs needing a
    # reset), so the shared-memory staging (pairwise named barriers over the
    # dead ppc-1 grid) and the programmatic-dependent-launch early start are
    # stress-tested instead: 48 back-to-back config-2 launches into distinct
    # buffers on one stream (grids overlap their neighbours' tails), then two
    # streams racing the same map, must all be bit-identical to an isolated
    # launch — a race shows up as a nondeterministic pixel.
    c = make_cfg(method=0, smoothstep=5, seed=1, resolution=4096, base_frequency=8, octaves=12)
    ref = gen(c, 0, 0, 2048, 1024)
    torch.cuda.synchronize()
    lib = _abi.load()
    outs = [torch.empty((1024, 2048), dtype=torch.float32, device="cuda") for _ in range(48)]
    s = torch.cuda.current_stream().cuda_stream
    for o in outs:
        assert lib.tg_fbm_generate_rect_f32(C.byref(c), 0, 0, 2048, 1024, o.data_ptr(), 2048, s) == 0
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    more = [torch.empty((1024, 2048), dtype=torch.float32, device="cuda") for _ in range(16)]
    for i, o in enumerate(more):
        st = (s1 if i % 2 else s2).cuda_stream
        assert lib.tg_fbm_generate_rect_f32(C.byref(c), 0, 0, 2048, 1024, o.data_ptr(), 2048, st) == 0
    torch.cuda.synchronize()
    for o in outs + more:
        assert torch.equal(o, ref)


def test_device_normalized_heightmap_equals_host_normalize(oracle):
    # generate_region with normalize: widening + normalize_map fused on the
    # device must give the host form's doubles bit for bit (fbm.hpp:638-656)
    for m in (0, 3, 6):
        cfg = pt.FbmConfig(method=m, seed=13, resolution=512, base_frequency=4, octaves=9, normalize=True)
        hm = pt.generate_region(cfg, (0, 0), 512)
        raw = pt.generate_region(pt.FbmConfig(method=m, seed=13, resolution=512, base_frequency=4, octaves=9),
                                 (0, 0), 512)
        ref = pt.normalize_map(raw)
        assert hm.normalized and np.array_equal(hm.data, ref.data)
        assert hm.source_min == ref.source_min and hm.source_max == ref.source_max
        assert len(hm.octave_seconds) == 9 and min(hm.octave_seconds) >= 0.0
    z = pt.generate_region(pt.FbmConfig(seed=1, resolution=64, octaves=3, normalize=True, zero_lattice=True),
                           (0, 0), 64)
    assert z.constant_source and not z.normalized and np.all(z.data == 0.0)


def test_octave_times_are_prefix_increments():
    c = make_cfg(method=0, smoothstep=5, seed=1, resolution=4096, base_frequency=8, octaves=12)
    t = (C.c_double * 12)()
    assert _abi.load().tg_fbm_octave_times(C.byref(c), 0, 0, 4096, t, None) == 0, _abi.last_error()
    assert all(v >= 0.0 for v in t) and 5e-6 < sum(t) < 5e-3
