"""GPU variogram: the register-ring walks (csrc/vgring.cu) against fp64 sums.

The variogram is new (the reference has none): parity is against the
oracle's double restatement (`or_variogram`) and, for band windows, a numpy
fp64 restatement of the same pair definition — pair counts exact, sums within
1e-10 relative (the GPU adds the same fp64 terms in another order).  Power-of-
two lags up to 4096 take the ring path; every case is also run through the
generic kernels (TG_VG_GENERIC) so both paths agree on the same map.
"""
import ctypes as C
import os

import numpy as np
import pytest

from helpers import make_cfg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1610_03525_b200 import _abi  # noqa: E402

POW2 = [1 << i for i in range(13)]  # 1 .. 4096 (config 5)


def gen(c, w, h):
    out = torch.empty((h, w), dtype=torch.float32, device="cuda")
    assert _abi.load().tg_fbm_generate_rect_f32(C.byref(c), 0, 0, w, h, out.data_ptr(), w,
                                                torch.cuda.current_stream().cuda_stream) == 0
    return out


def band_variogram_np(z, lags, P):
    """Pairs along x in rows [0, P); along y (r, r + h) with r < P, r + h < H."""
    H, W = z.shape
    ss = np.zeros((len(lags), 2))
    pr = np.zeros((len(lags), 2), dtype=np.int64)
    for i, h in enumerate(lags):
        if h < W:
            d = z[:P, h:] - z[:P, :W - h]
            ss[i, 0], pr[i, 0] = float(np.sum(d * d)), d.size
        ny = min(P, H - h)
        if ny > 0:
            d = z[h:h + ny, :] - z[:ny, :]
            ss[i, 1], pr[i, 1] = float(np.sum(d * d)), d.size
    return ss, pr


def run_band(dev, W, H, ld, P, lags, generic=False):
    arr = (C.c_int32 * len(lags))(*lags)
    ss = (C.c_double * (2 * len(lags)))()
    pr = (C.c_int64 * (2 * len(lags)))()
    if generic:
        os.environ["TG_VG_GENERIC"] = "1"
    try:
        st = _abi.load().tg_variogram_band_f32(dev.data_ptr(), W, H, ld, P, arr, len(lags), ss, pr, None)
    finally:
        os.environ.pop("TG_VG_GENERIC", None)
    assert st == 0, _abi.last_error()
    return np.array(ss[:]).reshape(-1, 2), np.array(pr[:], dtype=np.int64).reshape(-1, 2)


def _map(W, H, seed=9):
    c = make_cfg(method=0, smoothstep=5, seed=seed, resolution=16384, base_frequency=32, octaves=12)
    return gen(c, W, H)


def _close(a, b):
    # lags without pairs sum to exactly 0 on both sides
    assert np.allclose(a, b, rtol=1e-10, atol=0), np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))


@pytest.mark.parametrize("W,H", [(512, 512), (700, 300), (4097, 33), (20000, 40), (33, 5000), (1, 70), (70, 1),
                                 (16384, 17), (4096, 4200)])
def test_ring_whole_map_matches_oracle(oracle, W, H):
    m = _map(W, H)
    lags = [h for h in POW2]
    ss, pr = run_band(m, W, H, W, H, lags)
    rss, rpr = oracle.variogram(m.cpu().numpy().astype(np.float64), lags)
    assert np.array_equal(pr, rpr)
    _close(ss, rss)
    gss, gpr = run_band(m, W, H, W, H, lags, generic=True)
    assert np.array_equal(gpr, pr)
    _close(ss, gss)


@pytest.mark.parametrize("lags", [[2, 64, 2048], [16, 1, 4, 4096], [1024], [512, 32], [8, 8, 1, 8], [4096, 1]])
def test_ring_partial_lag_sets_and_repeats(oracle, lags):
    W, H = 5000, 4500
    m = _map(W, H, seed=3)
    ss, pr = run_band(m, W, H, W, H, lags)
    rss, rpr = oracle.variogram(m.cpu().numpy().astype(np.float64), lags)
    assert np.array_equal(pr, rpr)
    _close(ss, rss)


@pytest.mark.parametrize("W,H,P,ld", [(3000, 2600, 1000, 3000), (2048, 5000, 4999, 2051), (600, 1200, 37, 640),
                                      (9000, 1100, 64, 9000)])
def test_ring_band_windows(W, H, P, ld):
    """Band mode (pair_rows P < H, the rows below regenerated as look-ahead) with
    a row pitch ld >= W (unaligned pitches take the scalar staging loads)."""
    full = _map(ld, H, seed=5)
    ss, pr = run_band(full, W, H, ld, P, POW2)
    z = full[:, :W].cpu().numpy().astype(np.float64)
    rss, rpr = band_variogram_np(z, POW2, P)
    assert np.array_equal(pr, rpr)
    _close(ss, rss)
    gss, _ = run_band(full, W, H, ld, P, POW2, generic=True)
    _close(ss, gss)


def test_ring_special_values():
    """Zeros, signed zeros, subnormals and a huge row (inf squares) on the ring path."""
    g = torch.Generator().manual_seed(4)
    m = torch.randn((300, 1100), generator=g)
    m[::3, ::5] = 0.0
    m[1::7, ::3] = -0.0
    m[2::5, 1::4] = 1e-40
    m[3::9, 2::6] = -3e-42
    m[5, :] = 3.0e38
    dev = m.cuda()
    lags = [1, 2, 4, 8, 16, 32, 64, 128, 256, 1024]
    ss, pr = run_band(dev, 1100, 300, 1100, 300, lags)
    rss, rpr = band_variogram_np(m.numpy().astype(np.float64), lags, 300)
    assert np.array_equal(pr, rpr)
    fin = np.isfinite(rss)
    assert np.array_equal(fin, np.isfinite(ss))
    _close(ss[fin], rss[fin])


def test_ring_config5_shape_properties():
    """Config-5 width (32768) on a 64-row band + 4096 look-ahead rows: the ring path
    and the generic kernels agree on every lag, pair counts by formula."""
    W, H, P = 32768, 64 + 4096, 64
    c = make_cfg(method=0, smoothstep=5, seed=1, resolution=32768, base_frequency=32, octaves=16)
    m = gen(c, W, H)
    ss, pr = run_band(m, W, H, W, P, POW2)
    gss, gpr = run_band(m, W, H, W, P, POW2, generic=True)
    assert np.array_equal(pr, gpr)
    _close(ss, gss)
    for i, h in enumerate(POW2):
        assert pr[i, 0] == (W - h) * P and pr[i, 1] == W * min(P, H - h)
