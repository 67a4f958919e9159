"""Full-shape GPU parity on every BASELINE.json config (north-star tolerance).

Each map is generated on the device through the C-ABI and compared pixel by
pixel against the threaded C oracle (`or_generate_mt`, bit-identical to the
single-thread restatement that tests/test_oracle_golden.py pins to the
compiled reference):

* config 1 (1024^2, zg_paper S3, 8 octaves) and config 2 (4096^2, zg_paper
  S5, 12 octaves) — entire maps;
* config 3 (4096^2, 12 octaves) — entire maps for zg paper / separable,
  generic, Perlin S3 and S5, OpenSimplex and the permutation-table Perlin;
* config 5 (32768^2, f0 = 32, 16 octaves, S5) — four full 1024^2 chunks
  (interior, last column, last row, bottom-right corner) and one whole row
  band of 1024 x 32768;
* config 4 (512^3, zg separable S3, 8 octaves, f0 = 8) — 64^3 windows at
  three corners of the volume plus 10^5 random voxels.

The bar is max|dh| <= 1e-5 * A with A = max|h_ref| over the compared window
(helpers.height_tolerance).  Because A is a window maximum, the tightest case
is a window of small amplitude; `_every_window` therefore also applies the
bound to EVERY 64 x 64 window of configs 2 and 5 with that window's own A.
"""
import ctypes as C
import os

import numpy as np
import pytest

from helpers import height_tolerance, make_cfg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1610_03525_b200 as pt  # noqa: E402
from paper_1610_03525_b200 import _abi  # noqa: E402

THREADS = os.cpu_count() or 1


def gen(c, ox, oy, w, h=None):
    h = w if h is None else h
    out = torch.empty((h, w), dtype=torch.float32, device="cuda")
    st = _abi.load().tg_fbm_generate_rect_f32(C.byref(c), ox, oy, w, h, out.data_ptr(), w,
                                              torch.cuda.current_stream().cuda_stream)
    assert st == 0, _abi.last_error()
    return out.cpu().numpy()


def check_close(got, ref, c, what):
    tol = height_tolerance(ref, c)
    err = float(np.max(np.abs(got.astype(np.float64) - ref)))
    assert err <= tol, f"{what}: max|dh|={err:.3e} > tol={tol:.3e}"
    return err


def _every_window(got, ref, what, win=64):
    """max|dh| <= 1e-5 * A_w in every win x win window w (A_w its own max|h_ref|)."""
    H, W = ref.shape
    d = np.abs(got.astype(np.float64) - ref)[: H // win * win, : W // win * win]
    a = np.abs(ref)[: H // win * win, : W // win * win]
    shape = (H // win, win, W // win, win)
    err_w = d.reshape(shape).max(axis=(1, 3))
    amp_w = a.reshape(shape).max(axis=(1, 3))
    ratio = err_w / (1e-5 * amp_w)
    i = np.unravel_index(int(np.argmax(ratio)), ratio.shape)
    j = np.unravel_index(int(np.argmin(amp_w)), amp_w.shape)
    assert ratio[i] <= 1.0, (f"{what}: window {i} max|dh|={err_w[i]:.3e} > 1e-5*A={1e-5 * amp_w[i]:.3e} "
                             f"(smallest-amplitude window {j}: A={amp_w[j]:.3e}, max|dh|={err_w[j]:.3e})")
    return float(amp_w[j]), float(err_w[j])


def test_config1_entire_map(oracle):
    c = make_cfg(method=0, seed=1, resolution=1024, base_frequency=8, octaves=8)
    check_close(gen(c, 0, 0, 1024), oracle.generate_mt(c, 0, 0, 1024, threads=THREADS), c, "cfg1")


def test_config2_entire_map_and_every_window(oracle):
    c = make_cfg(method=0, smoothstep=5, seed=1, resolution=4096, base_frequency=8, octaves=12)
    got = gen(c, 0, 0, 4096)
    ref = oracle.generate_mt(c, 0, 0, 4096, threads=THREADS)
    check_close(got, ref, c, "cfg2 full map")
    _every_window(got, ref, "cfg2")


# zg paper, zg separable, generic, perlin3, perlin5, OpenSimplex, permutation-table Perlin
@pytest.mark.parametrize("method", [0, 1, 2, 3, 4, 5, 6])
def test_config3_entire_maps(oracle, method):
    c = make_cfg(method=method, seed=1, resolution=4096, base_frequency=8, octaves=12)
    check_close(gen(c, 0, 0, 4096), oracle.generate_mt(c, 0, 0, 4096, threads=THREADS), c,
                f"cfg3 method {method}")


CFG5 = dict(method=0, smoothstep=5, seed=1, resolution=32768, base_frequency=32, octaves=16)


@pytest.mark.parametrize("cx,cy", [(17, 29), (31, 5), (7, 31), (31, 31)])
def test_config5_full_chunks(oracle, cx, cy):
    # 1024^2 chunks of the 32768^2 terrain (interior, last column, last row, corner)
    c = make_cfg(**CFG5)
    ox, oy = cx * 1024, cy * 1024
    got = gen(c, ox, oy, 1024)
    ref = oracle.generate_mt(c, ox, oy, 1024, threads=THREADS)
    check_close(got, ref, c, f"cfg5 chunk ({cx},{cy})")
    _every_window(got, ref, f"cfg5 chunk ({cx},{cy})")


def test_config5_whole_row_band(oracle):
    # one multi-GPU row band (the sharding unit, 1024 rows x the full width)
    c = make_cfg(**CFG5)
    oy = 12 * 1024
    got = gen(c, 0, oy, 32768, 1024)
    ref = oracle.generate_mt(c, 0, oy, 32768, 1024, threads=THREADS)
    check_close(got, ref, c, "cfg5 row band")
    _every_window(got, ref, "cfg5 row band")


def test_config4_volume_windows_and_random_voxels(oracle):
    cfg = pt.FbmConfig(method=1, seed=1, resolution=512, base_frequency=8, octaves=8)
    c = cfg.to_c()
    vol = torch.empty((512, 512, 512), dtype=torch.float32, device="cuda")
    pt.generate3d_device(cfg, (0, 0, 0), (512, 512, 512), vol)
    torch.cuda.synchronize()
    for (x, y, z) in [(0, 0, 0), (448, 448, 448), (448, 0, 192)]:
        got = vol[z:z + 64, y:y + 64, x:x + 64].cpu().numpy()
        ref = oracle.generate3d(c, x, y, z, 64, 64, 64)
        check_close(got, ref, c, f"cfg4 window ({x},{y},{z})")
    rng = np.random.default_rng(4)
    n = 100_000
    xs, ys, zs = (rng.integers(0, 512, n) for _ in range(3))
    ref = oracle.sample3d(c, xs, ys, zs)
    got = vol[torch.from_numpy(zs).cuda(), torch.from_numpy(ys).cuda(), torch.from_numpy(xs).cuda()]
    check_close(got.cpu().numpy(), ref, c, "cfg4 random voxels")
