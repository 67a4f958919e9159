"""GPU upper median (radix select with a sampled candidate window, analysis.cu
select_hist) against numpy: the selected element must be EXACTLY the
reference's `nth_element` at n/2 (analysis.hpp:244-250), whichever path the
window takes (kept candidates, or the full-read fallback when the sample
misleads or the window is too wide)."""
import numpy as np
import pytest

from helpers import make_cfg

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - GPU box only
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1610_03525_b200 as pt  # noqa: E402


def ref_median(t):
    h = t.detach().cpu().numpy().ravel()
    return float(np.partition(h, h.size // 2)[h.size // 2])


def gen(R, H, seed=3, octaves=12):
    import ctypes as C

    from paper_1610_03525_b200 import _abi

    c = make_cfg(seed=seed, resolution=max(R, H), base_frequency=8, octaves=octaves, smoothstep=5)
    out = torch.empty((H, R), dtype=torch.float32, device="cuda")
    assert _abi.load().tg_fbm_generate_rect_f32(C.byref(c), 0, 0, R, H, out.data_ptr(), R, None) == 0
    return out


@pytest.mark.parametrize("R,H", [(4096, 4096), (5000, 5000), (8192, 1031), (2048, 2049)])
def test_median_generated_maps(R, H):
    m = gen(R, H)
    assert pt.upper_median_device(m) == ref_median(m)


def test_median_constant_and_two_valued():
    n = 1 << 23
    z = torch.full((n,), 0.25, device="cuda")
    assert pt.upper_median_device(z) == 0.25  # window holds every key: full-read fallback
    z[: n // 2 + 1] = -3.0
    assert pt.upper_median_device(z) == ref_median(z)


def test_median_sample_misled_by_period():
    """Every sampled position (multiples of n / 65536) holds 1.0, all others lie
    in [-1, 0): the window misses the true median and the later passes read
    the map again."""
    n = 1 << 24
    g = torch.Generator(device="cuda").manual_seed(7)
    z = -torch.rand(n, device="cuda", generator=g)
    z[:: n // 65536] = 1.0
    assert pt.upper_median_device(z) == ref_median(z)


def test_median_duplicates_and_signs():
    n = (1 << 22) + 12345
    g = torch.Generator(device="cuda").manual_seed(11)
    z = torch.randint(-20, 21, (n,), device="cuda", generator=g).float() * 0.125
    z[::17] = -0.0
    z[1::19] = 0.0
    assert pt.upper_median_device(z) == ref_median(z)
    w = torch.randn(n, device="cuda", generator=g) * 1e-30  # tiny magnitudes, both signs
    assert pt.upper_median_device(w) == ref_median(w)
