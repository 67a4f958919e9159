"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/polyterrain_b200.h declares, and its host logic (validation,
octave_spec, window rules) matches the reference's rules.  No kernels launch."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from helpers import make_cfg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1610_03525_b200 import _abi
    from paper_1610_03525_b200.build import build

    build()
    return _abi.load()


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "polyterrain_b200.h")).read()
    return sorted(set(re.findall(r"\b(tg_[a-z0-9_]+)\s*\(", txt)))


def test_header_and_bindings_agree():
    from paper_1610_03525_b200._abi import SIGNATURES

    assert set(declared_symbols()) == set(SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.tg_abi_version() == 1


def test_validation_matches_reference_rules(lib, oracle):
    cases = [dict(), dict(octaves=0), dict(octaves=32), dict(octaves=33), dict(resolution=0),
             dict(persistence=0.0), dict(persistence=1.0), dict(persistence=1.5),
             dict(frequency_ratio=1.0), dict(frequency_ratio=float("inf")),
             dict(base_amplitude=0.0), dict(base_amplitude=-1.0), dict(threads=-1), dict(threads=257),
             dict(has_gradient_weight=1, gradient_weight=-0.1),
             dict(has_gradient_weight=1, gradient_weight=float("nan")), dict(base_frequency=0),
             dict(method=5), dict(smoothstep=4), dict(smoothstep=5), dict(resolution=32768)]
    for kw in cases:
        c = make_cfg(**kw)
        assert lib.tg_fbm_validate(C.byref(c)) == oracle.validate(c), kw


def test_octave_spec_matches_oracle(lib, oracle):
    from paper_1610_03525_b200._abi import TgOctaveSpec

    rng = np.random.default_rng(3)
    for _ in range(200):
        c = make_cfg(resolution=int(rng.choice([8, 9, 48, 1000, 1024, 4096, 32768])),
                     base_frequency=int(rng.integers(1, 40)), octaves=int(rng.integers(1, 20)),
                     frequency_ratio=float(rng.choice([2.0, 1.7, 3.0, 2.5])))
        for o in range(c.octaves):
            a, b = TgOctaveSpec(), oracle.octave_spec(c, o)
            assert lib.tg_fbm_octave_spec(C.byref(c), o, C.byref(a)) == 0
            assert (a.freq, a.amp, a.fast, a.cells, a.ppc) == (b.freq, b.amp, b.fast, b.cells, b.ppc)


def test_window_rules(lib):
    c = make_cfg(resolution=64)  # f0 = 2 -> octave-0 cells of 32 px (fbm.hpp:551-558)
    assert lib.tg_fbm_validate_window(C.byref(c), 5, 0, 16, 16) == 1
    assert lib.tg_fbm_validate_window(C.byref(c), 0, 33, 16, 16) == 1
    assert lib.tg_fbm_validate_window(C.byref(c), 32, -32, 16, 16) == 0
    assert lib.tg_fbm_validate_window(C.byref(c), 1 << 41, 0, 16, 16) == 1
    assert lib.tg_fbm_validate_window(C.byref(c), 0, 0, 0, 16) == 1


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback(lib):
    import paper_1610_03525_b200 as pt

    assert lib.tg_device_count() == 0
    with pytest.raises(pt.DeviceError):
        pt.generate_heightmap(pt.FbmConfig(resolution=16, octaves=2))
    c = make_cfg()
    assert lib.tg_fbm_generate_rect_f32(C.byref(c), 0, 0, 4, 4, C.c_void_p(16), 4, None) == 4
    assert "no CPU fallback" in lib.tg_last_error().decode()


def test_terrain_stats_buffer_validation(lib):
    """tg_terrain_stats_band_buf rejects a null band buffer before touching a device."""
    from paper_1610_03525_b200 import _abi

    c = make_cfg()
    t = _abi.TgTerrain(0, 64, 0, 64, 64, 1)
    b = _abi.TgBand(0, 64, 0, 0)
    sz = (C.c_int32 * 3)(2, 4, 8)
    lg = (C.c_int32 * 1)(1)
    st = _abi.TgTerrainStats()
    assert lib.tg_terrain_stats_band_buf(C.byref(c), C.byref(t), C.byref(b), None, 1, sz, 3, lg, 1, None, None,
                                         C.byref(st), None) == 1
    assert "null argument" in lib.tg_last_error().decode()


def test_python_mirror_surface():
    import paper_1610_03525_b200 as pt

    for m in pt.Method:
        assert pt.parse_method(pt.method_name(m)) == m
    assert pt.parse_method("simplex") is None
    cfg = pt.FbmConfig(base_amplitude=2.0)
    assert cfg.gradient_weight_value() == 0.02
    cfg.gradient_weight = 0.5
    assert cfg.gradient_weight_value() == 0.5
    assert pt.FbmConfig(method=pt.Method.perlin5).smoothstep_order() == 5
    with pytest.raises(pt.ValidationError):
        pt.FbmConfig(octaves=0).validate()
    fit = pt.linear_fit([0.0, 1.0, 2.0, 3.0], [2.5 * x - 1.25 for x in (0.0, 1.0, 2.0, 3.0)])
    assert abs(fit.slope - 2.5) < 1e-14 and fit.r2 == 1.0
