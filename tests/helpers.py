"""Shared test helpers (config construction mirrors FbmConfig defaults, fbm.hpp:49-60)."""
from __future__ import annotations

import numpy as np

from paper_1610_03525_b200._abi import TgFbmConfig


def make_cfg(**kw) -> TgFbmConfig:
    c = TgFbmConfig()
    c.seed, c.method, c.smoothstep, c.octaves, c.threads = 0, 0, 0, 1, 1
    c.resolution, c.base_frequency = 256, 2
    c.frequency_ratio, c.persistence, c.base_amplitude = 2.0, 0.5, 1.0
    c.gradient_weight, c.has_gradient_weight, c.normalize, c.zero_lattice = 0.0, 0, 0, 0
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def cfg_from_dict(d: dict) -> TgFbmConfig:
    return make_cfg(**d)


def keys_from_golden(lat: dict) -> np.ndarray:
    dt = np.dtype([("seed", "<u8"), ("octave", "<u4"), ("pad", "<u4"), ("ix", "<i8"), ("iy", "<i8")])
    k = np.zeros(len(lat["seed"]), dtype=dt)
    k["seed"], k["octave"], k["ix"], k["iy"] = lat["seed"], lat["octave"], lat["ix"], lat["iy"]
    return k


def amplitude_sum(cfg: TgFbmConfig) -> float:
    """h0 * sum_{i<N} p^i: the map amplitude scale used when max|h_ref| ~ 0."""
    return cfg.base_amplitude * sum(cfg.persistence ** i for i in range(cfg.octaves))


def height_tolerance(ref: np.ndarray, cfg: TgFbmConfig) -> float:
    """North-star bound: max |dh| <= 1e-5 * A, A = max |h_ref| over the window
    (falls back to h0 * sum p^i when the window is ~0)."""
    a = float(np.max(np.abs(ref))) if ref.size else 0.0
    if a < 1e-12:
        a = amplitude_sum(cfg)
    return 1e-5 * a
