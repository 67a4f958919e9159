"""Permutation-table Perlin (TG_METHOD_PERLIN_PERM, new; parity unpinned):
properties of the restated oracle (oracle.c or_perm_table / or_perm_gradient)
that the GPU kernel (csrc/perm2d.cu) is then compared against."""
import math

import numpy as np

from helpers import make_cfg


def test_table_is_a_seeded_permutation(oracle):
    tabs = [oracle.perm_table(s) for s in (0, 1, 42, 2**64 - 1)]
    for t in tabs:
        assert sorted(t.tolist()) == list(range(256))
    assert len({t.tobytes() for t in tabs}) == len(tabs)  # seeds give different tables
    assert np.array_equal(oracle.perm_table(42), tabs[2])  # deterministic


def test_gradients_are_the_8_unit_vectors_and_cover_them(oracle):
    seen = set()
    for ix in range(-20, 20):
        for iy in range(-20, 20):
            gx, gy = oracle.perm_gradient(7, 3, ix, iy)
            assert abs(math.hypot(gx, gy) - 1.0) < 1e-15
            seen.add((round(gx, 6), round(gy, 6)))
    assert len(seen) == 8
    # periodic with period 256 in each lattice direction (the classic table)
    assert oracle.perm_gradient(7, 3, 5, 9) == oracle.perm_gradient(7, 3, 5 + 256, 9 - 512)


def test_octaves_are_decorrelated_and_lattice_points_are_zero(oracle):
    c = make_cfg(method=6, seed=5, resolution=256, base_frequency=32, octaves=1)
    m0 = oracle.generate(c, 0, 0, 256)  # 32 x 32 cells
    assert abs(float(m0.mean())) < 0.05 and 0.05 < float(m0.std()) < 0.6
    # an octave sampled on lattice points (freq = 2R) contributes exactly 0
    c2 = make_cfg(method=6, seed=5, resolution=64, base_frequency=128, octaves=1)
    assert np.all(oracle.generate(c2, 0, 0, 64) == 0.0)
    g = [oracle.perm_gradient(11, o, 3, 4) for o in range(8)]
    assert len(set(g)) > 1
