"""Pin the 3D restatement (oracle.c) by the properties SURVEY §8c prescribes.

The reference has no 3D fBm; these properties anchor the
3D oracle on the reference's own 2D code (fixtures from
tests/golden/gen_pins3d.py via oracle/_ref), so that the GPU-vs-oracle 3D
tests (tests/test_gpu_fullshape.py, tests/test_gpu_parity.py) compare against
a pinned oracle:

1. face reduction — the separable 3D cell on z = 0 / z = 1 equals the
   reference's `kernels2d::zg_eval(..., ZgVariant::separable, order)` of the
   face's corners (kernels2d.hpp:62-76) within 1e-15;
2. corner exactness — the cell takes its corner values exactly
   (test_kernels2d.cpp:124-137 pattern, in 3D);
3. zero corner gradients — by finite differences along each axis at all 8
   corners (the boundary constraint of the paper's zero-gradient cell);
4. iz = 0 is the 2D lattice — pack3(seed, oct, ix, iy, 0) hashes to the
   reference's mix(pack(...)) and corner_height3 equals corner_height, bit for
   bit (lattice.hpp:35-64).
"""
import os

import numpy as np
import pytest

FIX = os.path.join(os.path.dirname(__file__), "golden", "pins3d.npz")


@pytest.fixture(scope="module")
def pins():
    return dict(np.load(FIX))


def test_face_reduces_to_reference_zg_separable(oracle, pins):
    h, xy, order = pins["h"], pins["xy"], pins["order"]
    worst = 0.0
    for i in range(len(h)):
        x, y, o = float(xy[i, 0]), float(xy[i, 1]), int(order[i])
        v0 = oracle.cell3(h[i], x, y, 0.0, o)
        v1 = oracle.cell3(h[i], x, y, 1.0, o)
        worst = max(worst, abs(v0 - pins["face_z0"][i]), abs(v1 - pins["face_z1"][i]))
    assert worst <= 1e-15, worst


def test_face_reduction_live_reference(oracle):
    from oracle.pyoracle import REF_SO, Reference

    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built here")
    ref = Reference()
    rng = np.random.default_rng(11)
    for _ in range(500):
        h = rng.uniform(-1, 1, 8)
        x, y = rng.uniform(0, 1, 2)
        for o in (3, 5):
            for z, face in ((0.0, h[0:4]), (1.0, h[4:8])):
                want = ref.lib.ref_zg_eval(*face, x, y, 1, o)
                assert abs(oracle.cell3(h, x, y, z, o) - want) <= 1e-15


@pytest.mark.parametrize("order", [3, 5])
def test_corner_exactness(oracle, order):
    rng = np.random.default_rng(5)
    for _ in range(200):
        h = rng.uniform(-1, 1, 8)
        for q in range(8):
            x, y, z = float(q & 1), float((q >> 1) & 1), float((q >> 2) & 1)
            assert oracle.cell3(h, x, y, z, order) == h[q]


@pytest.mark.parametrize("order", [3, 5])
def test_zero_corner_gradients_finite_difference(oracle, order):
    rng = np.random.default_rng(6)
    eps = 1e-5
    for _ in range(100):
        h = rng.uniform(-1, 1, 8)
        span = float(np.max(h) - np.min(h))
        for q in range(8):
            c = [float(q & 1), float((q >> 1) & 1), float((q >> 2) & 1)]
            v = oracle.cell3(h, *c, order)
            for ax in range(3):
                p = list(c)
                p[ax] += eps if c[ax] == 0.0 else -eps  # step into the cell
                slope = abs(oracle.cell3(h, *p, order) - v) / eps
                # S'(0) = S'(1) = 0: the one-sided difference is O(eps) (S3) or O(eps^2) (S5)
                assert slope <= 4.0 * eps * span + 1e-9, (q, ax, slope)


def test_iz0_is_the_2d_lattice(oracle, pins):
    seeds, octs, ixs, iys = pins["key_seed"], pins["key_octave"], pins["key_ix"], pins["key_iy"]
    for i in range(len(seeds)):
        s, o, x, y = int(seeds[i]), int(octs[i]), int(ixs[i]), int(iys[i])
        assert oracle.lib.or_mix(oracle.lib.or_pack3(s, o, x, y, 0)) == int(pins["hash_iz0"][i])
        assert oracle.lib.or_corner_height3(s, o, x, y, 0) == float(pins["height_iz0"][i])
    # and iz != 0 moves the key by iz * K5 (a different lattice point)
    assert oracle.lib.or_pack3(7, 0, 1, 2, 1) != oracle.lib.or_pack3(7, 0, 1, 2, 0)


def test_2d_separable_map_is_the_3d_cell_on_the_iz0_face(oracle):
    # The restated 2D separable map (pinned to the reference by
    # test_oracle_golden.py) equals, pixel for pixel, the restated 3D cell
    # evaluated at z = 0 over the 3D lattice's corners: properties 1 and 4
    # together, end to end through the octave's sampling.
    from helpers import make_cfg

    c = make_cfg(method=1, seed=21, resolution=64, base_frequency=4, octaves=1)
    h2 = oracle.generate(c, 0, 0, 64)
    rng = np.random.default_rng(8)
    for _ in range(64):
        gx, gy = (int(v) for v in rng.integers(0, 64, 2))
        ix, iy = gx // 16, gy // 16
        x, y = ((gx % 16) + 0.5) / 16, ((gy % 16) + 0.5) / 16
        hc = [oracle.lib.or_corner_height3(21, 0, ix + (q & 1), iy + ((q >> 1) & 1), (q >> 2) & 1)
              for q in range(8)]
        assert abs(oracle.cell3(hc, x, y, 0.0, 3) - h2[gy, gx]) <= 1e-15
