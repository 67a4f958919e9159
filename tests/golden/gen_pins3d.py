"""Generate tests/golden/pins3d.npz from the REAL reference (3D property pins).

The reference has no 3D path, so the 3D restatement
(oracle.c `or_cell3`, `or_corner_height3`) is pinned through the properties
SURVEY §8c prescribes, each anchored on the reference's own 2D code:

* face reduction: the separable 3D cell on z = 0 (z = 1) equals
  `kernels2d::zg_eval(zg_params(face corners), x, y, ZgVariant::separable,
  order)` (kernels2d.hpp:62-76) of that face's four corners;
* the 3D key at iz = 0 is the 2D key: `or_pack3(..., iz = 0)` hashed equals
  `lattice::detail::mix(pack(...))` (lattice.hpp:35-50) and the corner height
  equals `corner_height` (lattice.hpp:56-64) bit for bit.

This script records the reference side (ref_zg_eval, ref_hash_keys,
ref_corner_heights through oracle/_ref) for seeded random inputs; the test
(tests/test_pins3d.py) evaluates the restatement on the same inputs.

    python tests/golden/gen_pins3d.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Reference, build, keys_array  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "pins3d.npz")


def face_cases(rng, n):
    h = rng.uniform(-1.0, 1.0, (n, 8))
    xy = rng.uniform(0.0, 1.0, (n, 2))
    # cell edges and centre too (the reference's own probe points,
    # test_kernels2d.cpp:124-143)
    edge = np.array([[0, 0], [1, 0], [0, 1], [1, 1], [0.5, 0.5], [0.25, 0.75], [1, 0.5], [0.5, 0]])
    xy[: len(edge)] = edge
    order = np.where(rng.integers(0, 2, n) == 1, 5, 3).astype(np.int32)
    return h, xy, order


def main() -> None:
    build()
    ref = Reference()
    rng = np.random.default_rng(3303)
    n = 4000
    h, xy, order = face_cases(rng, n)
    z0 = np.array([ref.lib.ref_zg_eval(*h[i, 0:4], xy[i, 0], xy[i, 1], 1, int(order[i])) for i in range(n)])
    z1 = np.array([ref.lib.ref_zg_eval(*h[i, 4:8], xy[i, 0], xy[i, 1], 1, int(order[i])) for i in range(n)])
    keys = [(int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2)), int(rng.integers(0, 32)),
             int(rng.integers(-2**40, 2**40)), int(rng.integers(-2**40, 2**40))) for _ in range(1000)]
    keys += [(7, 0, ix, iy) for ix in range(-4, 4) for iy in range(-4, 4)]
    keys += [(2**64 - 1, 31, -(2**40), 2**40), (0, 0, 0, 0), (42, 3, -17, 2891)]
    ka = keys_array(keys)
    hashes = np.zeros(len(ka), dtype=np.uint64)
    ref.lib.ref_hash_keys(ka.ctypes.data, len(ka), 0, hashes.ctypes.data)
    heights = np.zeros(len(ka))
    ref.lib.ref_corner_heights(ka.ctypes.data, len(ka), heights.ctypes.data)
    np.savez_compressed(OUT, h=h, xy=xy, order=order, face_z0=z0, face_z1=z1,
                        key_seed=ka["seed"], key_octave=ka["octave"], key_ix=ka["ix"], key_iy=ka["iy"],
                        hash_iz0=hashes, height_iz0=heights)
    print(f"wrote {OUT}: {n} face cases, {len(ka)} keys")


if __name__ == "__main__":
    main()
