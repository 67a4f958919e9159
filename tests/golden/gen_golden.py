"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Runs only where /root/reference exists (this container): it builds
oracle/_ref/libtgref.so from the unmodified reference headers
(oracle/Makefile) and records the reference's own outputs.  The fixtures
are committed; the GPU box never reads /root/reference.

    python tests/golden/gen_golden.py

Fixtures:
  lattice.npz   keys + mix(pack(key)^lane) for the 3 lanes (u64), corner
                heights / angles / unit gradients / gradients (lattice.hpp)
  maps.npz      generate_into / generate_region windows per method and path
                (fbm.hpp), the S5 zero-gradient maps through the reference's
                own kernels (test_fbm.cpp:20-80 pattern), and the
                config-2 / config-5 scale proxies
  analysis.npz  coastline + box-count known answers (test_analysis.cpp)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.pyoracle import Reference, build, keys_array  # noqa: E402
from paper_1610_03525_b200._abi import TgFbmConfig  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
LANES = {"height": 0, "angle": 0xA0761D6478BD642F, "magnitude": 0xE7037ED1A0B428DB}


def cfg(**kw) -> TgFbmConfig:
    """FbmConfig defaults (fbm.hpp:49-60) plus overrides."""
    c = TgFbmConfig()
    c.seed, c.method, c.smoothstep, c.octaves, c.threads = 0, 0, 0, 1, 1
    c.resolution, c.base_frequency = 256, 2
    c.frequency_ratio, c.persistence, c.base_amplitude = 2.0, 0.5, 1.0
    c.gradient_weight, c.has_gradient_weight, c.normalize, c.zero_lattice = 0.0, 0, 0, 0
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def cfg_dict(c: TgFbmConfig) -> dict:
    return {name: getattr(c, name) for name, _ in c._fields_}


def lattice_fixture(ref: Reference) -> None:
    rng = np.random.default_rng(20240)
    keys = []
    for iy in range(32):
        for ix in range(32):
            keys.append((7, 0, ix, iy))
    keys += [(42, 3, -17, 2891), (0, 0, 0, 0), (1, 0, -1, -1), (2, 0, 5, -5),
             (2**64 - 1, 31, -(2**40), 2**40), (2**63, 7, 2**40, -(2**40)),
             (123456789, 12, -(2**31), 2**31 - 1), (99, 1, 2**62, -(2**62))]
    for _ in range(1000):
        keys.append((int(rng.integers(0, 2**63)) * 2 + int(rng.integers(0, 2)),
                     int(rng.integers(0, 32)),
                     int(rng.integers(-(2**41), 2**41)), int(rng.integers(-(2**41), 2**41))))
    k = keys_array(keys)
    data = {"seed": k["seed"], "octave": k["octave"], "ix": k["ix"], "iy": k["iy"]}
    for name, lane in LANES.items():
        data[f"hash_{name}"] = ref.hash_keys(k, lane)
    data["height"] = ref.corner_heights(k)
    data["angle"] = ref.corner_angles(k)
    data["unit_gradient"] = ref.unit_gradients(k)
    data["gradient_w037"] = ref.gradients(k, 0.37)
    np.savez_compressed(os.path.join(OUT, "lattice.npz"), **data)


def map_cases():
    """(name, cfg, kind, window) — kind: into | region | pixels (S5 zg)."""
    cases = []
    for m in range(5):
        for R in (8, 9):  # test_fbm.cpp:165-177 — fast and general (non-dividing) path
            cases.append((f"m{m}_R{R}_N3", cfg(method=m, seed=1234, resolution=R, octaves=3), "into", (0, 0, R)))
        cases.append((f"m{m}_R16_ratio17", cfg(method=m, seed=5, resolution=16, octaves=4, frequency_ratio=1.7),
                      "into", (0, 0, 16)))  # test_fbm.cpp:179-190
        cases.append((f"m{m}_R8_subpixel", cfg(method=m, seed=99, resolution=8, octaves=5), "into", (0, 0, 8)))
        cases.append((f"m{m}_R64_N6", cfg(method=m, seed=31337, resolution=64, octaves=6), "into", (0, 0, 64)))
        for ratio in (2.0, 1.7):  # test_fbm.cpp:256-273 — region == submap
            cases.append((f"m{m}_region_ratio{int(ratio*10)}",
                          cfg(method=m, seed=909, resolution=64, octaves=3, frequency_ratio=ratio),
                          "region", (32, 32, 32)))
        cases.append((f"m{m}_negorigin", cfg(method=m, seed=3, resolution=64, octaves=4), "region", (32, -32, 16)))
        cases.append((f"m{m}_R48_f3", cfg(method=m, seed=77, resolution=48, base_frequency=3, octaves=6),
                      "into", (0, 0, 48)))  # ppc 16, 8, 4, 2, 1 then sub-pixel k=2 (non power-of-2 R)
    cases.append(("zg_R128_N4_tiles", cfg(seed=4242, resolution=128, octaves=4), "into", (0, 0, 128)))
    cases.append(("zg_normalize", cfg(seed=21, resolution=32, octaves=3, normalize=1), "region", (0, 0, 32)))
    cases.append(("generic_w05", cfg(method=2, seed=8, resolution=32, octaves=3, gradient_weight=0.5,
                                     has_gradient_weight=1), "into", (0, 0, 32)))
    cases.append(("zero_source", cfg(method=0, resolution=16, octaves=4, zero_lattice=1), "into", (0, 0, 16)))
    # zero-gradient S5 (not expressible in FbmConfig): reference kernels per pixel.
    for sep in (0, 1):
        cases.append((f"zg{sep}_S5_R64_N6", cfg(method=sep, smoothstep=5, seed=42, resolution=64, octaves=6),
                      "pixels", (0, 0, 64)))
    # Config 2 scale proxy: (R=512, f0=1) has the ppc sequence of (4096, f0=8), so
    # its map equals the top-left 512^2 of config 2.  S5 zg_paper, 12 octaves.
    cases.append(("cfg2_proxy_S5", cfg(method=0, smoothstep=5, seed=1, resolution=512, base_frequency=1,
                                       octaves=12), "pixels", (0, 0, 128)))
    cases.append(("cfg2_proxy_S3", cfg(method=0, seed=1, resolution=512, base_frequency=1, octaves=12),
                  "into", (0, 0, 512)))
    # Config 5 proxy: (R=1024, f0=1, N=16) = top-left chunk of (32768, f0=32).
    cases.append(("cfg5_proxy_S5", cfg(method=0, smoothstep=5, seed=1, resolution=1024, base_frequency=1,
                                       octaves=16), "pixels", (0, 0, 64)))
    # Config 1: R=1024 N=8 f0=8 zg_paper S3 (window).
    cases.append(("cfg1_window", cfg(method=0, seed=1, resolution=1024, base_frequency=8, octaves=8),
                  "region", (0, 0, 128)))
    # Perlin on the config-3 grid proxy (R=512, f0=1, N=12).
    for m in (3, 4):
        cases.append((f"cfg3_proxy_m{m}", cfg(method=m, seed=1, resolution=512, base_frequency=1, octaves=12),
                      "region", (0, 0, 64)))
    return cases


def maps_fixture(ref: Reference) -> None:
    data, meta = {}, {}
    for name, c, kind, (ox, oy, ext) in map_cases():
        if kind == "into":
            st, m, nw = ref.generate_into(c, ox, oy, ext)
            assert st == 0, (name, ref.last_error())
            info = {"warnings": nw}
        elif kind == "region":
            m, info = ref.generate_region(c, ox, oy, ext)
        else:
            m = ref.oracle_pixels(c, ox, oy, ext)
            info = {}
        if name == "cfg2_proxy_S3":
            m = m[:128, :128]  # keep the fixture small; the window is a pure function of pixels
            ext = 128
        data[name] = m
        meta[name] = {"cfg": cfg_dict(c), "kind": kind, "origin": [ox, oy], "extent": ext, **info}
    np.savez_compressed(os.path.join(OUT, "maps.npz"), **data)
    with open(os.path.join(OUT, "maps.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


def analysis_fixture(ref: Reference) -> None:
    data = {}
    col = np.zeros((64, 64), np.uint8)
    col[:, 31] = 1  # test_analysis.cpp:218-229
    st, counts, d, k, r2 = ref.box_count_mask(col, [2, 4, 8, 16])
    data["column_counts"], data["column_dkr2"] = counts, np.array([d, k, r2])
    filled = np.ones((64, 64), np.uint8)  # 231-240
    st, counts, d, k, r2 = ref.box_count_mask(filled, [2, 4, 8, 16])
    data["filled_counts"], data["filled_dkr2"] = counts, np.array([d, k, r2])
    half = np.where(np.arange(8)[None, :] < 4, 1.0, -1.0) * np.ones((8, 1))  # 189-200
    r = ref.coastline_boxcount(half, [], sea=0.0, want_mask=True)
    data["halfplane_mask"] = r["mask"]
    # test_map(128, 6): seed 42 generated map, median coastline, default sizes (242-251)
    m, _ = ref.generate_region(cfg(seed=42, resolution=128, octaves=6), 0, 0, 128)
    r = ref.coastline_boxcount(m, [2, 4, 8, 16, 32, 64], sea=None, want_mask=True)
    data["testmap128"] = m
    data["testmap128_counts"] = r["counts"]
    data["testmap128_mask"] = r["mask"]
    data["testmap128_stats"] = np.array([r["d"], r["k"], r["r2"], r["land_fraction"], r["sea"],
                                         r["coast_pixels"]])
    np.savez_compressed(os.path.join(OUT, "analysis.npz"), **data)


def main() -> None:
    build()
    ref = Reference()
    lattice_fixture(ref)
    maps_fixture(ref)
    analysis_fixture(ref)
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
