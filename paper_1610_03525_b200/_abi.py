"""ctypes view of the C-ABI declared in include/polyterrain_b200.h.

Only plain pointers and sizes cross this boundary (no torch types).  The
library is built in-tree by ``paper_1610_03525_b200/build.py`` into
``paper_1610_03525_b200/lib/libpolyterrain_b200.so``; there is no CPU
fallback — loading fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TG_LIB_PATH") or os.path.join(HERE, "lib", "libpolyterrain_b200.so")

TG_OK, TG_EVALIDATION, TG_EIO, TG_ENUMERICAL, TG_EDEVICE = 0, 1, 2, 3, 4

TG_METHOD_ZG_PAPER = 0
TG_METHOD_ZG_SEPARABLE = 1
TG_METHOD_GENERIC = 2
TG_METHOD_PERLIN3 = 3
TG_METHOD_PERLIN5 = 4
TG_METHOD_OPENSIMPLEX = 5
TG_METHOD_PERLIN_PERM = 6

TG_MAX_RESOLUTION = 1 << 22
TG_MAX_EXTENT = 1 << 17
TG_MAX_OCTAVES = 32

TG_LANE_HEIGHT = 0
TG_LANE_ANGLE = 0xA0761D6478BD642F
TG_LANE_MAGNITUDE = 0xE7037ED1A0B428DB
TG_LANE_SIMPLEX = 0x8EBC6AF09C88C6E3
TG_PACK_K5 = 0xA24BAED4963EE407
TG_LANE_PERM = 0x5851F42D4C957F2D
TG_PERM_KI = 0xD1B54A32D192ED03
TG_MAX_BOX_SIZES = 16
TG_MAX_LAGS = 32


class TgFbmConfig(C.Structure):
    """struct tg_fbm_config (mirror of terrain::fbm::FbmConfig, fbm.hpp:49-89)."""

    _fields_ = [
        ("seed", C.c_uint64),
        ("method", C.c_int32),
        ("smoothstep", C.c_int32),
        ("octaves", C.c_int32),
        ("threads", C.c_int32),
        ("resolution", C.c_int64),
        ("base_frequency", C.c_int64),
        ("frequency_ratio", C.c_double),
        ("persistence", C.c_double),
        ("base_amplitude", C.c_double),
        ("gradient_weight", C.c_double),
        ("has_gradient_weight", C.c_int32),
        ("normalize", C.c_int32),
        ("zero_lattice", C.c_int32),
        ("reserved", C.c_int32),
    ]


class TgOctaveSpec(C.Structure):
    """struct tg_octave_spec (fbm.hpp:143-149)."""

    _fields_ = [
        ("freq", C.c_double),
        ("amp", C.c_double),
        ("fast", C.c_int32),
        ("ppc", C.c_int32),
        ("cells", C.c_int64),
    ]


class TgLatticeKey(C.Structure):
    """struct tg_lattice_key (lattice.hpp:16-21)."""

    _fields_ = [
        ("seed", C.c_uint64),
        ("octave", C.c_uint32),
        ("pad", C.c_uint32),
        ("ix", C.c_int64),
        ("iy", C.c_int64),
    ]


P = C.c_void_p
PCFG = C.POINTER(TgFbmConfig)
I32, I64, U64, F64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double

class TgTerrain(C.Structure):
    """tg_terrain: the terrain window of a sharded run."""

    _fields_ = [("x0", C.c_int64), ("width", C.c_int64), ("y_origin", C.c_int64), ("height", C.c_int64),
                ("align", C.c_int32), ("max_lag", C.c_int32)]


class TgBand(C.Structure):
    """tg_band: one rank's rows (global) plus regenerated halo / lookahead."""

    _fields_ = [("y0", C.c_int64), ("rows", C.c_int64), ("halo_top", C.c_int64), ("below", C.c_int64)]


class TgTerrainStats(C.Structure):
    _fields_ = [("sea_level", C.c_double), ("land_fraction", C.c_double), ("land_pixels", C.c_int64),
                ("coast_pixels", C.c_int64), ("n_sizes", C.c_int32), ("n_lags", C.c_int32),
                ("counts", C.c_int64 * 16), ("d_box", C.c_double), ("k_box", C.c_double), ("r2_box", C.c_double),
                ("sum_sq", (C.c_double * 2) * 32), ("pairs", (C.c_int64 * 2) * 32), ("gamma", C.c_double * 32),
                ("hurst", C.c_double), ("d_variogram", C.c_double)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int32, C.c_int32)
OPS_GENERATE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(TgBand))
OPS_HISTOGRAM = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_int32, C.c_int32, C.c_void_p)
OPS_BOXCOUNT = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_double, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                           C.c_void_p)
OPS_VARIOGRAM = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p)


class TgBandOps(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("generate", OPS_GENERATE), ("histogram", OPS_HISTOGRAM),
                ("boxcount", OPS_BOXCOUNT), ("variogram", OPS_VARIOGRAM)]


# name -> (restype, argtypes); every symbol include/polyterrain_b200.h declares.
SIGNATURES = {
    "tg_abi_version": (C.c_int, []),
    "tg_last_error": (C.c_char_p, []),
    "tg_fbm_validate": (C.c_int, [PCFG]),
    "tg_fbm_octave_spec": (C.c_int, [PCFG, I32, C.POINTER(TgOctaveSpec)]),
    "tg_fbm_validate_window": (C.c_int, [PCFG, I64, I64, I64, I64]),
    "tg_device_count": (C.c_int, []),
    "tg_fbm_generate_f32": (C.c_int, [PCFG, I64, I64, I64, P, U64, P]),
    "tg_fbm_generate_rect_f32": (C.c_int, [PCFG, I64, I64, I64, I64, P, I64, P]),
    "tg_fbm_octave_times": (C.c_int, [PCFG, I64, I64, I32, P, P]),
    "tg_fbm_generate_normalized_f64_host": (C.c_int, [PCFG, I64, I64, I32, P, U64, C.POINTER(F64), C.POINTER(F64),
                                                      C.POINTER(I32)]),
    "tg_fbm_generate_batch_f32": (C.c_int, [PCFG, P, I32, I64, I64, I64, I64, P, P]),
    "tg_fbm_generate_f64_host": (C.c_int, [PCFG, I64, I64, I64, P, U64]),
    "tg_fbm_generate_f32_host": (C.c_int, [PCFG, I64, I64, I64, P, U64]),
    "tg_texture_generate_f32": (C.c_int, [PCFG, I32, F64, F64, P, P]),
    "tg_norm_map_f32": (C.c_int, [P, I64, I64, I32, P, P]),
    "tg_fbm3d_generate_f32": (C.c_int, [PCFG, I64, I64, I64, I64, I64, I64, P, P]),
    "tg_lattice_hash": (C.c_int, [P, U64, U64, P, P]),
    "tg_lattice_height_f32": (C.c_int, [P, U64, P, P]),
    "tg_lattice_unit_gradient_f32": (C.c_int, [P, U64, P, P]),
    "tg_minmax_f32": (C.c_int, [P, U64, C.POINTER(F64), C.POINTER(F64), P]),
    "tg_rescale_f32": (C.c_int, [P, U64, F64, F64, P]),
    "tg_pack16_f32": (C.c_int, [P, I64, I64, I64, F64, F64, I32, P, P]),
    "tg_median_f32": (C.c_int, [P, U64, C.POINTER(C.c_float), P]),
    "tg_coastline_mask": (C.c_int, [P, I64, F64, P, C.POINTER(I64), P]),
    "tg_coastline_boxcount": (C.c_int, [P, I64, F64, P, I32, P, C.POINTER(I64), C.POINTER(I64), P]),
    "tg_coastline_boxcount_band": (C.c_int, [P, I64, I64, I64, I32, I32, F64, P, I32, P, C.POINTER(I64),
                                             C.POINTER(I64), P]),
    "tg_boxcount_mask": (C.c_int, [P, I64, P, I32, P, P]),
    "tg_variogram_band_f32": (C.c_int, [P, I64, I64, I64, I64, P, I32, P, P, P]),
    "tg_histogram_f32": (C.c_int, [P, I64, I64, I64, C.c_uint32, C.c_uint32, I32, I32, P, P]),
    "tg_variogram_f32": (C.c_int, [P, I64, I64, I64, P, I32, P, P, P]),
    "tg_measure_ffma_peak": (C.c_int, [C.POINTER(F64), C.POINTER(F64)]),
    "tg_comm_unique_id": (C.c_int, [P]),
    "tg_comm_init_nccl": (C.c_int, [P, I32, I32, C.POINTER(C.c_void_p)]),
    "tg_comm_init_host": (C.c_int, [ALLREDUCE_FN, P, I32, I32, C.POINTER(C.c_void_p)]),
    "tg_comm_allreduce": (C.c_int, [P, P, U64, I32, I32]),
    "tg_comm_destroy": (C.c_int, [P]),
    "tg_plan_band": (C.c_int, [C.POINTER(TgTerrain), I32, I32, C.POINTER(TgBand)]),
    "tg_terrain_stats_band": (C.c_int, [PCFG, C.POINTER(TgTerrain), C.POINTER(TgBand), P, I32, P, I32,
                                        C.POINTER(F64), P, C.POINTER(TgTerrainStats), P]),
    "tg_terrain_stats_band_buf": (C.c_int, [PCFG, C.POINTER(TgTerrain), C.POINTER(TgBand), P, I32, P, I32, P,
                                            I32, C.POINTER(F64), P, C.POINTER(TgTerrainStats), P]),
    "tg_terrain_stats_ops": (C.c_int, [C.POINTER(TgTerrain), C.POINTER(TgBand), P, I32, P, I32, C.POINTER(F64), P,
                                       C.POINTER(TgBandOps), C.POINTER(TgTerrainStats)]),
}

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the CUDA C-ABI library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"polyterrain_b200: CUDA library missing at {path}; run "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().tg_last_error()
    return msg.decode() if msg else ""
