"""Python mirror of the reference generator API over the C-ABI.

Mirrors terrain::fbm (fbm.hpp:27-107, 538-685) and the analysis pass
(analysis.hpp:29-346) with the same names, argument meaning and error
behaviour (ValidationError / NumericalError / IoError, errors.hpp:9-36).
Device buffers are torch CUDA tensors (plumbing only); every compute call
goes through libpolyterrain_b200.so — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi


class ValidationError(ValueError):
    """terrain::ValidationError (errors.hpp:9-12)."""


class NumericalError(ArithmeticError):
    """terrain::NumericalError (errors.hpp:27-30)."""


class IoError(OSError):
    """terrain::IoError (errors.hpp:33-36)."""


class DeviceError(RuntimeError):
    """CUDA failure (std::runtime_error in the reference's terms)."""


def _check(status: int) -> None:
    if status == _abi.TG_OK:
        return
    msg = _abi.last_error()
    if status == _abi.TG_EVALIDATION:
        raise ValidationError(msg)
    if status == _abi.TG_ENUMERICAL:
        raise NumericalError(msg)
    if status == _abi.TG_EIO:
        raise IoError(msg)
    raise DeviceError(msg)


class Method(enum.IntEnum):
    """terrain::fbm::Method (fbm.hpp:27)."""

    zg_paper = 0
    zg_separable = 1
    generic = 2
    perlin3 = 3
    perlin5 = 4
    opensimplex = 5  # B200 extension: the paper's third baseline (parity unpinned)
    perlin_perm = 6  # B200 extension: permutation-table Perlin (BASELINE config 3; parity unpinned)


def method_name(m: Method) -> str:  # fbm.hpp:29-38
    return Method(m).name


def parse_method(name: str) -> Optional[Method]:  # fbm.hpp:40-47
    return {"zg_paper": Method.zg_paper, "zg": Method.zg_paper,
            "zg_separable": Method.zg_separable, "generic": Method.generic,
            "perlin3": Method.perlin3, "perlin": Method.perlin3,
            "perlin5": Method.perlin5, "opensimplex": Method.opensimplex,
            "perlin_perm": Method.perlin_perm}.get(name)


@dataclass
class FbmConfig:
    """terrain::fbm::FbmConfig (fbm.hpp:49-89) plus `smoothstep` (SURVEY D2:
    0 = reference default, or 3 / 5 for any method) and `zero_lattice`
    (the ZeroSource hook, fbm.hpp:125-133)."""

    seed: int = 0
    method: Method = Method.zg_paper
    octaves: int = 1
    resolution: int = 256
    base_frequency: int = 2
    frequency_ratio: float = 2.0
    persistence: float = 0.5
    base_amplitude: float = 1.0
    gradient_weight: Optional[float] = None
    normalize: bool = False
    threads: int = 1
    smoothstep: int = 0
    zero_lattice: bool = False

    def gradient_weight_value(self) -> float:  # fbm.hpp:62-64
        return self.gradient_weight if self.gradient_weight is not None else self.base_amplitude / 100.0

    def smoothstep_order(self) -> int:  # fbm.hpp:66-69 (+ explicit override)
        if self.smoothstep:
            return self.smoothstep
        return 5 if self.method in (Method.perlin5, Method.perlin_perm) else 3

    def to_c(self) -> _abi.TgFbmConfig:
        c = _abi.TgFbmConfig()
        c.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        c.method = int(self.method)
        c.smoothstep = int(self.smoothstep)
        c.octaves = int(self.octaves)
        c.threads = int(self.threads)
        c.resolution = int(self.resolution)
        c.base_frequency = int(self.base_frequency)
        c.frequency_ratio = float(self.frequency_ratio)
        c.persistence = float(self.persistence)
        c.base_amplitude = float(self.base_amplitude)
        c.has_gradient_weight = 0 if self.gradient_weight is None else 1
        c.gradient_weight = 0.0 if self.gradient_weight is None else float(self.gradient_weight)
        c.normalize = 1 if self.normalize else 0
        c.zero_lattice = 1 if self.zero_lattice else 0
        return c

    def validate(self) -> None:  # fbm.hpp:71-88
        _check(_abi.load().tg_fbm_validate(C.byref(self.to_c())))


@dataclass
class OctaveSpec:
    freq: float
    amp: float
    fast: bool
    cells: int
    ppc: int


def octave_spec(cfg: FbmConfig, octave: int) -> OctaveSpec:  # fbm.hpp:151-168
    s = _abi.TgOctaveSpec()
    _check(_abi.load().tg_fbm_octave_spec(C.byref(cfg.to_c()), octave, C.byref(s)))
    return OctaveSpec(s.freq, s.amp, bool(s.fast), s.cells, s.ppc)


@dataclass
class Heightmap:
    """terrain::fbm::Heightmap (fbm.hpp:91-107); data is row-major, at(x, y) = data[y, x]."""

    resolution: int = 0
    data: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))
    config: FbmConfig = field(default_factory=FbmConfig)
    origin: tuple = (0, 0)
    octave_seconds: List[float] = field(default_factory=list)
    source_min: float = 0.0
    source_max: float = 0.0
    normalized: bool = False
    constant_source: bool = False
    warnings: List[str] = field(default_factory=list)

    def at(self, x: int, y: int) -> float:
        return float(self.data[y, x])


def _warnings(cfg: FbmConfig) -> List[str]:
    out = []
    for o in range(cfg.octaves):  # fbm.hpp:566-569 (std::to_string(double) = "%f")
        s = octave_spec(cfg, o)
        if s.freq > float(cfg.resolution):
            out.append(f"octave {o}: cell size below one pixel (frequency {s.freq:f} exceeds resolution)")
    return out


def _stream_ptr(stream) -> int:
    import torch

    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _check_device_out(out, need: int) -> None:
    """`out` must be a contiguous CUDA float32 tensor of at least `need`
    elements (else ValidationError, never an out-of-bounds device write)."""
    import torch

    if not (isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == torch.float32
            and out.is_contiguous()):
        raise ValidationError("generate: output must be a contiguous CUDA float32 tensor")
    if out.numel() < need:
        raise ValidationError("generate: output buffer size mismatch")


def generate_into_device(cfg: FbmConfig, origin, extent: int, out, stream=None) -> None:
    """Device form of generate_into (fbm.hpp:541-628): `out` is a CUDA fp32
    tensor of extent^2 elements, written stream-ordered (no host sync)."""
    _check_device_out(out, int(extent) * int(extent))
    _check(_abi.load().tg_fbm_generate_f32(C.byref(cfg.to_c()), int(origin[0]), int(origin[1]),
                                            int(extent), out.data_ptr(), out.numel(),
                                            _stream_ptr(stream)))


def generate_rect_device(cfg: FbmConfig, origin, width: int, height: int, out, ld: Optional[int] = None,
                         stream=None) -> None:
    """Rectangular window with row pitch `ld` (chunks and row bands)."""
    ld = width if ld is None else ld
    if width < 1 or height < 1 or ld < width:
        raise ValidationError("generate: bad window shape or row pitch")
    _check_device_out(out, (int(height) - 1) * int(ld) + int(width))
    _check(_abi.load().tg_fbm_generate_rect_f32(C.byref(cfg.to_c()), int(origin[0]), int(origin[1]),
                                                 int(width), int(height), out.data_ptr(), int(ld),
                                                 _stream_ptr(stream)))


def generate_batch_device(cfg: FbmConfig, seeds: Sequence[int], origin, width: int, height: int, out,
                          stream=None) -> None:
    """Maps differing only in seed, one launch per 64 seeds."""
    if width < 1 or height < 1:
        raise ValidationError("generate: bad window shape")
    _check_device_out(out, len(seeds) * int(width) * int(height))
    arr = (C.c_uint64 * len(seeds))(*[int(s) & 0xFFFFFFFFFFFFFFFF for s in seeds])
    _check(_abi.load().tg_fbm_generate_batch_f32(C.byref(cfg.to_c()), arr, len(seeds), int(origin[0]),
                                                  int(origin[1]), int(width), int(height),
                                                  out.data_ptr(), _stream_ptr(stream)))


def generate_into(cfg: FbmConfig, origin, extent: int, out: np.ndarray,
                  octave_seconds: Optional[list] = None, warnings: Optional[list] = None) -> None:
    """Drop-in for generate_into(cfg, origin, extent, std::span<double> out)
    (fbm.hpp:630-634): host float64 (or float32) buffer of extent^2, overwritten."""
    cfg.validate()
    if extent < 1 or extent > _abi.TG_MAX_EXTENT:  # fbm.hpp:547-550
        raise ValidationError("generate: extent must be in [1, 131072]")
    if out.size != extent * extent:
        raise ValidationError("generate: output buffer size mismatch")
    if not out.flags["C_CONTIGUOUS"]:
        raise ValidationError("generate: output buffer must be contiguous")
    t0 = time.perf_counter()
    lib = _abi.load()
    if out.dtype == np.float64:
        st = lib.tg_fbm_generate_f64_host(C.byref(cfg.to_c()), int(origin[0]), int(origin[1]), int(extent),
                                          out.ctypes.data, out.size)
    elif out.dtype == np.float32:
        st = lib.tg_fbm_generate_f32_host(C.byref(cfg.to_c()), int(origin[0]), int(origin[1]), int(extent),
                                          out.ctypes.data, out.size)
    else:
        raise ValidationError("generate: output buffer must be float64 or float32")
    _check(st)
    dt = time.perf_counter() - t0
    if warnings is not None:
        warnings.extend(_warnings(cfg))
    if octave_seconds is not None:
        # The fused kernel renders every octave in one pass: octave k's time is
        # the device-time increment between diagnostic launches of the octave
        # prefixes 0..k (tg_fbm_octave_times), one entry per octave as the
        # reference's contract requires (fbm.hpp:564,624-626).
        t = (C.c_double * cfg.octaves)()
        _check(lib.tg_fbm_octave_times(C.byref(cfg.to_c()), int(origin[0]), int(origin[1]), int(extent), t, None))
        octave_seconds.extend(list(t))


def normalize_map(hm: Heightmap) -> Heightmap:
    """normalize_map (fbm.hpp:638-656) on a host Heightmap (exact fp64 rescale)."""
    import copy

    out = copy.copy(hm)
    if hm.data.size == 0:
        return out
    lo, hi = float(hm.data.min()), float(hm.data.max())
    out.source_min, out.source_max = lo, hi
    if lo == hi:
        out.constant_source = True
        return out
    out.data = -1.0 + 2.0 * (hm.data - lo) / (hi - lo)
    out.normalized = True
    return out


def generate_region(cfg: FbmConfig, origin, extent: int) -> Heightmap:
    """generate_region (fbm.hpp:658-685)."""
    hm = Heightmap(resolution=extent, config=cfg, origin=tuple(origin))
    cfg.validate()
    if extent < 1 or extent > _abi.TG_MAX_EXTENT:
        raise ValidationError("generate: extent must be in [1, 131072]")
    hm.data = np.empty((extent, extent), dtype=np.float64)
    if not cfg.normalize:
        generate_into(cfg, origin, extent, hm.data, hm.octave_seconds, hm.warnings)
        return hm
    # normalize_map fused on the device (the same doubles as the host form)
    lib = _abi.load()
    c = cfg.to_c()
    lo, hi, const = C.c_double(), C.c_double(), C.c_int32()
    _check(lib.tg_fbm_generate_normalized_f64_host(C.byref(c), int(origin[0]), int(origin[1]), int(extent),
                                                   hm.data.ctypes.data, hm.data.size, C.byref(lo), C.byref(hi),
                                                   C.byref(const)))
    hm.source_min, hm.source_max = lo.value, hi.value
    hm.constant_source, hm.normalized = bool(const.value), not const.value
    t = (C.c_double * cfg.octaves)()
    _check(lib.tg_fbm_octave_times(C.byref(c), int(origin[0]), int(origin[1]), int(extent), t, None))
    hm.octave_seconds.extend(list(t))
    hm.warnings.extend(_warnings(cfg))
    return hm


def generate_heightmap(cfg: FbmConfig) -> Heightmap:  # fbm.hpp:672-680
    cfg.validate()
    return generate_region(cfg, (0, 0), cfg.resolution)


# ---- analysis (analysis.hpp) ---------------------------------------------------


@dataclass
class LinearFit:
    slope: float = 0.0
    intercept: float = 0.0
    r2: float = 1.0


def linear_fit(xs, ys) -> LinearFit:
    """OLS (analysis.hpp:29-63), host-side (a handful of points)."""
    xs = [float(v) for v in xs]
    ys = [float(v) for v in ys]
    if len(xs) != len(ys):
        raise ValidationError("linear_fit: mismatched series lengths")
    n = len(xs)
    if n < 2:
        raise ValidationError("linear_fit: need at least two points")
    mx = sum(xs) / n
    my = sum(ys) / n
    sxx = sum((x - mx) * (x - mx) for x in xs)
    sxy = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    syy = sum((y - my) * (y - my) for y in ys)
    if sxx == 0.0:
        raise ValidationError("linear_fit: x values are all equal")
    slope = sxy / sxx
    icept = my - slope * mx
    if syy == 0.0:
        return LinearFit(slope, icept, 1.0)
    ssr = sum((y - (slope * x + icept)) ** 2 for x, y in zip(xs, ys))
    return LinearFit(slope, icept, 1.0 - ssr / syy)


def default_box_sizes() -> List[int]:  # analysis.hpp:261
    return [2, 4, 8, 16, 32, 64]


@dataclass
class BoxCountReport:
    sizes: List[int] = field(default_factory=list)
    counts: List[int] = field(default_factory=list)
    lengths: List[float] = field(default_factory=list)
    d: float = 0.0
    k: float = 0.0
    r2: float = 0.0
    sea_level: float = 0.0
    land_fraction: float = 0.0
    coast_pixels: int = 0


def upper_median_device(dev_map, stream=None) -> float:
    """nth_element upper median (analysis.hpp:244-250) by device radix select."""
    out = C.c_float()
    _check(_abi.load().tg_median_f32(dev_map.data_ptr(), dev_map.numel(), C.byref(out), _stream_ptr(stream)))
    return float(out.value)


def coastline_mask_device(dev_map, resolution: int, sea_level: Optional[float] = None, stream=None):
    """coastline_mask (analysis.hpp:213-250) -> (uint8 CUDA mask, sea, land_fraction)."""
    import torch

    if sea_level is None:
        sea_level = upper_median_device(dev_map, stream)
    mask = torch.empty((resolution, resolution), dtype=torch.uint8, device=dev_map.device)
    land = C.c_int64()
    _check(_abi.load().tg_coastline_mask(dev_map.data_ptr(), resolution, float(sea_level), mask.data_ptr(),
                                         C.byref(land), _stream_ptr(stream)))
    return mask, sea_level, land.value / float(resolution * resolution)


def _fit_report(sizes, counts) -> BoxCountReport:
    rep = BoxCountReport(sizes=list(sizes), counts=[int(c) for c in counts])
    rep.lengths = [float(c) * float(s) for s, c in zip(sizes, counts)]
    fit = linear_fit([math.log(float(s)) for s in sizes], [math.log(float(c)) for c in counts])
    rep.d, rep.k, rep.r2 = -fit.slope, math.exp(fit.intercept), fit.r2  # analysis.hpp:300-304
    return rep


def box_count_device(dev_map, resolution: int, sizes: Optional[Sequence[int]] = None,
                     sea_level: Optional[float] = None, stream=None) -> BoxCountReport:
    """Fused coastline + box count (analysis.hpp:213-305) on a device map."""
    sizes = default_box_sizes() if sizes is None else list(sizes)
    if sea_level is None:
        sea_level = upper_median_device(dev_map, stream)
    arr = (C.c_int32 * len(sizes))(*sizes)
    counts = (C.c_int64 * len(sizes))()
    coast, land = C.c_int64(), C.c_int64()
    _check(_abi.load().tg_coastline_boxcount(dev_map.data_ptr(), resolution, float(sea_level), arr, len(sizes),
                                             counts, C.byref(coast), C.byref(land), _stream_ptr(stream)))
    rep = _fit_report(sizes, list(counts))
    rep.sea_level = float(sea_level)
    rep.land_fraction = land.value / float(resolution * resolution)
    rep.coast_pixels = coast.value
    return rep


def box_count_mask_device(dev_mask, resolution: int, sizes: Sequence[int], stream=None) -> BoxCountReport:
    """box_count on an explicit uint8 CUDA mask (analysis.hpp:269-305)."""
    arr = (C.c_int32 * len(sizes))(*sizes)
    counts = (C.c_int64 * len(sizes))()
    _check(_abi.load().tg_boxcount_mask(dev_mask.data_ptr(), resolution, arr, len(sizes), counts,
                                        _stream_ptr(stream)))
    return _fit_report(sizes, list(counts))


def variogram_device(dev_map, width: int, height: int, lags: Sequence[int], ld: Optional[int] = None,
                     stream=None):
    """Height-difference variogram (new): returns (sum_sq[n,2], pairs[n,2])."""
    ld = width if ld is None else ld
    arr = (C.c_int32 * len(lags))(*lags)
    ss = (C.c_double * (2 * len(lags)))()
    pr = (C.c_int64 * (2 * len(lags)))()
    _check(_abi.load().tg_variogram_f32(dev_map.data_ptr(), width, height, ld, arr, len(lags), ss, pr,
                                        _stream_ptr(stream)))
    return np.array(ss[:]).reshape(-1, 2), np.array(pr[:], dtype=np.int64).reshape(-1, 2)


def variogram_dimension(sum_sq, pairs, lags) -> tuple:
    """gamma(h) = sum / (2 pairs); gamma ~ h^(2H), D = 3 - H for a surface."""
    gam = np.asarray(sum_sq).sum(axis=1) / (2.0 * np.asarray(pairs).sum(axis=1))
    fit = linear_fit([math.log(h) for h in lags], [math.log(g) for g in gam])
    hurst = fit.slope / 2.0
    return gam, hurst, 3.0 - hurst, fit.r2


def _pack16(dev_map, width: int, height: int, png: bool):
    import torch

    lo, hi = C.c_double(), C.c_double()
    _check(_abi.load().tg_minmax_f32(dev_map.data_ptr(), width * height, C.byref(lo), C.byref(hi),
                                     _stream_ptr(None)))
    nbytes = height * (2 * width + (1 if png else 0))
    out = torch.empty(nbytes, dtype=torch.uint8, device=dev_map.device)
    _check(_abi.load().tg_pack16_f32(dev_map.data_ptr(), width, height, width, lo.value, hi.value,
                                     1 if png else 0, out.data_ptr(), _stream_ptr(None)))
    return out.cpu().numpy().tobytes(), lo.value, hi.value


def encode_pgm16(dev_map, width: int, height: int) -> bytes:
    """write_pgm16 (io.hpp:91-106) of a contiguous CUDA fp32 map: range and
    quantize16 on the device, header on the host."""
    body, lo, hi = _pack16(dev_map, width, height, False)
    return f"P5\n# hmin={lo:.17g} hmax={hi:.17g}\n{width} {height}\n65535\n".encode() + body


def encode_png16(dev_map, width: int, height: int) -> bytes:
    """write_png16 (io.hpp:203-250): device-packed raw rows, zlib level 9."""
    import struct
    import zlib

    raw, lo, hi = _pack16(dev_map, width, height, True)

    def chunk(t: bytes, data: bytes) -> bytes:
        return struct.pack(">I", len(data)) + t + data + struct.pack(">I", zlib.crc32(t + data) & 0xFFFFFFFF)

    ihdr = struct.pack(">II", width, height) + bytes([16, 0, 0, 0, 0])
    text = b"Comment\0" + f"hmin={lo:.17g} hmax={hi:.17g}".encode()
    return (bytes([137, 80, 78, 71, 13, 10, 26, 10]) + chunk(b"IHDR", ihdr) + chunk(b"tEXt", text)
            + chunk(b"IDAT", zlib.compress(raw, 9)) + chunk(b"IEND", b""))


def write_pgm16(path: str, dev_map, width: int, height: int) -> None:
    with open(path, "wb") as f:
        f.write(encode_pgm16(dev_map, width, height))


def write_png16(path: str, dev_map, width: int, height: int) -> None:
    with open(path, "wb") as f:
        f.write(encode_png16(dev_map, width, height))


class TextureKind(enum.IntEnum):
    """terrain::texture::Kind (texture.hpp:19)."""

    marble = 0
    wood = 1
    cloud = 2


def texture_device(cfg: FbmConfig, kind: TextureKind, out, gain: float = 1.0, pattern_frequency: float = 4.0,
                   stream=None) -> None:
    """texture::render (texture.hpp:50-72) of the full map into a CUDA fp32
    tensor; marble/wood are fused into the generation store."""
    _check(_abi.load().tg_texture_generate_f32(C.byref(cfg.to_c()), int(kind), float(gain),
                                               float(pattern_frequency), out.data_ptr(), _stream_ptr(stream)))


def norm_map_device(dev_map, width: int, height: int, out, hessian: bool = False, stream=None) -> None:
    """gradient_norm_map / hessian_norm_map (terrain_cli.cpp:148-182) on the device."""
    _check(_abi.load().tg_norm_map_f32(dev_map.data_ptr(), width, height, 1 if hessian else 0, out.data_ptr(),
                                       _stream_ptr(stream)))


def generate3d_device(cfg: FbmConfig, origin, shape, out, stream=None) -> None:
    """3D fBm volume (new): out is a CUDA fp32 tensor [nz, ny, nx]."""
    nz, ny, nx = shape
    if nx < 1 or ny < 1 or nz < 1:
        raise ValidationError("generate3d: bad volume shape")
    _check_device_out(out, int(nx) * int(ny) * int(nz))
    _check(_abi.load().tg_fbm3d_generate_f32(C.byref(cfg.to_c()), int(origin[0]), int(origin[1]), int(origin[2]),
                                             nx, ny, nz, out.data_ptr(), _stream_ptr(stream)))


def ffma_peak_tflops() -> float:
    t, ms = C.c_double(), C.c_double()
    _check(_abi.load().tg_measure_ffma_peak(C.byref(t), C.byref(ms)))
    return t.value
