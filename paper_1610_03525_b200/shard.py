"""Multi-GPU terrain: row-band shards, no data-path collective.

Every sample is a pure function of (config, global pixel) (fbm.hpp:7-8), so a
large terrain splits into contiguous row bands, one per rank, generated with
no exchange at all.  The analysis pass needs neighbours across band edges;
they are REGENERATED locally instead of exchanged:

* a 1-row halo above/below each band for the 4-neighbour coastline test
  (analysis.hpp:228-229);
* `max_lag` lookahead rows below the band for the vertical variogram pairs
  (option (i) of SURVEY §8e).

Only statistics cross GPUs, through ``torch.distributed`` all-reduce (NCCL
over NVLink on the GPU box, gloo in the CPU tests): the radix-select
histograms of the global upper-median sea level (analysis.hpp:244-250), the
box counts (boxes anchored at band starts that are multiples of every box
size, so per-band counts add up), land/coast pixel counts, and the variogram
sums and pair counts.

The compute is a pluggable backend so the sharding and reduction logic runs
on CPU in the tests; :class:`DeviceBackend` is the product (C-ABI kernels).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _abi
from .fbm import FbmConfig, ValidationError, _check, linear_fit


@dataclass
class Band:
    """One rank's shard of a width x height terrain window at (x0, y0)."""

    rank: int
    world: int
    x0: int
    width: int
    y0: int          # first owned row (global)
    rows: int        # owned rows
    height: int      # whole terrain height (rows)
    halo_top: int    # regenerated rows above (0 or 1)
    below: int       # regenerated rows below: max(halo, lookahead), clipped to the terrain
    y_origin: int = 0  # global row of the terrain's first row (y0 - y_origin is band-local)
    max_lag: int = 0   # lookahead the band was planned for (vertical variogram lags)

    @property
    def local_y0(self) -> int:
        return self.y0 - self.y_origin

    @property
    def is_last(self) -> bool:
        return self.local_y0 + self.rows >= self.height

    @property
    def gen_y0(self) -> int:
        return self.y0 - self.halo_top

    @property
    def gen_rows(self) -> int:
        return self.halo_top + self.rows + self.below


def plan_band(width: int, height: int, world: int, rank: int, align: int = 64, max_lag: int = 0,
              x0: int = 0, y_origin: int = 0) -> Band:
    """Split `height` rows into `world` contiguous bands whose starts are
    multiples of `align` (octave-0 cell size and every box size must divide
    it).  Bands differ by at most `align` rows."""
    if world < 1 or not (0 <= rank < world):
        raise ValidationError("plan_band: bad rank/world")
    if height % align != 0:
        raise ValidationError("plan_band: height must be a multiple of the alignment")
    units = height // align
    if units < world:
        raise ValidationError("plan_band: fewer aligned row blocks than ranks")
    u0 = units * rank // world
    u1 = units * (rank + 1) // world
    y0, y1 = u0 * align, u1 * align
    halo_top = 1 if y0 > 0 else 0
    below = min(max(1, max_lag), height - y1)
    return Band(rank, world, x0, width, y_origin + y0, y1 - y0, height, halo_top, below, y_origin, max_lag)


class Comm:
    """Sum/max all-reduce of small host arrays over torch.distributed."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist

        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.device = device

    def allreduce(self, arr: np.ndarray, op: str = "sum") -> np.ndarray:
        if self.dist is None:
            return arr
        import torch

        t = torch.from_numpy(np.ascontiguousarray(arr).copy())
        if self.device is not None:
            t = t.to(self.device)
        red = self.dist.ReduceOp.SUM if op == "sum" else self.dist.ReduceOp.MAX
        self.dist.all_reduce(t, op=red, group=self.group)
        return t.cpu().numpy()


def float_from_key(k: int) -> float:
    """Inverse of the order-preserving fp32 key used by the device kernels."""
    b = (k & 0x7FFFFFFF) if k & 0x80000000 else (~k & 0xFFFFFFFF)
    return float(np.array([b], dtype=np.uint32).view(np.float32)[0])


def distributed_upper_median(hist_fn, total: int, comm: Comm) -> float:
    """Upper median (element total//2 of the sorted union, analysis.hpp:247)
    by a 3-pass radix select whose per-rank histograms are all-reduced."""
    prefix, mask, k = 0, 0, total // 2
    for shift, bits in ((21, 11), (10, 11), (0, 10)):
        h = comm.allreduce(np.asarray(hist_fn(prefix, mask, shift, bits), dtype=np.int64))
        c = np.cumsum(h)
        b = int(np.searchsorted(c, k, side="right"))
        k -= int(c[b - 1]) if b > 0 else 0
        prefix |= b << shift
        mask |= ((1 << bits) - 1) << shift
    return float_from_key(prefix)


@dataclass
class TerrainStats:
    sea_level: float
    land_fraction: float
    coast_pixels: int
    sizes: list
    counts: list
    d_box: float
    r2_box: float
    lags: list
    sum_sq: np.ndarray
    pairs: np.ndarray
    gamma: np.ndarray
    hurst: float
    d_variogram: float


def terrain_stats(band: Band, backend, comm: Comm, sizes: Sequence[int], lags: Sequence[int],
                  sea_level: Optional[float] = None) -> TerrainStats:
    """Generate this rank's band (+ regenerated halo/lookahead rows) and
    reduce the fractal statistics of the whole terrain across ranks."""
    for s in sizes:
        if band.local_y0 % s != 0 or (band.rows % s != 0 and not band.is_last):
            raise ValidationError("terrain_stats: band starts/ends must be multiples of every box size")
    # vertical pairs need max(lags) rows below the band, or every row left in the terrain
    if lags and max(lags) > band.below and band.below < band.height - (band.local_y0 + band.rows):
        raise ValidationError("terrain_stats: a variogram lag exceeds the band's regenerated lookahead "
                              "(plan_band max_lag)")
    backend.generate(band)
    total = band.width * band.height
    if sea_level is None:
        sea_level = distributed_upper_median(backend.histogram, total, comm)
    counts, coast, land = backend.boxcount(sea_level, list(sizes))
    red = comm.allreduce(np.array(list(counts) + [coast, land], dtype=np.int64))
    counts, coast, land = [int(v) for v in red[:-2]], int(red[-2]), int(red[-1])
    if land == 0 or land == total:
        raise ValidationError("coastline_mask: map is entirely land or entirely water")
    ss, pr = backend.variogram(list(lags))
    ss = comm.allreduce(np.asarray(ss, dtype=np.float64))
    pr = comm.allreduce(np.asarray(pr, dtype=np.int64))
    fit = linear_fit([math.log(s) for s in sizes], [math.log(c) for c in counts])
    gam = ss.sum(axis=1) / (2.0 * pr.sum(axis=1))
    ok = gam > 0
    vf = linear_fit([math.log(h) for h, g in zip(lags, ok) if g], [math.log(v) for v in gam[ok]]) \
        if ok.sum() >= 2 else None
    hurst = vf.slope / 2.0 if vf else float("nan")
    return TerrainStats(sea_level, land / total, coast, list(sizes), counts, -fit.slope, fit.r2, list(lags),
                        ss, pr, gam, hurst, 3.0 - hurst)


class DeviceBackend:
    """The product backend: C-ABI kernels on this rank's GPU."""

    def __init__(self, cfg: FbmConfig, device=None, stream=None):
        import torch

        self.cfg = cfg
        self.ccfg = cfg.to_c()
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.stream = stream
        self.buf = None
        self.band = None

    def _sp(self) -> int:
        import torch

        s = self.stream or torch.cuda.current_stream(self.device)
        return int(s.cuda_stream)

    def generate(self, band: Band) -> None:
        import torch

        self.band = band
        n = band.gen_rows * band.width
        if self.buf is None or self.buf.numel() < n:
            self.buf = torch.empty(n, dtype=torch.float32, device=self.device)
        _check(_abi.load().tg_fbm_generate_rect_f32(C.byref(self.ccfg), band.x0, band.gen_y0, band.width,
                                                    band.gen_rows, self.buf.data_ptr(), band.width, self._sp()))

    def _owned_ptr(self) -> int:
        return self.buf.data_ptr() + 4 * self.band.halo_top * self.band.width

    def histogram(self, prefix: int, mask: int, shift: int, bits: int) -> np.ndarray:
        out = np.zeros(1 << bits, dtype=np.uint64)
        _check(_abi.load().tg_histogram_f32(self._owned_ptr(), self.band.width, self.band.rows, self.band.width,
                                            prefix, mask, shift, bits, out.ctypes.data, self._sp()))
        return out.astype(np.int64)

    def boxcount(self, sea: float, sizes: list):
        b = self.band
        arr = (C.c_int32 * len(sizes))(*sizes)
        cnt = (C.c_int64 * len(sizes))()
        coast, land = C.c_int64(), C.c_int64()
        has_bot = 0 if b.is_last else 1
        _check(_abi.load().tg_coastline_boxcount_band(self._owned_ptr(), b.width, b.rows, b.width, b.halo_top,
                                                      has_bot, float(sea), arr, len(sizes), cnt,
                                                      C.byref(coast), C.byref(land), self._sp()))
        return list(cnt), coast.value, land.value

    def variogram(self, lags: list):
        b = self.band
        arr = (C.c_int32 * len(lags))(*lags)
        ss = (C.c_double * (2 * len(lags)))()
        pr = (C.c_int64 * (2 * len(lags)))()
        _check(_abi.load().tg_variogram_band_f32(self._owned_ptr(), b.width, b.rows + b.below, b.width, b.rows,
                                                 arr, len(lags), ss, pr, self._sp()))
        return np.array(ss[:]).reshape(-1, 2), np.array(pr[:], dtype=np.int64).reshape(-1, 2)
