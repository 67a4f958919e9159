"""Multi-GPU terrain: row-band shards, no data-path collective.

A thin Python face over the C-ABI (include/polyterrain_b200.h, csrc/terrain.cpp):

* :func:`plan_band` -> ``tg_plan_band`` (contiguous row bands whose starts are
  multiples of ``align``; a 1-row halo above and ``max_lag`` lookahead rows
  below each band are REGENERATED locally, never exchanged — option (i) of
  SURVEY §8e);
* :class:`Comm` -> ``tg_comm``: NCCL over NVLink (``tg_comm_init_nccl``, the
  unique id broadcast once through torch.distributed), or a host all-reduce
  hook over ``torch.distributed`` (gloo in the CPU tests);
* :func:`terrain_stats` -> ``tg_terrain_stats_band`` (device band, the
  product) or ``tg_terrain_stats_ops`` (caller-supplied band operations: the
  test hook that runs the same C++ driver over the CPU oracle).

Only statistics cross GPUs: the radix-select histograms of the global upper
median sea level (analysis.hpp:244-250), box counts (boxes anchored at band
starts that are multiples of every box size, so per-band counts add up),
land / coast pixel counts, and the variogram sums and pair counts.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _abi
from .fbm import FbmConfig, _check


@dataclass
class Band:
    """One rank's shard of a width x height terrain window at (x0, y_origin)."""

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
    align: int = 1

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

    def c_terrain(self) -> _abi.TgTerrain:
        return _abi.TgTerrain(self.x0, self.width, self.y_origin, self.height, self.align, self.max_lag)

    def c_band(self) -> _abi.TgBand:
        return _abi.TgBand(self.y0, self.rows, self.halo_top, self.below)


def plan_band(width: int, height: int, world: int, rank: int, align: int = 64, max_lag: int = 0,
              x0: int = 0, y_origin: int = 0) -> Band:
    """Split `height` rows into `world` contiguous bands whose starts are
    multiples of `align` (octave-0 cell size and every box size must divide
    it).  Bands differ by at most `align` rows (tg_plan_band)."""
    t = _abi.TgTerrain(x0, width, y_origin, height, align, max_lag)
    b = _abi.TgBand()
    _check(_abi.load().tg_plan_band(C.byref(t), world, rank, C.byref(b)))
    return Band(rank, world, x0, width, b.y0, b.rows, height, b.halo_top, b.below, y_origin, max_lag, align)


class Comm:
    """A ``tg_comm``: the statistics all-reduce of one process group.

    ``Comm()`` reduces host buffers through ``torch.distributed`` when it is
    initialised (any backend), and is a no-op for a single process.
    ``Comm.nccl(device)`` builds the native NCCL communicator (libnccl over
    NVLink): rank 0's unique id is broadcast once through torch.distributed.
    """

    def __init__(self, group=None, device=None):
        self._setup(group, device)
        self._cb = _abi.ALLREDUCE_FN(self._allreduce_cb)
        h = C.c_void_p()
        _check(_abi.load().tg_comm_init_host(self._cb, None, self.world, self.rank, C.byref(h)))
        self.handle = h

    def _setup(self, group, device):
        import torch.distributed as dist

        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.device = device
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.handle = None

    @classmethod
    def nccl(cls, device=None, group=None) -> "Comm":
        import torch

        self = cls.__new__(cls)
        self._setup(group, device)
        self._cb = None
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            _check(_abi.load().tg_comm_unique_id(uid))
        if self.dist:
            on_gpu = self.dist.get_backend(group) == "nccl"
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
            if on_gpu:
                t = t.to(device or torch.device("cuda", torch.cuda.current_device()))
            self.dist.broadcast(t, src=0, group=group)
            uid = (C.c_uint8 * 128)(*t.cpu().tolist())
        h = C.c_void_p()
        _check(_abi.load().tg_comm_init_nccl(uid, self.world, self.rank, C.byref(h)))
        self.handle = h
        return self

    def _allreduce_cb(self, ctx, buf, count, dtype, op) -> int:
        try:
            import torch

            arr = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_int64 if dtype == 0 else C.c_double)),
                                        shape=(count,))
            t = torch.from_numpy(arr.copy())
            if self.dist.get_backend(self.group) == "nccl":
                t = t.to(self.device or torch.device("cuda", torch.cuda.current_device()))
            red = self.dist.ReduceOp.SUM if op == 0 else self.dist.ReduceOp.MAX
            self.dist.all_reduce(t, op=red, group=self.group)
            arr[:] = t.cpu().numpy()
            return 0
        except Exception:  # pragma: no cover - surfaces as TG_EDEVICE from the driver
            return 1

    def allreduce(self, arr: np.ndarray, op: str = "sum") -> np.ndarray:
        a = np.ascontiguousarray(arr).copy()
        if a.dtype.kind in "iu":
            a, dt = a.astype(np.int64), 0
        else:
            a, dt = a.astype(np.float64), 1
        _check(_abi.load().tg_comm_allreduce(self.handle, a.ctypes.data, a.size, dt, 0 if op == "sum" else 1))
        return a

    def close(self) -> None:
        if getattr(self, "handle", None):
            _abi.load().tg_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def float_from_key(k: int) -> float:
    """Inverse of the order-preserving fp32 key used by the device kernels."""
    b = (k & 0x7FFFFFFF) if k & 0x80000000 else (~k & 0xFFFFFFFF)
    return float(np.array([b], dtype=np.uint32).view(np.float32)[0])


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


def _stats_from_c(st: _abi.TgTerrainStats, sizes, lags) -> TerrainStats:
    n, m = len(sizes), len(lags)
    ss = np.array([[st.sum_sq[i][0], st.sum_sq[i][1]] for i in range(m)])
    pr = np.array([[st.pairs[i][0], st.pairs[i][1]] for i in range(m)], dtype=np.int64)
    return TerrainStats(st.sea_level, st.land_fraction, st.coast_pixels, list(sizes),
                        [st.counts[i] for i in range(n)], st.d_box, st.r2_box, list(lags), ss, pr,
                        np.array(st.gamma[:m]), st.hurst, st.d_variogram)


def terrain_stats(band: Band, backend, comm: Comm, sizes: Sequence[int], lags: Sequence[int],
                  sea_level: Optional[float] = None) -> TerrainStats:
    """Generate this rank's band (+ regenerated halo / lookahead rows) and
    reduce the fractal statistics of the whole terrain across ranks — the
    C++ driver of csrc/terrain.cpp, on the device (DeviceBackend) or over a
    caller's band operations (test backends)."""
    lib = _abi.load()
    t, b = band.c_terrain(), band.c_band()
    sz = (C.c_int32 * len(sizes))(*sizes)
    lg = (C.c_int32 * len(lags))(*lags)
    sea = C.byref(C.c_double(sea_level)) if sea_level is not None else None
    st = _abi.TgTerrainStats()
    if isinstance(backend, DeviceBackend) and backend.buffer is not None:
        buf = backend.buffer
        if buf.numel() < band.gen_rows * band.width or not buf.is_contiguous() or buf.device.type != "cuda":
            raise ValueError("terrain_stats: band buffer must be a contiguous CUDA tensor of gen_rows x width")
        _check(lib.tg_terrain_stats_band_buf(C.byref(backend.ccfg), C.byref(t), C.byref(b), buf.data_ptr(),
                                             1 if backend.owned_ready else 0, sz, len(sizes), lg, len(lags), sea,
                                             comm.handle, C.byref(st), backend._sp()))
    elif isinstance(backend, DeviceBackend):
        _check(lib.tg_terrain_stats_band(C.byref(backend.ccfg), C.byref(t), C.byref(b), sz, len(sizes), lg,
                                         len(lags), sea, comm.handle, C.byref(st), backend._sp()))
    else:
        ops = _ops_for(backend, band)
        _check(lib.tg_terrain_stats_ops(C.byref(t), C.byref(b), sz, len(sizes), lg, len(lags), sea, comm.handle,
                                        C.byref(ops), C.byref(st)))
    return _stats_from_c(st, sizes, lags)


def _ops_for(backend, band: Band) -> _abi.TgBandOps:
    """tg_band_ops over a Python backend with the generate / histogram /
    boxcount / variogram method set (tests/shard_oracle.py)."""

    def generate(ctx, b):
        try:
            backend.generate(band)
            return 0
        except Exception:
            return _abi.TG_EDEVICE

    def histogram(ctx, prefix, mask, shift, bits, out):
        h = np.ascontiguousarray(backend.histogram(prefix, mask, shift, bits), dtype=np.uint64)
        C.memmove(out, h.ctypes.data, h.nbytes)
        return 0

    def boxcount(ctx, sea, sizes_p, n, counts_p, coast_p, land_p):
        sizes = np.ctypeslib.as_array(C.cast(sizes_p, C.POINTER(C.c_int32)), shape=(n,)).tolist()
        counts, coast, land = backend.boxcount(sea, sizes)
        np.ctypeslib.as_array(C.cast(counts_p, C.POINTER(C.c_int64)), shape=(n,))[:] = counts
        C.cast(coast_p, C.POINTER(C.c_int64))[0] = int(coast)
        C.cast(land_p, C.POINTER(C.c_int64))[0] = int(land)
        return 0

    def variogram(ctx, lags_p, n, ss_p, pr_p):
        lags = np.ctypeslib.as_array(C.cast(lags_p, C.POINTER(C.c_int32)), shape=(n,)).tolist()
        ss, pr = backend.variogram(lags)
        np.ctypeslib.as_array(C.cast(ss_p, C.POINTER(C.c_double)), shape=(2 * n,))[:] = np.asarray(ss).ravel()
        np.ctypeslib.as_array(C.cast(pr_p, C.POINTER(C.c_int64)), shape=(2 * n,))[:] = np.asarray(pr).ravel()
        return 0

    ops = _abi.TgBandOps(None, _abi.OPS_GENERATE(generate), _abi.OPS_HISTOGRAM(histogram),
                         _abi.OPS_BOXCOUNT(boxcount), _abi.OPS_VARIOGRAM(variogram))
    ops._keep = (generate, histogram, boxcount, variogram)
    return ops


def distributed_upper_median(hist_fn, total: int, comm: Comm) -> float:
    """Upper median (element total//2 of the sorted union, analysis.hpp:247)
    by a 3-pass radix select whose per-rank histograms are all-reduced (the
    digits of tg_terrain_stats_band; used for whole-map batches)."""
    prefix, mask, k = 0, 0, total // 2
    for shift, bits in ((21, 11), (10, 11), (0, 10)):
        h = comm.allreduce(np.asarray(hist_fn(prefix, mask, shift, bits), dtype=np.int64))
        c = np.cumsum(h)
        b = int(np.searchsorted(c, k, side="right"))
        k -= int(c[b - 1]) if b > 0 else 0
        prefix |= b << shift
        mask |= ((1 << bits) - 1) << shift
    return float_from_key(prefix)


class DeviceBackend:
    """The product backend: the band generated and analysed on this rank's GPU
    inside tg_terrain_stats_band — or, with `buffer` (a float32 CUDA tensor of
    gen_rows x width whose owned rows the caller has generated when
    `owned_ready`), tg_terrain_stats_band_buf, which regenerates only the halo
    and lookahead rows."""

    def __init__(self, cfg: FbmConfig, device=None, stream=None, buffer=None, owned_ready: bool = False):
        import torch

        self.cfg = cfg
        self.ccfg = cfg.to_c()
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.stream = stream
        self.buffer = buffer
        self.owned_ready = owned_ready

    def _sp(self) -> int:
        import torch

        s = self.stream or torch.cuda.current_stream(self.device)
        return int(s.cuda_stream)
