"""ctypes bindings for the CPU checkers — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
``--impl reference``) may import this module.  It exposes:

* ``Oracle`` — oracle/liboracle.so, the plain-C restatement (oracle.c);
* ``Reference`` — oracle/_ref/libtgref.so, the unmodified reference headers
  behind oracle/ref_shim.cpp (absent when /root/reference was never present).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1610_03525_b200._abi import TgFbmConfig, TgLatticeKey, TgOctaveSpec

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtgref.so")

P = C.c_void_p
PCFG = C.POINTER(TgFbmConfig)
I32, I64, U64, F64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double


def build(verbose: bool = False) -> None:
    """Compile oracle.c (and the reference shim where /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if verbose:
        print(out.stdout)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def keys_array(keys) -> np.ndarray:
    """Pack (seed, octave, ix, iy) tuples into a tg_lattice_key numpy array."""
    dt = np.dtype([("seed", "<u8"), ("octave", "<u4"), ("pad", "<u4"), ("ix", "<i8"), ("iy", "<i8")])
    arr = np.zeros(len(keys), dtype=dt)
    for i, (s, o, x, y) in enumerate(keys):
        arr[i] = (s, o, 0, x, y)
    return arr


class Oracle:
    """The C restatement of the reference path (oracle/oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        sig = {
            "or_mix": (U64, [U64]),
            "or_pack": (U64, [U64, C.c_uint32, I64, I64]),
            "or_pack3": (U64, [U64, C.c_uint32, I64, I64, I64]),
            "or_hash": (U64, [U64, C.c_uint32, I64, I64, U64]),
            "or_hash_keys": (None, [P, U64, U64, P]),
            "or_corner_height": (F64, [U64, C.c_uint32, I64, I64]),
            "or_corner_height3": (F64, [U64, C.c_uint32, I64, I64, I64]),
            "or_corner_angle": (F64, [U64, C.c_uint32, I64, I64]),
            "or_corner_gradient": (None, [U64, C.c_uint32, I64, I64, F64, P]),
            "or_corner_unit_gradient": (None, [U64, C.c_uint32, I64, I64, P]),
            "or_smoothstep": (F64, [C.c_int, F64]),
            "or_zg_eval": (F64, [F64, F64, F64, F64, F64, F64, C.c_int, C.c_int]),
            "or_validate": (C.c_int, [PCFG]),
            "or_octave_spec": (C.c_int, [PCFG, C.c_int, C.POINTER(TgOctaveSpec)]),
            "or_generate": (C.c_int, [PCFG, I64, I64, I64, I64, P]),
            "or_sample": (C.c_int, [PCFG, P, P, I64, P]),
            "or_generate3d": (C.c_int, [PCFG, I64, I64, I64, I64, I64, I64, P]),
            "or_generate_mt": (C.c_int, [PCFG, I64, I64, I64, I64, P, I32]),
            "or_sample3d": (C.c_int, [PCFG, P, P, P, I64, P]),
            "or_cell3": (F64, [P, F64, F64, F64, C.c_int]),
            "or_perm_table": (None, [U64, P]),
            "or_perm_gradient": (None, [U64, C.c_uint32, I64, I64, P]),
            "or_normalize": (C.c_int, [P, I64, C.POINTER(F64), C.POINTER(F64), C.POINTER(C.c_int)]),
            "or_upper_median": (F64, [P, I64]),
            "or_coastline_mask": (C.c_int, [P, I64, F64, P, C.POINTER(I64)]),
            "or_box_count": (C.c_int, [P, I64, P, I32, P, C.POINTER(F64), C.POINTER(F64), C.POINTER(F64)]),
            "or_linear_fit": (C.c_int, [P, P, I64, C.POINTER(F64), C.POINTER(F64), C.POINTER(F64)]),
            "or_variogram": (C.c_int, [P, I64, I64, P, I32, P, P]),
            "or_norm_map": (C.c_int, [P, I64, I64, C.c_int, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        self.lib = lib

    def hash_keys(self, keys: np.ndarray, lane: int) -> np.ndarray:
        out = np.zeros(len(keys), dtype=np.uint64)
        self.lib.or_hash_keys(_ptr(keys), len(keys), lane, _ptr(out))
        return out

    def corner_heights(self, keys: np.ndarray) -> np.ndarray:
        return np.array([self.lib.or_corner_height(int(k["seed"]), int(k["octave"]), int(k["ix"]),
                                                   int(k["iy"])) for k in keys])

    def unit_gradients(self, keys: np.ndarray) -> np.ndarray:
        out = np.zeros((len(keys), 2))
        buf = (C.c_double * 2)()
        for i, k in enumerate(keys):
            self.lib.or_corner_unit_gradient(int(k["seed"]), int(k["octave"]), int(k["ix"]),
                                             int(k["iy"]), buf)
            out[i] = buf[0], buf[1]
        return out

    def gradients(self, keys: np.ndarray, w: float) -> np.ndarray:
        out = np.zeros((len(keys), 2))
        buf = (C.c_double * 2)()
        for i, k in enumerate(keys):
            self.lib.or_corner_gradient(int(k["seed"]), int(k["octave"]), int(k["ix"]),
                                        int(k["iy"]), w, buf)
            out[i] = buf[0], buf[1]
        return out

    def validate(self, cfg: TgFbmConfig) -> int:
        return self.lib.or_validate(C.byref(cfg))

    def octave_spec(self, cfg: TgFbmConfig, octave: int) -> TgOctaveSpec:
        os_ = TgOctaveSpec()
        self.lib.or_octave_spec(C.byref(cfg), octave, C.byref(os_))
        return os_

    def generate(self, cfg: TgFbmConfig, ox: int, oy: int, width: int, height: int | None = None):
        height = width if height is None else height
        out = np.zeros((height, width), dtype=np.float64)
        st = self.lib.or_generate(C.byref(cfg), ox, oy, width, height, _ptr(out))
        if st != 0:
            raise ValueError(f"oracle generate: status {st}")
        return out

    def generate_mt(self, cfg: TgFbmConfig, ox: int, oy: int, width: int, height: int | None = None,
                    threads: int | None = None):
        """or_generate over row bands on `threads` host threads (bit-identical)."""
        height = width if height is None else height
        threads = threads or os.cpu_count() or 1
        out = np.empty((height, width), dtype=np.float64)
        st = self.lib.or_generate_mt(C.byref(cfg), ox, oy, width, height, _ptr(out), threads)
        if st != 0:
            raise ValueError(f"oracle generate_mt: status {st}")
        return out

    def sample3d(self, cfg: TgFbmConfig, gx, gy, gz) -> np.ndarray:
        x = np.ascontiguousarray(gx, dtype=np.int64)
        y = np.ascontiguousarray(gy, dtype=np.int64)
        z = np.ascontiguousarray(gz, dtype=np.int64)
        out = np.zeros(len(x))
        st = self.lib.or_sample3d(C.byref(cfg), _ptr(x), _ptr(y), _ptr(z), len(x), _ptr(out))
        if st != 0:
            raise ValueError(f"oracle sample3d: status {st}")
        return out

    def cell3(self, h, x: float, y: float, z: float, order: int) -> float:
        hh = np.ascontiguousarray(h, dtype=np.float64)
        return self.lib.or_cell3(_ptr(hh), x, y, z, order)

    def perm_table(self, seed: int) -> np.ndarray:
        out = np.zeros(256, dtype=np.uint8)
        self.lib.or_perm_table(seed, _ptr(out))
        return out

    def perm_gradient(self, seed: int, octave: int, ix: int, iy: int):
        buf = (C.c_double * 2)()
        self.lib.or_perm_gradient(seed, octave, ix, iy, buf)
        return buf[0], buf[1]

    def sample(self, cfg: TgFbmConfig, gx, gy) -> np.ndarray:
        x = np.ascontiguousarray(gx, dtype=np.int64)
        y = np.ascontiguousarray(gy, dtype=np.int64)
        out = np.zeros(len(x))
        st = self.lib.or_sample(C.byref(cfg), _ptr(x), _ptr(y), len(x), _ptr(out))
        if st != 0:
            raise ValueError(f"oracle sample: status {st}")
        return out

    def generate3d(self, cfg, ox, oy, oz, nx, ny, nz):
        out = np.zeros((nz, ny, nx), dtype=np.float64)
        st = self.lib.or_generate3d(C.byref(cfg), ox, oy, oz, nx, ny, nz, _ptr(out))
        if st != 0:
            raise ValueError(f"oracle generate3d: status {st}")
        return out

    def normalize(self, data: np.ndarray):
        d = np.ascontiguousarray(data, dtype=np.float64).copy()
        lo, hi, const = F64(), F64(), C.c_int()
        self.lib.or_normalize(_ptr(d), d.size, C.byref(lo), C.byref(hi), C.byref(const))
        return d, lo.value, hi.value, bool(const.value)

    def upper_median(self, data: np.ndarray) -> float:
        d = np.ascontiguousarray(data, dtype=np.float64)
        return self.lib.or_upper_median(_ptr(d), d.size)

    def coastline_mask(self, data: np.ndarray, sea: float):
        d = np.ascontiguousarray(data, dtype=np.float64)
        R = d.shape[0]
        mask = np.zeros((R, R), dtype=np.uint8)
        land = I64()
        st = self.lib.or_coastline_mask(_ptr(d), R, sea, _ptr(mask), C.byref(land))
        return st, mask, land.value

    def box_count(self, mask: np.ndarray, sizes):
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        sz = np.asarray(sizes, dtype=np.int32)
        counts = np.zeros(len(sz), dtype=np.int64)
        d, k, r2 = F64(), F64(), F64()
        st = self.lib.or_box_count(_ptr(m), m.shape[0], _ptr(sz), len(sz), _ptr(counts),
                                   C.byref(d), C.byref(k), C.byref(r2))
        return st, counts, d.value, k.value, r2.value

    def linear_fit(self, xs, ys):
        x = np.ascontiguousarray(xs, dtype=np.float64)
        y = np.ascontiguousarray(ys, dtype=np.float64)
        s, i, r = F64(), F64(), F64()
        st = self.lib.or_linear_fit(_ptr(x), _ptr(y), len(x), C.byref(s), C.byref(i), C.byref(r))
        return st, s.value, i.value, r.value

    def norm_map(self, z: np.ndarray, hessian: bool) -> np.ndarray:
        d = np.ascontiguousarray(z, dtype=np.float64)
        out = np.zeros_like(d)
        self.lib.or_norm_map(_ptr(d), d.shape[1], d.shape[0], 1 if hessian else 0, _ptr(out))
        return out

    def variogram(self, z: np.ndarray, lags):
        d = np.ascontiguousarray(z, dtype=np.float64)
        lg = np.asarray(lags, dtype=np.int32)
        ss = np.zeros(2 * len(lg))
        pr = np.zeros(2 * len(lg), dtype=np.int64)
        st = self.lib.or_variogram(_ptr(d), d.shape[1], d.shape[0], _ptr(lg), len(lg), _ptr(ss), _ptr(pr))
        if st != 0:
            raise ValueError("oracle variogram: bad lags")
        return ss.reshape(-1, 2), pr.reshape(-1, 2)


class Reference:
    """The unmodified reference (oracle/_ref/libtgref.so via ref_shim.cpp)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference build missing: {path}")
        lib = C.CDLL(path)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_hash": (U64, [U64, C.c_uint32, I64, I64, U64]),
            "ref_hash_keys": (None, [P, U64, U64, P]),
            "ref_corner_heights": (None, [P, U64, P]),
            "ref_corner_angles": (None, [P, U64, P]),
            "ref_corner_unit_gradients": (None, [P, U64, P]),
            "ref_corner_gradients": (None, [P, U64, F64, P]),
            "ref_validate": (C.c_int, [PCFG]),
            "ref_octave_spec": (C.c_int, [PCFG, C.c_int, C.POINTER(TgOctaveSpec)]),
            "ref_generate_into": (C.c_int, [PCFG, I64, I64, I32, P, U64, C.POINTER(I32)]),
            "ref_generate_region": (C.c_int, [PCFG, I64, I64, I32, P, C.POINTER(F64), C.POINTER(F64),
                                              C.POINTER(I32), C.POINTER(I32), C.c_char_p, I32]),
            "ref_oracle_pixels": (C.c_int, [PCFG, I64, I64, I32, I32, P]),
            "ref_zg_eval": (F64, [F64, F64, F64, F64, F64, F64, C.c_int, C.c_int]),
            "ref_normalize": (C.c_int, [P, I64, C.POINTER(F64), C.POINTER(F64), C.POINTER(I32), C.POINTER(I32)]),
            "ref_coastline_boxcount": (C.c_int, [P, I32, I32, F64, P, I32, P, C.POINTER(F64), C.POINTER(F64),
                                                 C.POINTER(F64), C.POINTER(F64), C.POINTER(F64),
                                                 C.POINTER(I64), P]),
            "ref_box_count_mask": (C.c_int, [P, I32, P, I32, P, C.POINTER(F64), C.POINTER(F64), C.POINTER(F64)]),
            "ref_linear_fit": (C.c_int, [P, P, I32, C.POINTER(F64), C.POINTER(F64), C.POINTER(F64)]),
            "ref_run_bench": (C.c_int, [PCFG, I32, I32, C.POINTER(F64), C.POINTER(F64), C.POINTER(F64)]),
            "ref_encode_pgm16": (I64, [P, I32, I32, P, I64]),
            "ref_texture": (C.c_int, [PCFG, I32, F64, F64, P]),
            "ref_encode_png16": (I64, [P, I32, I32, P, I64]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        self.lib = lib

    def last_error(self) -> str:
        return self.lib.ref_last_error().decode()

    def hash_keys(self, keys: np.ndarray, lane: int) -> np.ndarray:
        out = np.zeros(len(keys), dtype=np.uint64)
        self.lib.ref_hash_keys(_ptr(keys), len(keys), lane, _ptr(out))
        return out

    def corner_heights(self, keys: np.ndarray) -> np.ndarray:
        out = np.zeros(len(keys))
        self.lib.ref_corner_heights(_ptr(keys), len(keys), _ptr(out))
        return out

    def corner_angles(self, keys: np.ndarray) -> np.ndarray:
        out = np.zeros(len(keys))
        self.lib.ref_corner_angles(_ptr(keys), len(keys), _ptr(out))
        return out

    def unit_gradients(self, keys: np.ndarray) -> np.ndarray:
        out = np.zeros((len(keys), 2))
        self.lib.ref_corner_unit_gradients(_ptr(keys), len(keys), _ptr(out))
        return out

    def gradients(self, keys: np.ndarray, w: float) -> np.ndarray:
        out = np.zeros((len(keys), 2))
        self.lib.ref_corner_gradients(_ptr(keys), len(keys), w, _ptr(out))
        return out

    def validate(self, cfg) -> int:
        return self.lib.ref_validate(C.byref(cfg))

    def octave_spec(self, cfg, octave: int) -> TgOctaveSpec:
        os_ = TgOctaveSpec()
        self.lib.ref_octave_spec(C.byref(cfg), octave, C.byref(os_))
        return os_

    def generate_into(self, cfg, ox: int, oy: int, extent: int, n_out: int | None = None):
        n = extent * extent if n_out is None else n_out
        out = np.full(max(n, 1), 123.0)
        nw = I32()
        st = self.lib.ref_generate_into(C.byref(cfg), ox, oy, extent, _ptr(out), n, C.byref(nw))
        if st != 0:
            return st, None, 0
        return st, out[: extent * extent].reshape(extent, extent), nw.value

    def generate_region(self, cfg, ox: int, oy: int, extent: int):
        out = np.zeros((extent, extent))
        lo, hi, nz, cs = F64(), F64(), I32(), I32()
        buf = C.create_string_buffer(4096)
        st = self.lib.ref_generate_region(C.byref(cfg), ox, oy, extent, _ptr(out), C.byref(lo),
                                          C.byref(hi), C.byref(nz), C.byref(cs), buf, 4096)
        if st != 0:
            raise ValueError(f"reference generate_region: {self.last_error()}")
        warnings = [w for w in buf.value.decode().split("\n") if w]
        return out, dict(source_min=lo.value, source_max=hi.value, normalized=bool(nz.value),
                         constant_source=bool(cs.value), warnings=warnings)

    def oracle_pixels(self, cfg, ox: int, oy: int, width: int, height: int | None = None):
        height = width if height is None else height
        out = np.zeros((height, width))
        self.lib.ref_oracle_pixels(C.byref(cfg), ox, oy, width, height, _ptr(out))
        return out

    def coastline_boxcount(self, data: np.ndarray, sizes, sea: float | None = None, want_mask=False):
        d = np.ascontiguousarray(data, dtype=np.float64)
        R = d.shape[0]
        sz = np.asarray(sizes, dtype=np.int32)
        counts = np.zeros(max(len(sz), 1), dtype=np.int64)
        dd, kk, r2, lf, so = F64(), F64(), F64(), F64(), F64()
        cp = I64()
        mask = np.zeros((R, R), dtype=np.uint8) if want_mask else None
        st = self.lib.ref_coastline_boxcount(_ptr(d), R, 1 if sea is None else 0, 0.0 if sea is None else sea,
                                             _ptr(sz), len(sz), _ptr(counts), C.byref(dd), C.byref(kk),
                                             C.byref(r2), C.byref(lf), C.byref(so), C.byref(cp),
                                             _ptr(mask) if want_mask else None)
        return dict(status=st, counts=counts[: len(sz)], d=dd.value, k=kk.value, r2=r2.value,
                    land_fraction=lf.value, sea=so.value, coast_pixels=cp.value, mask=mask)

    def box_count_mask(self, mask: np.ndarray, sizes):
        m = np.ascontiguousarray(mask, dtype=np.uint8)
        sz = np.asarray(sizes, dtype=np.int32)
        counts = np.zeros(len(sz), dtype=np.int64)
        d, k, r2 = F64(), F64(), F64()
        st = self.lib.ref_box_count_mask(_ptr(m), m.shape[0], _ptr(sz), len(sz), _ptr(counts),
                                         C.byref(d), C.byref(k), C.byref(r2))
        return st, counts, d.value, k.value, r2.value

    def texture(self, cfg, kind: int, gain: float, pattern_frequency: float) -> np.ndarray:
        R = cfg.resolution
        out = np.zeros((R, R))
        st = self.lib.ref_texture(C.byref(cfg), kind, gain, pattern_frequency, _ptr(out))
        if st != 0:
            raise ValueError(self.last_error())
        return out

    def encode16(self, data: np.ndarray, png: bool) -> bytes:
        d = np.ascontiguousarray(data, dtype=np.float64)
        h, w = d.shape
        cap = 2 * d.size + h + 4096
        buf = np.zeros(cap, dtype=np.uint8)
        fn = self.lib.ref_encode_png16 if png else self.lib.ref_encode_pgm16
        n = fn(_ptr(d), w, h, _ptr(buf), cap)
        if n < 0:
            raise ValueError(self.last_error())
        return buf[:n].tobytes()

    def run_bench(self, cfg, reps: int, warmup: int):
        med, mn, mean = F64(), F64(), F64()
        st = self.lib.ref_run_bench(C.byref(cfg), reps, warmup, C.byref(med), C.byref(mn), C.byref(mean))
        if st != 0:
            raise ValueError(f"reference run_bench: {self.last_error()}")
        return med.value, mn.value, mean.value
