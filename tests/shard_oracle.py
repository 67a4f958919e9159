"""CPU backend for paper_1610_03525_b200.shard — TEST INFRASTRUCTURE.

Same interface as shard.DeviceBackend, computed with the oracle restatement
(oracle/oracle.c) and numpy on fp32-rounded values, so the multi-rank
sharding and all-reduce logic is exercised with gloo on CPU."""
import numpy as np

from oracle.pyoracle import Oracle


def fkey(v: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(v, dtype=np.float32).view(np.uint32)
    return np.where(b & 0x80000000, ~b, b | 0x80000000).astype(np.uint32)


class OracleBackend:
    def __init__(self, ccfg):
        self.c = ccfg
        self.o = Oracle()

    def generate(self, band):
        self.band = band
        ys, xs = np.meshgrid(np.arange(band.gen_y0, band.gen_y0 + band.gen_rows),
                             np.arange(band.x0, band.x0 + band.width), indexing="ij")
        v = self.o.sample(self.c, xs.ravel(), ys.ravel()).reshape(band.gen_rows, band.width)
        self.win = v.astype(np.float32)

    def owned(self):
        b = self.band
        return self.win[b.halo_top:b.halo_top + b.rows]

    def histogram(self, prefix, mask, shift, bits):
        k = fkey(self.owned().ravel())
        sel = k[(k & np.uint32(mask)) == np.uint32(prefix)]
        return np.bincount(((sel >> np.uint32(shift)) & np.uint32((1 << bits) - 1)).astype(np.int64),
                           minlength=1 << bits)

    def boxcount(self, sea, sizes):
        b = self.band
        land = self.win.astype(np.float64) >= sea
        r0 = b.halo_top
        own = land[r0:r0 + b.rows]
        up = np.ones_like(own)
        dn = np.ones_like(own)
        up[1:] = own[:-1]
        if b.halo_top:
            up[0] = land[r0 - 1]
        dn[:-1] = own[1:]
        if not b.is_last:
            dn[-1] = land[r0 + b.rows]
        lf = np.ones_like(own)
        rt = np.ones_like(own)
        lf[:, 1:] = own[:, :-1]
        rt[:, :-1] = own[:, 1:]
        coast = own & ~(up & dn & lf & rt)
        counts = []
        for e in sizes:
            by = (np.arange(b.rows) // e)[:, None]
            bx = (np.arange(b.width) // e)[None, :]
            ids = (by * ((b.width + e - 1) // e) + bx)[coast]
            counts.append(len(np.unique(ids)))
        return counts, int(coast.sum()), int(own.sum())

    def variogram(self, lags):
        b = self.band
        z = self.win[b.halo_top:].astype(np.float64)  # owned rows + lookahead
        ss = np.zeros((len(lags), 2))
        pr = np.zeros((len(lags), 2), dtype=np.int64)
        for i, h in enumerate(lags):
            a = z[:b.rows]
            if h < b.width:
                d = a[:, h:] - a[:, :-h]
                ss[i, 0], pr[i, 0] = (d * d).sum(), d.size
            ny = min(b.rows, z.shape[0] - h)
            if ny > 0:
                d = z[h:h + ny] - z[:ny]
                ss[i, 1], pr[i, 1] = (d * d).sum(), d.size
        return ss, pr
