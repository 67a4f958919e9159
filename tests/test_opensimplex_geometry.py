"""The geometric property the GPU OpenSimplex kernel's fp32 lattice selection
rests on (csrc/simplex2d.cu region_case): the four vertices the 2014 region
logic picks include EVERY lattice vertex with 2 - |d|^2 > 0.  So the sum is
the sum over all positive-attenuation vertices, and a pixel within eps of a
region or cell boundary that an fp32 decision puts on the other side only
swaps in/out a vertex whose attenuation is O(eps) there — a change of
O(eps^4) in the value, not a different lattice.

CPU test (numpy), restating oracle/oracle.c or_opensimplex's region logic.
"""
import numpy as np

STRETCH = -0.211324865405187117745425609749
SQUISH = 0.366025403784438646763723170753


def _chosen(x, y):
    """The oracle's four vertices (stretched lattice coordinates) per point."""
    so = (x + y) * STRETCH
    xs, ys = x + so, y + so
    xb, yb = np.floor(xs), np.floor(ys)
    xi, yi = xs - xb, ys - yb
    s = xi + yi
    up = s > 1.0
    z = np.where(up, 2.0 - s, 1.0 - s)
    edge = np.where(up, (z < xi) | (z < yi), (z > xi) | (z > yi))
    xgt = xi > yi
    ea = np.where(up, np.where(edge, np.where(xgt, 2, 0), 0), np.where(edge, np.where(xgt, 1, -1), 1))
    eb = np.where(up, np.where(edge, np.where(xgt, 0, 2), 0), np.where(edge, np.where(xgt, -1, 1), 1))
    c = up.astype(np.int64)
    verts = [(np.ones_like(c), np.zeros_like(c)), (np.zeros_like(c), np.ones_like(c)), (c, c), (ea, eb)]
    return xb, yb, verts


def _uncovered_positive(x, y):
    xb, yb, verts = _chosen(x, y)
    worst = 0.0
    for a in range(-2, 4):
        for b in range(-2, 4):
            vx, vy = xb + a, yb + b
            sq = (vx + vy) * SQUISH
            dx, dy = x - (vx + sq), y - (vy + sq)
            attn = 2.0 - dx * dx - dy * dy
            chosen = np.zeros(x.shape, dtype=bool)
            for (va, vb) in verts:
                chosen |= (va == a) & (vb == b)
            bad = (attn > 0) & ~chosen
            if bad.any():
                worst = max(worst, float(attn[bad].max()))
    return worst


def test_chosen_vertices_cover_every_positive_attenuation():
    rng = np.random.default_rng(5)
    x = rng.uniform(-300.0, 300.0, 400_000)
    y = rng.uniform(-300.0, 300.0, 400_000)
    assert _uncovered_positive(x, y) == 0.0


def test_points_on_region_boundaries():
    """Points placed on (and 1e-9 around) every boundary of the region logic:
    cell edges, the rhombus diagonal, the edge/interior lines and x = y."""
    rng = np.random.default_rng(6)
    n = 20_000
    t = rng.uniform(0.0, 1.0, n)
    cells = rng.integers(-1000, 1000, (n, 2)).astype(np.float64)
    # boundaries in the unit stretched cell: xi = 0, yi = 0, s = 1, 2xi + yi = 1 / 2,
    # xi + 2yi = 1 / 2, xi = yi
    lines = [(np.zeros(n), t), (t, np.zeros(n)), (t, 1 - t), (t / 2, 1 - t), (0.5 + t / 2, 1 - t),
             (1 - t, t / 2), (1 - t, 0.5 + t / 2), (t, t)]
    for xi, yi in lines:
        for eps in (0.0, 1e-9, -1e-9):
            xs = cells[:, 0] + xi + eps
            ys = cells[:, 1] + yi - eps
            # invert the stretch: x = xs + (xs + ys) * SQUISH
            sq = (xs + ys) * SQUISH
            assert _uncovered_positive(xs + sq, ys + sq) == 0.0
