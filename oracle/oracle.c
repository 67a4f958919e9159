/*
 * oracle.c — plain-C restatement of the reference fBm path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Parity pinned against the
 * compiled reference (oracle/_ref/libtgref.so) by tests/test_oracle_golden.py
 * and the fixtures in tests/golden/.  The 3D kernel and the variogram have no
 * reference ("parity unpinned"): they are checked by properties only.
 *
 * Citations are into /root/reference/proj/include/terrain/.
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction, like the reference's
 * x86-64 -O3 build which has no FMA instructions), see oracle/Makefile.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define C_SEED 0x9E3779B97F4A7C15ULL
#define C_OCT 0xBF58476D1CE4E5B9ULL
#define C_IX 0x94D049BB133111EBULL
#define C_IY 0xD6E8FEB86659FD93ULL

/* lattice.hpp:35-42 — murmur3 fmix64 */
uint64_t or_mix(uint64_t z) {
    z ^= z >> 33;
    z *= 0xFF51AFD7ED558CCDULL;
    z ^= z >> 33;
    z *= 0xC4CEB9FE1A85EC53ULL;
    z ^= z >> 33;
    return z;
}

/* lattice.hpp:46-50 — signed ix/iy wrap two's-complement into u64 */
uint64_t or_pack(uint64_t seed, uint32_t octave, int64_t ix, int64_t iy) {
    return seed * C_SEED + (uint64_t)octave * C_OCT + (uint64_t)ix * C_IX + (uint64_t)iy * C_IY;
}

/* 3D extension (new): iz = 0 reproduces the 2D key. */
uint64_t or_pack3(uint64_t seed, uint32_t octave, int64_t ix, int64_t iy, int64_t iz) {
    return or_pack(seed, octave, ix, iy) + (uint64_t)iz * TG_PACK_K5;
}

uint64_t or_hash(uint64_t seed, uint32_t octave, int64_t ix, int64_t iy, uint64_t lane) {
    return or_mix(or_pack(seed, octave, ix, iy) ^ lane);
}

void or_hash_keys(const tg_lattice_key* keys, uint64_t n, uint64_t lane, uint64_t* out) {
    for (uint64_t i = 0; i < n; ++i)
        out[i] = or_hash(keys[i].seed, keys[i].octave, keys[i].ix, keys[i].iy, lane);
}

/* lattice.hpp:56-58 */
static double to_unit(uint64_t z) { return (double)(z >> 11) * 0x1.0p-53; }

/* lattice.hpp:62-64 */
double or_corner_height(uint64_t seed, uint32_t octave, int64_t ix, int64_t iy) {
    return to_unit(or_mix(or_pack(seed, octave, ix, iy))) * 2.0 - 1.0;
}

double or_corner_height3(uint64_t seed, uint32_t octave, int64_t ix, int64_t iy, int64_t iz) {
    return to_unit(or_mix(or_pack3(seed, octave, ix, iy, iz))) * 2.0 - 1.0;
}

/* lattice.hpp:66-69 (std::numbers::pi) */
double or_corner_angle(uint64_t seed, uint32_t octave, int64_t ix, int64_t iy) {
    return to_unit(or_mix(or_pack(seed, octave, ix, iy) ^ TG_LANE_ANGLE)) * 2.0 *
           3.141592653589793238462643383279502884;
}

/* lattice.hpp:72-77 */
void or_corner_gradient(uint64_t seed, uint32_t octave, int64_t ix, int64_t iy, double w,
                        double out[2]) {
    const double angle = or_corner_angle(seed, octave, ix, iy);
    const double magnitude = to_unit(or_mix(or_pack(seed, octave, ix, iy) ^ TG_LANE_MAGNITUDE)) * w;
    out[0] = magnitude * cos(angle);
    out[1] = magnitude * sin(angle);
}

/* lattice.hpp:80-83 */
void or_corner_unit_gradient(uint64_t seed, uint32_t octave, int64_t ix, int64_t iy,
                             double out[2]) {
    const double angle = or_corner_angle(seed, octave, ix, iy);
    out[0] = cos(angle);
    out[1] = sin(angle);
}

/* kernels2d.hpp:26-38 */
double or_smoothstep(int order, double t) {
    if (order == 5) return t * t * t * (10.0 + t * (6.0 * t - 15.0));
    return t * t * (3.0 - 2.0 * t);
}

/* kernels2d.hpp:62-76: zg_params then zg_eval (cross term 66-68) */
double or_zg_eval(double h00, double h10, double h01, double h11, double x, double y,
                  int separable, int order) {
    const double dx = h10 - h00, dy = h01 - h00, a = h11 + h00 - h10 - h01;
    const double sx = or_smoothstep(order, x), sy = or_smoothstep(order, y);
    const double cross = separable ? sx * sy : sx * y + sy * x - x * y;
    return h00 + sx * dx + sy * dy + a * cross;
}

/* kernels2d.hpp:103-122; corners = {h,f,g} x (00, 10, 01, 11); c[i*4+j] on x^i y^j */
void or_generic_coeffs(const double k[12], double c[16]) {
    const double h00 = k[0], f00 = k[1], g00 = k[2];
    const double h10 = k[3], f10 = k[4], g10 = k[5];
    const double h01 = k[6], f01 = k[7], g01 = k[8];
    const double h11 = k[9], f11 = k[10], g11 = k[11];
    memset(c, 0, 16 * sizeof(double));
#define AT(i, j) c[(i) * 4 + (j)]
    AT(0, 0) = h00;
    AT(1, 0) = f00;
    AT(0, 1) = g00;
    AT(2, 0) = 3.0 * (h10 - h00) - 2.0 * f00 - f10;
    AT(3, 0) = f10 + f00 - 2.0 * (h10 - h00);
    AT(0, 2) = 3.0 * (h01 - h00) - 2.0 * g00 - g01;
    AT(0, 3) = g01 + g00 - 2.0 * (h01 - h00);
    AT(2, 1) = 3.0 * (h11 - h01) - 2.0 * f01 - f11 - AT(2, 0);
    AT(3, 1) = f11 + f01 - 2.0 * (h11 - h01) - AT(3, 0);
    AT(1, 2) = 3.0 * (h11 - h10) - 2.0 * g10 - g11 - AT(0, 2);
    AT(1, 3) = g11 + g10 - 2.0 * (h11 - h10) - AT(0, 3);
    AT(1, 1) = h01 + h10 - h00 - h11 + f01 + g10 - g00 - f00;
#undef AT
}

/* kernels2d.hpp:124-134 — Horner in y per x-power, then in x */
double or_generic_eval(const double c[16], double x, double y) {
    double acc = 0.0;
    for (int i = 3; i >= 0; --i) {
        double row = c[i * 4 + 3];
        row = row * y + c[i * 4 + 2];
        row = row * y + c[i * 4 + 1];
        row = row * y + c[i * 4 + 0];
        acc = acc * x + row;
    }
    return acc;
}

/* kernels2d.hpp:163-173 */
double or_perlin_eval(const double f[4], const double g[4], int order, double x, double y) {
    const double sx = or_smoothstep(order, x), sy = or_smoothstep(order, y);
    const double v00 = f[0] * x + g[0] * y;
    const double v10 = f[1] * (x - 1.0) + g[1] * y;
    const double v01 = f[2] * x + g[2] * (y - 1.0);
    const double v11 = f[3] * (x - 1.0) + g[3] * (y - 1.0);
    const double h0 = v00 + sx * (v10 - v00);
    const double h1 = v01 + sx * (v11 - v01);
    return h0 + sy * (h1 - h0);
}

/* OpenSimplex 2D (new, parity unpinned): the 2014 OpenSimplex
 * geometry restated from its published description — stretch the input onto
 * a skewed square lattice, locate the rhombus and its triangle, sum
 * (2 - d^2)^4 * (g . d) over the two fixed vertices, the closest corner and
 * one extra vertex, divide by 47.  Gradients: the 8 vectors (+-5, +-2),
 * (+-2, +-5), chosen by the lattice hash (lane TG_LANE_SIMPLEX). */
#define OS_STRETCH (-0.211324865405187117745425609749)
#define OS_SQUISH 0.366025403784438646763723170753
static const double OS_GRAD[16] = {5, 2, 2, 5, -5, 2, -2, 5, 5, -2, 2, -5, -5, -2, -2, -5};

static double os_contrib(uint64_t seed, uint32_t oct, int64_t xsv, int64_t ysv, double dx, double dy) {
    double attn = 2.0 - dx * dx - dy * dy;
    if (attn <= 0.0) return 0.0;
    const int gi = (int)(or_hash(seed, oct, xsv, ysv, TG_LANE_SIMPLEX) >> 61) * 2;
    attn *= attn;
    return attn * attn * (OS_GRAD[gi] * dx + OS_GRAD[gi + 1] * dy);
}

double or_opensimplex(uint64_t seed, uint32_t oct, double x, double y) {
    const double so = (x + y) * OS_STRETCH;
    const double xs = x + so, ys = y + so;
    int64_t xsb = (int64_t)floor(xs), ysb = (int64_t)floor(ys);
    const double sq = (double)(xsb + ysb) * OS_SQUISH;
    const double xins = xs - (double)xsb, yins = ys - (double)ysb;
    const double in_sum = xins + yins;
    double dx0 = x - ((double)xsb + sq), dy0 = y - ((double)ysb + sq);
    double v = 0.0;
    /* the two vertices (1,0) and (0,1) of the rhombus */
    v += os_contrib(seed, oct, xsb + 1, ysb, dx0 - 1.0 - OS_SQUISH, dy0 - OS_SQUISH);
    v += os_contrib(seed, oct, xsb, ysb + 1, dx0 - OS_SQUISH, dy0 - 1.0 - OS_SQUISH);
    int64_t xe, ye;
    double dxe, dye;
    if (in_sum <= 1.0) { /* triangle (0,0), (1,0), (0,1) */
        const double zins = 1.0 - in_sum;
        if (zins > xins || zins > yins) {
            if (xins > yins) {
                xe = xsb + 1; ye = ysb - 1; dxe = dx0 - 1.0; dye = dy0 + 1.0;
            } else {
                xe = xsb - 1; ye = ysb + 1; dxe = dx0 + 1.0; dye = dy0 - 1.0;
            }
        } else {
            xe = xsb + 1; ye = ysb + 1; dxe = dx0 - 1.0 - 2.0 * OS_SQUISH; dye = dy0 - 1.0 - 2.0 * OS_SQUISH;
        }
    } else { /* triangle (1,0), (0,1), (1,1) */
        const double zins = 2.0 - in_sum;
        if (zins < xins || zins < yins) {
            if (xins > yins) {
                xe = xsb + 2; ye = ysb; dxe = dx0 - 2.0 - 2.0 * OS_SQUISH; dye = dy0 - 2.0 * OS_SQUISH;
            } else {
                xe = xsb; ye = ysb + 2; dxe = dx0 - 2.0 * OS_SQUISH; dye = dy0 - 2.0 - 2.0 * OS_SQUISH;
            }
        } else {
            xe = xsb; ye = ysb; dxe = dx0; dye = dy0;
        }
        xsb += 1;
        ysb += 1;
        dx0 = dx0 - 1.0 - 2.0 * OS_SQUISH;
        dy0 = dy0 - 1.0 - 2.0 * OS_SQUISH;
    }
    v += os_contrib(seed, oct, xsb, ysb, dx0, dy0); /* (0,0) or (1,1) */
    v += os_contrib(seed, oct, xe, ye, dxe, dye);   /* extra vertex */
    return v / 47.0;
}

/* FbmConfig::validate (fbm.hpp:71-88) with the lifted caps. */
int or_validate(const tg_fbm_config* c) {
    if (c->octaves < 1 || c->octaves > TG_MAX_OCTAVES) return TG_EVALIDATION;
    if (c->resolution < 1 || c->resolution > TG_MAX_RESOLUTION) return TG_EVALIDATION;
    if (c->base_frequency < 1 || c->base_frequency > TG_MAX_RESOLUTION) return TG_EVALIDATION;
    if (!(c->frequency_ratio > 1.0) || !isfinite(c->frequency_ratio)) return TG_EVALIDATION;
    if (!(c->persistence > 0.0 && c->persistence <= 1.0)) return TG_EVALIDATION;
    if (!(c->base_amplitude > 0.0) || !isfinite(c->base_amplitude)) return TG_EVALIDATION;
    if (c->has_gradient_weight && (!(c->gradient_weight >= 0.0) || !isfinite(c->gradient_weight)))
        return TG_EVALIDATION;
    if (c->threads < 0 || c->threads > 256) return TG_EVALIDATION;
    if (c->method < 0 || c->method > TG_METHOD_PERLIN_PERM) return TG_EVALIDATION;
    if (c->smoothstep != 0 && c->smoothstep != 3 && c->smoothstep != 5) return TG_EVALIDATION;
    return TG_OK;
}

static int order_of(const tg_fbm_config* c) {
    if (c->smoothstep) return c->smoothstep;
    return c->method == TG_METHOD_PERLIN5 || c->method == TG_METHOD_PERLIN_PERM ? 5 : 3; /* fbm.hpp:66-69 */
}

static double weight_of(const tg_fbm_config* c) {
    return c->has_gradient_weight ? c->gradient_weight : c->base_amplitude / 100.0; /* 62-64 */
}

/* fbm.hpp:151-168 — repeated multiplication, fast iff integer cells dividing R */
int or_octave_spec(const tg_fbm_config* c, int octave, tg_octave_spec* os) {
    os->freq = (double)c->base_frequency;
    os->amp = c->base_amplitude;
    for (int k = 0; k < octave; ++k) {
        os->freq *= c->frequency_ratio;
        os->amp *= c->persistence;
    }
    os->fast = 0;
    os->cells = 0;
    os->ppc = 0;
    const double rounded = floor(os->freq);
    if (rounded == os->freq && rounded >= 1.0 && rounded <= (double)c->resolution &&
        c->resolution % (long long)rounded == 0) {
        os->fast = 1;
        os->cells = (long long)rounded;
        os->ppc = (int32_t)(c->resolution / os->cells);
    }
    return TG_OK;
}

/* fbm.hpp:137-141 */
static int64_t floor_div(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

typedef struct {
    double h, f, g;
} corner_t;

/* Permutation-table Perlin (TG_METHOD_PERLIN_PERM, new; definition in
 * include/polyterrain_b200.h): P sorts the 256 keys mix(s ^ i*KI ^ lane). */
void or_perm_table(uint64_t seed, uint8_t out[256]) {
    const uint64_t s = seed * 0x9E3779B97F4A7C15ULL;
    uint64_t key[256];
    for (int i = 0; i < 256; ++i) key[i] = or_mix(s ^ ((uint64_t)i * TG_PERM_KI) ^ TG_LANE_PERM);
    for (int i = 0; i < 256; ++i) {
        int rank = 0;
        for (int j = 0; j < 256; ++j) rank += key[j] < key[i] || (key[j] == key[i] && j < i);
        out[rank] = (uint8_t)i;
    }
}

static _Thread_local uint64_t perm_seed_cached;
static _Thread_local int perm_cached;
static _Thread_local uint8_t perm_tab[256];

void or_perm_gradient(uint64_t seed, uint32_t oct, int64_t ix, int64_t iy, double out[2]) {
    static const double R = 0.70710678118654752440;
    static const double G[8][2] = {{1, 0}, {R, R}, {0, 1}, {-R, R}, {-1, 0}, {-R, -R}, {0, -1}, {R, -R}};
    if (!perm_cached || perm_seed_cached != seed) {
        or_perm_table(seed, perm_tab);
        perm_seed_cached = seed;
        perm_cached = 1;
    }
    const uint64_t s = seed * 0x9E3779B97F4A7C15ULL;
    const uint64_t t = or_mix((s + (uint64_t)oct * 0xBF58476D1CE4E5B9ULL) ^ TG_LANE_PERM);
    const int64_t ox = (int64_t)(t & 255), oy = (int64_t)((t >> 8) & 255);
    const int a = perm_tab[(ix + ox) & 255];
    const int k = perm_tab[(a + iy + oy) & 255] & 7;
    out[0] = G[k][0];
    out[1] = G[k][1];
}

static corner_t corner_data(const tg_fbm_config* c, int oct, double amp, int64_t ix, int64_t iy,
                            int need_h, int need_grad, int need_unit) {
    corner_t k = {0.0, 0.0, 0.0};
    if (c->zero_lattice) return k; /* ZeroSource, fbm.hpp:125-133 */
    if (need_h) k.h = amp * or_corner_height(c->seed, (uint32_t)oct, ix, iy);
    if (need_grad) {
        double g[2];
        or_corner_gradient(c->seed, (uint32_t)oct, ix, iy, weight_of(c), g);
        k.f = g[0];
        k.g = g[1];
    }
    if (need_unit) {
        double g[2];
        if (c->method == TG_METHOD_PERLIN_PERM)
            or_perm_gradient(c->seed, (uint32_t)oct, ix, iy, g);
        else
            or_corner_unit_gradient(c->seed, (uint32_t)oct, ix, iy, g);
        k.f = amp * g[0];
        k.g = amp * g[1];
    }
    return k;
}

/* One sample of one octave on the fast path: the LUT expressions of
 * kernels2d.hpp:214-239 (x = (i + 0.5)/ppc, cross[j*ppc+i]) and the inner
 * loops of render_zg_fast (fbm.hpp:193), render_generic_fast (362-375) and
 * render_perlin_fast (424-449), evaluated per pixel. */
static double fast_sample(const tg_fbm_config* c, int oct, const tg_octave_spec* os, int64_t gx,
                          int64_t gy, int order) {
    const int64_t ppc = os->ppc;
    const int64_t ix = floor_div(gx, ppc), iy = floor_div(gy, ppc);
    const int64_t rx = gx - ix * ppc, ry = gy - iy * ppc;
    const double xi = ((double)rx + 0.5) / (double)ppc;
    const double yj = ((double)ry + 0.5) / (double)ppc;
    const double si = or_smoothstep(order, xi), sj = or_smoothstep(order, yj);
    const double amp = os->amp;
    switch (c->method) {
        case TG_METHOD_ZG_PAPER:
        case TG_METHOD_ZG_SEPARABLE: {
            const double h00 = corner_data(c, oct, amp, ix, iy, 1, 0, 0).h;
            const double h10 = corner_data(c, oct, amp, ix + 1, iy, 1, 0, 0).h;
            const double h01 = corner_data(c, oct, amp, ix, iy + 1, 1, 0, 0).h;
            const double h11 = corner_data(c, oct, amp, ix + 1, iy + 1, 1, 0, 0).h;
            const double dx = h10 - h00, dy = h01 - h00, a = h11 + h00 - h10 - h01;
            const double cross = c->method == TG_METHOD_ZG_PAPER ? si * yj + sj * xi - xi * yj
                                                                 : si * sj;
            return h00 + si * dx + sj * dy + a * cross;
        }
        case TG_METHOD_GENERIC: {
            double k[12], cc[16];
            const int64_t off[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
            for (int q = 0; q < 4; ++q) {
                const corner_t t = corner_data(c, oct, amp, ix + off[q][0], iy + off[q][1], 1, 1, 0);
                k[q * 3 + 0] = t.h;
                k[q * 3 + 1] = t.f;
                k[q * 3 + 2] = t.g;
            }
            or_generic_coeffs(k, cc);
            return or_generic_eval(cc, xi, yj);
        }
        default: {
            const corner_t a00 = corner_data(c, oct, amp, ix, iy, 0, 0, 1);
            const corner_t a10 = corner_data(c, oct, amp, ix + 1, iy, 0, 0, 1);
            const corner_t a01 = corner_data(c, oct, amp, ix, iy + 1, 0, 0, 1);
            const corner_t a11 = corner_data(c, oct, amp, ix + 1, iy + 1, 0, 0, 1);
            const double y = yj, sy = sj, x = xi, sx = si;
            const double gy_lo = a00.g * y, gy_lo1 = a10.g * y;
            const double gy_hi = a01.g * (y - 1.0), gy_hi1 = a11.g * (y - 1.0);
            const double v00 = a00.f * x + gy_lo;
            const double v10 = a10.f * (x - 1.0) + gy_lo1;
            const double v01 = a01.f * x + gy_hi;
            const double v11 = a11.f * (x - 1.0) + gy_hi1;
            const double h0 = v00 + sx * (v10 - v00);
            const double h1 = v01 + sx * (v11 - v01);
            return h0 + sy * (h1 - h0);
        }
    }
}

/* render_general (fbm.hpp:460-527): per-pixel u = ((gx + 0.5)/R)*freq. */
static double general_sample(const tg_fbm_config* c, int oct, const tg_octave_spec* os,
                             int64_t gx, int64_t gy, int order) {
    const double R = (double)c->resolution;
    if (c->method == TG_METHOD_OPENSIMPLEX) { /* continuous sample position, every octave */
        if (c->zero_lattice) return 0.0;
        const double fr = os->freq / R; /* same operation order as the CUDA kernel */
        const double u = ((double)gx + 0.5) * fr, v = ((double)gy + 0.5) * fr;
        return os->amp * or_opensimplex(c->seed, (uint32_t)oct, u, v);
    }
    const double v = ((double)gy + 0.5) / R * os->freq;
    const int64_t iy = (int64_t)floor(v);
    const double cy = v - (double)iy;
    const double u = ((double)gx + 0.5) / R * os->freq;
    const int64_t ix = (int64_t)floor(u);
    const double cx = u - (double)ix;
    const double amp = os->amp;
    switch (c->method) {
        case TG_METHOD_ZG_PAPER:
        case TG_METHOD_ZG_SEPARABLE:
            return or_zg_eval(corner_data(c, oct, amp, ix, iy, 1, 0, 0).h,
                              corner_data(c, oct, amp, ix + 1, iy, 1, 0, 0).h,
                              corner_data(c, oct, amp, ix, iy + 1, 1, 0, 0).h,
                              corner_data(c, oct, amp, ix + 1, iy + 1, 1, 0, 0).h, cx, cy,
                              c->method == TG_METHOD_ZG_SEPARABLE, order);
        case TG_METHOD_GENERIC: {
            double k[12], cc[16];
            const int64_t off[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
            for (int q = 0; q < 4; ++q) {
                const corner_t t = corner_data(c, oct, amp, ix + off[q][0], iy + off[q][1], 1, 1, 0);
                k[q * 3 + 0] = t.h;
                k[q * 3 + 1] = t.f;
                k[q * 3 + 2] = t.g;
            }
            or_generic_coeffs(k, cc);
            return or_generic_eval(cc, cx, cy);
        }
        default: {
            double f[4], g[4];
            const int64_t off[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
            for (int q = 0; q < 4; ++q) {
                const corner_t t = corner_data(c, oct, amp, ix + off[q][0], iy + off[q][1], 0, 0, 1);
                f[q] = t.f;
                g[q] = t.g;
            }
            return or_perlin_eval(f, g, order, cx, cy);
        }
    }
}

/* generate_into_with_source (fbm.hpp:541-628) for a width x height window;
 * the window checks of 546-558 apply with extent = max(width, height). */
int or_generate(const tg_fbm_config* c, int64_t ox, int64_t oy, int64_t width, int64_t height,
                double* out) {
    if (or_validate(c) != TG_OK) return TG_EVALIDATION;
    if (width < 1 || height < 1 || width > TG_MAX_EXTENT || height > TG_MAX_EXTENT)
        return TG_EVALIDATION;
    const int64_t origin[2] = {ox, oy};
    for (int q = 0; q < 2; ++q) {
        const int64_t o = origin[q];
        if (o < -(1LL << 40) || o > (1LL << 40)) return TG_EVALIDATION;
        const int64_t prod = o * c->base_frequency;
        if (((prod % c->resolution) + c->resolution) % c->resolution != 0) return TG_EVALIDATION;
    }
    const int order = order_of(c);
    const size_t n = (size_t)width * (size_t)height;
    for (size_t i = 0; i < n; ++i) out[i] = 0.0;
    for (int oct = 0; oct < c->octaves; ++oct) {
        tg_octave_spec os;
        or_octave_spec(c, oct, &os);
        for (int64_t ly = 0; ly < height; ++ly) {
            double* row = out + (size_t)ly * (size_t)width;
            for (int64_t lx = 0; lx < width; ++lx) {
                const double v = os.fast && c->method != TG_METHOD_OPENSIMPLEX
                                     ? fast_sample(c, oct, &os, ox + lx, oy + ly, order)
                                     : general_sample(c, oct, &os, ox + lx, oy + ly, order);
                row[lx] += v;
            }
        }
    }
    return TG_OK;
}

/* or_generate split into row bands over `nthreads` host threads (test
 * infrastructure: full-map parity at the BASELINE sizes).  Every pixel still
 * accumulates its octaves 0..N-1 in order, so the result is bit-identical to
 * or_generate; only the window origin is validated (the bands themselves need
 * not be octave-0 aligned). */
typedef struct {
    const tg_fbm_config* c;
    int64_t ox, oy, width, y0, y1;
    int order;
    double* out;
} or_band;

static void* or_band_main(void* p) {
    const or_band* b = (const or_band*)p;
    const tg_fbm_config* c = b->c;
    for (int64_t ly = b->y0; ly < b->y1; ++ly) {
        double* row = b->out + (size_t)ly * (size_t)b->width;
        for (int64_t lx = 0; lx < b->width; ++lx) row[lx] = 0.0;
    }
    for (int oct = 0; oct < c->octaves; ++oct) {
        tg_octave_spec os;
        or_octave_spec(c, oct, &os);
        for (int64_t ly = b->y0; ly < b->y1; ++ly) {
            double* row = b->out + (size_t)ly * (size_t)b->width;
            for (int64_t lx = 0; lx < b->width; ++lx)
                row[lx] += os.fast && c->method != TG_METHOD_OPENSIMPLEX
                               ? fast_sample(c, oct, &os, b->ox + lx, b->oy + ly, b->order)
                               : general_sample(c, oct, &os, b->ox + lx, b->oy + ly, b->order);
        }
    }
    return NULL;
}

int or_generate_mt(const tg_fbm_config* c, int64_t ox, int64_t oy, int64_t width, int64_t height,
                   double* out, int32_t nthreads) {
    if (or_validate(c) != TG_OK) return TG_EVALIDATION;
    if (width < 1 || height < 1 || width > TG_MAX_EXTENT || height > TG_MAX_EXTENT)
        return TG_EVALIDATION;
    const int64_t origin[2] = {ox, oy};
    for (int q = 0; q < 2; ++q) {
        const int64_t o = origin[q];
        if (o < -(1LL << 40) || o > (1LL << 40)) return TG_EVALIDATION;
        const int64_t prod = o * c->base_frequency;
        if (((prod % c->resolution) + c->resolution) % c->resolution != 0) return TG_EVALIDATION;
    }
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (nthreads > height) nthreads = (int32_t)height;
    or_band bands[256];
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) {
        bands[t].c = c;
        bands[t].ox = ox;
        bands[t].oy = oy;
        bands[t].width = width;
        bands[t].y0 = height * t / nthreads;
        bands[t].y1 = height * (t + 1) / nthreads;
        bands[t].order = order_of(c);
        bands[t].out = out;
    }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, or_band_main, &bands[t]);
    or_band_main(&bands[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
    return TG_OK;
}

/* The same per-pixel values as or_generate at arbitrary global pixels
 * (a window's value is a pure function of (cfg, global pixel), fbm.hpp:7-8);
 * used to spot-check maps too large for a full oracle pass. */
int or_sample(const tg_fbm_config* c, const int64_t* gx, const int64_t* gy, int64_t n,
              double* out) {
    if (or_validate(c) != TG_OK) return TG_EVALIDATION;
    const int order = order_of(c);
    for (int64_t i = 0; i < n; ++i) out[i] = 0.0;
    for (int oct = 0; oct < c->octaves; ++oct) {
        tg_octave_spec os;
        or_octave_spec(c, oct, &os);
        for (int64_t i = 0; i < n; ++i)
            out[i] += os.fast && c->method != TG_METHOD_OPENSIMPLEX
                          ? fast_sample(c, oct, &os, gx[i], gy[i], order)
                          : general_sample(c, oct, &os, gx[i], gy[i], order);
    }
    return TG_OK;
}

/* 3D separable zero-gradient fBm (new): per axis the
 * sampling is the 2D one (fast: x = (r + 0.5)/ppc; general: u = (g+0.5)/R*f),
 * the cell is lerp_z(lerp_y(lerp_x(h, Sx), Sy), Sz) over 8 hashed corners. */
static void axis_coord(const tg_octave_spec* os, int64_t R, int64_t g, int64_t* i, double* t) {
    if (os->fast) {
        *i = floor_div(g, os->ppc);
        *t = ((double)(g - *i * os->ppc) + 0.5) / (double)os->ppc;
    } else {
        const double u = ((double)g + 0.5) / (double)R * os->freq;
        *i = (int64_t)floor(u);
        *t = u - (double)*i;
    }
}

/* The separable zero-gradient 3D cell over corners h[q], q = x + 2y + 4z:
 * lerp_z(lerp_y(lerp_x(h, Sx), Sy), Sz).  On the faces z = 0 / z = 1 it is
 * the 2D zg_eval(..., ZgVariant::separable, order) of that face's corners
 * (kernels2d.hpp:70-76), which tests/test_oracle_golden.py pins against the
 * compiled reference. */
double or_cell3(const double h[8], double x, double y, double z, int order) {
    const double sx = or_smoothstep(order, x), sy = or_smoothstep(order, y),
                 sz = or_smoothstep(order, z);
    const double e00 = h[0] + sx * (h[1] - h[0]);
    const double e10 = h[2] + sx * (h[3] - h[2]);
    const double e01 = h[4] + sx * (h[5] - h[4]);
    const double e11 = h[6] + sx * (h[7] - h[6]);
    const double f0 = e00 + sy * (e10 - e00);
    const double f1 = e01 + sy * (e11 - e01);
    return f0 + sz * (f1 - f0);
}

static double voxel3(const tg_fbm_config* c, int oct, const tg_octave_spec* os, int64_t gx,
                     int64_t gy, int64_t gz, int order) {
    int64_t ix, iy, iz;
    double x, y, z;
    axis_coord(os, c->resolution, gx, &ix, &x);
    axis_coord(os, c->resolution, gy, &iy, &y);
    axis_coord(os, c->resolution, gz, &iz, &z);
    double h[8];
    for (int q = 0; q < 8; ++q)
        h[q] = c->zero_lattice ? 0.0
                               : os->amp * or_corner_height3(c->seed, (uint32_t)oct, ix + (q & 1),
                                                             iy + ((q >> 1) & 1), iz + ((q >> 2) & 1));
    return or_cell3(h, x, y, z, order);
}

int or_generate3d(const tg_fbm_config* c, int64_t ox, int64_t oy, int64_t oz, int64_t nx,
                  int64_t ny, int64_t nz, double* out) {
    if (or_validate(c) != TG_OK) return TG_EVALIDATION;
    if (c->method != TG_METHOD_ZG_SEPARABLE) return TG_EVALIDATION;
    if (nx < 1 || ny < 1 || nz < 1) return TG_EVALIDATION;
    const int order = order_of(c);
    const size_t n = (size_t)nx * (size_t)ny * (size_t)nz;
    for (size_t i = 0; i < n; ++i) out[i] = 0.0;
    for (int oct = 0; oct < c->octaves; ++oct) {
        tg_octave_spec os;
        or_octave_spec(c, oct, &os);
        for (int64_t lz = 0; lz < nz; ++lz)
            for (int64_t ly = 0; ly < ny; ++ly)
                for (int64_t lx = 0; lx < nx; ++lx)
                    out[((size_t)lz * (size_t)ny + (size_t)ly) * (size_t)nx + (size_t)lx] +=
                        voxel3(c, oct, &os, ox + lx, oy + ly, oz + lz, order);
    }
    return TG_OK;
}

/* or_generate3d's values at arbitrary global voxels. */
int or_sample3d(const tg_fbm_config* c, const int64_t* gx, const int64_t* gy, const int64_t* gz,
                int64_t n, double* out) {
    if (or_validate(c) != TG_OK) return TG_EVALIDATION;
    if (c->method != TG_METHOD_ZG_SEPARABLE) return TG_EVALIDATION;
    const int order = order_of(c);
    for (int64_t i = 0; i < n; ++i) out[i] = 0.0;
    for (int oct = 0; oct < c->octaves; ++oct) {
        tg_octave_spec os;
        or_octave_spec(c, oct, &os);
        for (int64_t i = 0; i < n; ++i) out[i] += voxel3(c, oct, &os, gx[i], gy[i], gz[i], order);
    }
    return TG_OK;
}

/* normalize_map (fbm.hpp:638-656), in place. */
int or_normalize(double* data, int64_t n, double* lo_out, double* hi_out, int* constant_source) {
    *constant_source = 0;
    if (n <= 0) return TG_OK;
    double lo = data[0], hi = data[0];
    for (int64_t i = 0; i < n; ++i) {
        lo = data[i] < lo ? data[i] : lo;
        hi = data[i] > hi ? data[i] : hi;
    }
    *lo_out = lo;
    *hi_out = hi;
    if (lo == hi) {
        *constant_source = 1;
        return TG_OK;
    }
    const double span = hi - lo;
    for (int64_t i = 0; i < n; ++i) data[i] = -1.0 + 2.0 * (data[i] - lo) / span;
    return TG_OK;
}

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* analysis.hpp:244-250: nth_element at n/2 (upper median). */
double or_upper_median(const double* data, int64_t n) {
    double* tmp = (double*)malloc((size_t)n * sizeof(double));
    memcpy(tmp, data, (size_t)n * sizeof(double));
    qsort(tmp, (size_t)n, sizeof(double), cmp_double);
    const double m = tmp[n / 2];
    free(tmp);
    return m;
}

/* coastline_mask (analysis.hpp:213-240) */
int or_coastline_mask(const double* h, int64_t R, double sea, uint8_t* mask, int64_t* land_out) {
    if (R < 2) return TG_EVALIDATION;
    int64_t land_count = 0;
#define LAND(x, y) (h[(size_t)(y) * (size_t)R + (size_t)(x)] >= sea)
    for (int64_t y = 0; y < R; ++y)
        for (int64_t x = 0; x < R; ++x) {
            mask[(size_t)y * (size_t)R + (size_t)x] = 0;
            if (!LAND(x, y)) continue;
            ++land_count;
            const int wn = (x > 0 && !LAND(x - 1, y)) || (x + 1 < R && !LAND(x + 1, y)) ||
                           (y > 0 && !LAND(x, y - 1)) || (y + 1 < R && !LAND(x, y + 1));
            if (wn) mask[(size_t)y * (size_t)R + (size_t)x] = 1;
        }
#undef LAND
    *land_out = land_count;
    if (land_count == 0 || land_count == R * R) return TG_EVALIDATION;
    return TG_OK;
}

/* linear_fit (analysis.hpp:29-63) */
int or_linear_fit(const double* xs, const double* ys, int64_t n, double* slope,
                  double* intercept, double* r2) {
    if (n < 2) return TG_EVALIDATION;
    double mx = 0.0, my = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        mx += xs[i];
        my += ys[i];
    }
    mx /= (double)n;
    my /= (double)n;
    double sxx = 0.0, sxy = 0.0, syy = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double dx = xs[i] - mx, dy = ys[i] - my;
        sxx += dx * dx;
        sxy += dx * dy;
        syy += dy * dy;
    }
    if (sxx == 0.0) return TG_EVALIDATION;
    *slope = sxy / sxx;
    *intercept = my - *slope * mx;
    if (syy == 0.0) {
        *r2 = 1.0;
        return TG_OK;
    }
    double ssr = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double r = ys[i] - (*slope * xs[i] + *intercept);
        ssr += r * r;
    }
    *r2 = 1.0 - ssr / syy;
    return TG_OK;
}

/* box_count (analysis.hpp:269-305) */
int or_box_count(const uint8_t* mask, int64_t R, const int32_t* sizes, int32_t n_sizes,
                 int64_t* counts, double* d, double* k, double* r2) {
    if (R < 2) return TG_EVALIDATION;
    if (n_sizes < 3) return TG_EVALIDATION;
    for (int i = 0; i < n_sizes; ++i) {
        if (sizes[i] < 1 || sizes[i] > R) return TG_EVALIDATION;
        if (i > 0 && sizes[i] <= sizes[i - 1]) return TG_EVALIDATION;
    }
    int64_t pix = 0;
    for (int64_t i = 0; i < R * R; ++i) pix += mask[i];
    if (pix == 0) return TG_EVALIDATION;
    double* le = (double*)malloc((size_t)n_sizes * sizeof(double));
    double* lc = (double*)malloc((size_t)n_sizes * sizeof(double));
    for (int s = 0; s < n_sizes; ++s) {
        const int64_t eps = sizes[s];
        const int64_t bpa = (R + eps - 1) / eps;
        uint8_t* occ = (uint8_t*)calloc((size_t)(bpa * bpa), 1);
        for (int64_t y = 0; y < R; ++y)
            for (int64_t x = 0; x < R; ++x)
                if (mask[(size_t)y * (size_t)R + (size_t)x]) occ[(y / eps) * bpa + x / eps] = 1;
        int64_t nb = 0;
        for (int64_t i = 0; i < bpa * bpa; ++i) nb += occ[i];
        free(occ);
        counts[s] = nb;
        le[s] = log((double)eps);
        lc[s] = log((double)nb);
    }
    double slope = 0, icept = 0, rr = 0;
    const int st = or_linear_fit(le, lc, n_sizes, &slope, &icept, &rr);
    free(le);
    free(lc);
    if (st != TG_OK) return st;
    *d = -slope;
    *k = exp(icept);
    *r2 = rr;
    return TG_OK;
}

/* Height-difference variogram (new; no reference): for lag h along x and y,
 * sum of (z(p + h e) - z(p))^2 over in-window pairs, and the pair count. */
int or_variogram(const double* z, int64_t W, int64_t H, const int32_t* lags, int32_t n_lags,
                 double* sum_sq, int64_t* pairs) {
    for (int i = 0; i < n_lags; ++i) {
        const int64_t h = lags[i];
        if (h < 1) return TG_EVALIDATION;
        double sx = 0.0, sy = 0.0;
        int64_t px = 0, py = 0;
        for (int64_t y = 0; y < H; ++y)
            for (int64_t x = 0; x < W; ++x) {
                const double v = z[y * W + x];
                if (x + h < W) {
                    const double d = z[y * W + x + h] - v;
                    sx += d * d;
                    ++px;
                }
                if (y + h < H) {
                    const double d = z[(y + h) * W + x] - v;
                    sy += d * d;
                    ++py;
                }
            }
        sum_sq[2 * i] = sx;
        sum_sq[2 * i + 1] = sy;
        pairs[2 * i] = px;
        pairs[2 * i + 1] = py;
    }
    return TG_OK;
}

/* gradient_norm_map / hessian_norm_map (tools/terrain_cli.cpp:148-182):
 * central differences inside, clamped at the borders, pixel units. */
int or_norm_map(const double* m, int64_t W, int64_t H, int hessian, double* out) {
#define AT(xx, yy) m[(yy) * W + (xx)]
    for (int64_t y = 0; y < H; ++y) {
        const int64_t ym = y > 0 ? y - 1 : 0, yp = y + 1 < H ? y + 1 : H - 1;
        for (int64_t x = 0; x < W; ++x) {
            const int64_t xm = x > 0 ? x - 1 : 0, xp = x + 1 < W ? x + 1 : W - 1;
            if (!hessian) {
                const double gx = 0.5 * (AT(xp, y) - AT(xm, y));
                const double gy = 0.5 * (AT(x, yp) - AT(x, ym));
                out[y * W + x] = sqrt(gx * gx + gy * gy);
            } else {
                const double hxx = AT(xp, y) - 2.0 * AT(x, y) + AT(xm, y);
                const double hyy = AT(x, yp) - 2.0 * AT(x, y) + AT(x, ym);
                const double hxy = 0.25 * (AT(xp, yp) - AT(xm, yp) - AT(xp, ym) + AT(xm, ym));
                out[y * W + x] = sqrt(hxx * hxx + 2.0 * hxy * hxy + hyy * hyy);
            }
        }
    }
#undef AT
    return TG_OK;
}
