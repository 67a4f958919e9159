// fbm2d.cu — fused-octave 2D fBm kernel for sm_100a.
//
// Replaces the octave loop of generate_into_with_source
// (terrain/fbm.hpp:541-628) and its render paths render_zg_fast (231-312),
// render_generic_fast (321-379), render_perlin_fast (384-455) and
// render_general (460-527).  One CTA owns a 128 x 64 pixel tile whose
// accumulators stay in registers across ALL octaves; the map is written once
// (4 B/pixel) instead of the reference's read-modify-write of a double buffer
// per octave (fbm.hpp:187,193).
//
// The CTA runs one prologue for ALL octaves — every octave's unique lattice
// corners for the tile hashed once into shared memory (plus per-CTA sampling
// tables for general octaves) — then barrier-free loops over host-built,
// mode-homogeneous octave lists in which each thread evaluates its 4 x 8
// pixels from the shared corners with the cell polynomial factorised per
// (cell, row):
//   zg paper     v = c0 + sx*c1 + x*c2      (kernels2d.hpp:62-76)
//   zg separable v = c0 + sx*c1
//   perlin       v = a0 + x*a1 + sx*a2 + x*sx*a3   (kernels2d.hpp:163-173)
//   generic      v = ((r3*x + r2)*x + r1)*x + r0    (kernels2d.hpp:124-134)
// Octaves whose samples sit exactly on lattice points (kClsSubInt) need no
// grid: each pixel hashes its one corner in registers.
//
// Every pixel's arithmetic is a function of (config, global pixel) only, so
// any window / tile decomposition reproduces the same bits (fbm.hpp:7-8).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <mutex>
#include <type_traits>

#include "devattr.h"

// FFMA2 / FADD2 column pairs (bit-identical per lane) in the lattice-point,
// ppc-2 and ppc-1 zero-gradient octaves (config 2: 51.2 -> 50.2 us); the
// pixel formation of the separated form too would exceed 64 registers.
#ifndef TG_F2_SUB
#define TG_F2_SUB 1
#endif
#ifndef TG_F2_PPC2
#define TG_F2_PPC2 1
#endif
#ifndef TG_F2_PPC1
#define TG_F2_PPC1 1
#endif
#ifndef TG_F2_BLK
#define TG_F2_BLK 1
#endif
#ifndef TG_F2_FORM
#define TG_F2_FORM 0
#endif
#include "fbm_params.h"
#include "lattice.cuh"

namespace tg {

constexpr int kThreads = 256;
constexpr int kTW = kTileW;
constexpr int kTH = kTileH;

template <int ORDER>
__device__ __forceinline__ float smooth(float t) {
    if constexpr (ORDER == 5) return t * t * t * fmaf(t, fmaf(6.f, t, -15.f), 10.f);  // 26-38
    else return t * t * fmaf(-2.f, t, 3.f);
}

template <int KIND> struct Traits;
template <> struct Traits<kZgPaper> { static constexpr int kCh = 1; };
template <> struct Traits<kZgSeparable> { static constexpr int kCh = 1; };
template <> struct Traits<kPerlin> { static constexpr int kCh = 2; };
template <> struct Traits<kGeneric> { static constexpr int kCh = 3; };

// Corner data of one lattice point from its packed key (lattice.hpp:46-50),
// scaled like the reference's render paths: zg/generic heights x amp
// (fbm.hpp:270,349), Perlin unit gradients x amp (409-420), generic gradients
// x w, unscaled by amp (348).  amp63 = amp * kMapScale (map_height).
// ZeroSource (fbm.hpp:125-133) is amp = w = 0, set by the host planner.
template <int KIND>
__device__ __forceinline__ void corner_data_packed(uint64_t p, float amp, float amp63, float w, float* d) {
    if constexpr (KIND == kZgPaper || KIND == kZgSeparable) {
        d[0] = amp63 * map_height(p);
    } else if constexpr (KIND == kPerlin) {
        float c, s;
        fast_sincos_turns(unit_from_hash(mix64(p ^ kMapLane(kAngleLane))), &s, &c);
        d[0] = amp * c;
        d[1] = amp * s;
    } else {
        d[0] = amp63 * map_height(p);
        float c, s;
        fast_sincos_turns(unit_from_hash(mix64(p ^ kMapLane(kAngleLane))), &s, &c);
        const float m = unit_from_hash(mix64(p ^ kMapLane(kMagnitudeLane))) * w;
        d[1] = m * c;
        d[2] = m * s;
    }
}

template <int KIND>
__device__ __forceinline__ void corner_data(uint64_t base, int64_t ix, int64_t iy, float amp, float w,
                                            float* d) {
    corner_data_packed<KIND>(pack_xy(base, ix, iy), amp, amp * kMapScale, w, d);
}

// Per-cell constants (from the 4 corners) and per-(cell,row) coefficients.
template <int KIND> struct Cell;

template <> struct Cell<kZgPaper> {
    float h00, dx, dy, a;  // zg_params (kernels2d.hpp:62-64)
    __device__ __forceinline__ void make(const float* k00, const float* k10, const float* k01,
                                         const float* k11) {
        h00 = k00[0];
        dx = k10[0] - k00[0];
        dy = k01[0] - k00[0];
        a = (k11[0] - k10[0]) - dy;  // h11 + h00 - h10 - h01
    }
    struct Row { float c0, c1, c2; };
    __device__ __forceinline__ Row row(float y, float sy) const {
        // h00 + sx*dx + sy*dy + a*(sx*y + sy*x - x*y) = c0 + sx*c1 + x*c2
        return {fmaf(sy, dy, h00), fmaf(a, y, dx), a * (sy - y)};
    }
    __device__ __forceinline__ static float eval(const Row& r, float x, float sx, float) {
        return fmaf(x, r.c2, fmaf(sx, r.c1, r.c0));
    }
};

template <> struct Cell<kZgSeparable> {
    float h00, dx, dy, a;
    __device__ __forceinline__ void make(const float* k00, const float* k10, const float* k01,
                                         const float* k11) {
        h00 = k00[0];
        dx = k10[0] - k00[0];
        dy = k01[0] - k00[0];
        a = (k11[0] - k10[0]) - dy;
    }
    struct Row { float c0, c1; };
    __device__ __forceinline__ Row row(float, float sy) const {
        // h00 + sx*dx + sy*dy + a*sx*sy = c0 + sx*c1
        return {fmaf(sy, dy, h00), fmaf(a, sy, dx)};
    }
    __device__ __forceinline__ static float eval(const Row& r, float, float sx, float) {
        return fmaf(sx, r.c1, r.c0);
    }
};

template <> struct Cell<kPerlin> {
    // kernels2d.hpp:163-173: lerp_y of the two x-lerped gradient ramps.  For a
    // fixed cell every coefficient of the column features {1, x, sx, x*sx} is
    // a linear combination of the row features {1, y, sy, y*sy}.
    float a0y, a0ys, a0s, a1c, a1s, a2c, a2y, a2ys, a2s, a3c, a3s;
    __device__ __forceinline__ void make(const float* k00, const float* k10, const float* k01,
                                         const float* k11) {
        const float f0 = k00[0], g0 = k00[1], f1 = k10[0], g1 = k10[1];  // corners 00, 10
        const float f2 = k01[0], g2 = k01[1], f3 = k11[0], g3 = k11[1];  // corners 01, 11
        a0y = g0;
        a0ys = g2 - g0;
        a0s = -g2;
        a1c = f0;
        a1s = f2 - f0;
        a2c = -f1;
        a2y = g1 - g0;
        a2ys = (g3 - g2) - a2y;
        a2s = (f1 - f3) - (g3 - g2);
        a3c = f1 - f0;
        a3s = (f3 - f2) - a3c;
    }
    struct Row { float a0, a1, a2, a3; };
    __device__ __forceinline__ Row row(float y, float sy) const {
        const float ys = y * sy;
        return {fmaf(a0y, y, fmaf(a0ys, ys, a0s * sy)), fmaf(sy, a1s, a1c),
                fmaf(a2y, y, fmaf(a2ys, ys, fmaf(a2s, sy, a2c))), fmaf(sy, a3s, a3c)};
    }
    __device__ __forceinline__ static float eval(const Row& r, float x, float sx, float xs) {
        return fmaf(xs, r.a3, fmaf(sx, r.a2, fmaf(x, r.a1, r.a0)));
    }
};

template <> struct Cell<kGeneric> {
    // generic_coeffs (kernels2d.hpp:103-122): c[i][j] on x^i y^j, the
    // upper-right quad (i, j >= 2) identically zero.
    float c00, c01, c02, c03, c10, c11, c12, c13, c20, c21, c30, c31;
    __device__ __forceinline__ void make(const float* k00, const float* k10, const float* k01,
                                         const float* k11) {
        const float h00 = k00[0], f00 = k00[1], g00 = k00[2];
        const float h10 = k10[0], f10 = k10[1], g10 = k10[2];
        const float h01 = k01[0], f01 = k01[1], g01 = k01[2];
        const float h11 = k11[0], f11 = k11[1], g11 = k11[2];
        c00 = h00;
        c10 = f00;
        c01 = g00;
        c20 = 3.f * (h10 - h00) - 2.f * f00 - f10;
        c30 = f10 + f00 - 2.f * (h10 - h00);
        c02 = 3.f * (h01 - h00) - 2.f * g00 - g01;
        c03 = g01 + g00 - 2.f * (h01 - h00);
        c21 = 3.f * (h11 - h01) - 2.f * f01 - f11 - c20;
        c31 = f11 + f01 - 2.f * (h11 - h01) - c30;
        c12 = 3.f * (h11 - h10) - 2.f * g10 - g11 - c02;
        c13 = g11 + g10 - 2.f * (h11 - h10) - c03;
        c11 = h01 + h10 - h00 - h11 + f01 + g10 - g00 - f00;
    }
    struct Row { float r0, r1, r2, r3; };
    __device__ __forceinline__ Row row(float y, float) const {
        // Horner in y per x power (kernels2d.hpp:128-132)
        return {fmaf(fmaf(fmaf(c03, y, c02), y, c01), y, c00),
                fmaf(fmaf(fmaf(c13, y, c12), y, c11), y, c10), fmaf(c21, y, c20),
                fmaf(c31, y, c30)};
    }
    __device__ __forceinline__ static float eval(const Row& r, float x, float, float) {
        return fmaf(fmaf(fmaf(r.r3, x, r.r2), x, r.r1), x, r.r0);
    }
};

// Global coordinate -> (cell index, local coordinate) for one octave.
__device__ __forceinline__ void axis_coord(const OctDev& od, double R, int64_t g, int64_t* i,
                                           float* t) {
    if (od.cls == kClsFast) {
        int64_t q, r;
        if (od.shift >= 0) {  // floor_div by a power of two (fbm.hpp:137-141)
            q = g >> od.shift;
            r = g & (static_cast<int64_t>(od.ppc) - 1);
        } else {
            q = g / od.ppc;
            r = g - q * od.ppc;
            if (r < 0) {
                --q;
                r += od.ppc;
            }
        }
        *i = q;
        *t = (static_cast<float>(r) + 0.5f) * od.inv_ppc;  // RowLut x (kernels2d.hpp:231)
    } else {
        // render_general (fbm.hpp:468,474): ((g + 0.5) / R) * freq in fp64,
        // IEEE-rounded like the x86 reference so floor() picks identical cells.
        const double u = __dmul_rn(__ddiv_rn(__dadd_rn(static_cast<double>(g), 0.5), R), od.freq);
        const int64_t q = __double2ll_rd(u);
        *i = q;
        *t = static_cast<float>(__dsub_rn(u, static_cast<double>(q)));
    }
}

struct TabSlot {
    float colX[kTW], colS[kTW], colXS[kTW];
    int32_t colI[kTW];  // cell index relative to the tile's first cell
    float4 rowF[kTH];   // y, S(y), S(y) - y, cell row relative (bits)
};

// LEAN kernels (no general octaves) need no sampling tables.  The zg paper
// kernels add the per-tile column / row term arrays (kGBlkT) after the grid.
template <int KIND, bool LEAN>
constexpr size_t smem_grid_end() {
    return (LEAN ? 0 : sizeof(TabSlot) * kTabSlots) + sizeof(float) * Traits<KIND>::kCh * kGridCap;
}
// floats: Cw[2][128], C1[2][128], Rw[4][64], R1[4][64], then the kGBlkT
// octaves' cell coefficients: column float4 x 8 cells per slot, row float2 x 8
constexpr int kFeat = 4 * 256 + 6 * 8 * kMaxCellSlots;
template <int KIND, bool LEAN>
constexpr size_t smem_bytes() {
    return smem_grid_end<KIND, LEAN>() + (KIND == kZgPaper ? sizeof(float) * kFeat : 0);
}

// Corner weights of a zero-gradient cell at ppc = 2 (kernels2d.hpp:62-76):
// position (ix, iy) has x = (2 ix + 1)/4, y = (2 iy + 1)/4; corner k = 0..3 is
// h00, h10, h01, h11.  paper: c = Sx*y + Sy*x - x*y; separable: c = Sx*Sy;
// w = (1 - Sx - Sy + c, Sx - c, Sy - c, c).  Every term is exact in fp32.
template <int KIND, int ORDER>
struct Ppc2W {
    static constexpr float S(int i) {  // S(1/4), S(3/4) (smoothstep3/5, kernels2d.hpp:26-38)
        return ORDER == 5 ? (i ? 0.896484375f : 0.103515625f) : (i ? 0.84375f : 0.15625f);
    }
    static constexpr float X(int i) { return i ? 0.75f : 0.25f; }
    static constexpr float C(int ix, int iy) {
        return KIND == kZgSeparable ? S(ix) * S(iy) : S(ix) * X(iy) + S(iy) * X(ix) - X(ix) * X(iy);
    }
    static constexpr float w(int ix, int iy, int k) {
        return k == 0 ? 1.0f - S(ix) - S(iy) + C(ix, iy)
                      : k == 1 ? S(ix) - C(ix, iy) : k == 2 ? S(iy) - C(ix, iy) : C(ix, iy);
    }
};

// S(x) and S(x) - x at the ppc-4 sample positions x = (2i + 1)/8, i = 0..3
// (smoothstep3/5, kernels2d.hpp:26-38), exact in fp32 (the row LUT's fp64
// values rounded once: every one of them is a dyadic rational with < 24 bits).
template <int ORDER>
struct Ppc4S {
    static constexpr double Sd(int i) {
        const double x = (2.0 * i + 1.0) / 8.0;
        return ORDER == 5 ? x * x * x * (10.0 + x * (6.0 * x - 15.0)) : x * x * (3.0 - 2.0 * x);
    }
    static constexpr float S(int i) { return static_cast<float>(Sd(i)); }
    static constexpr float D(int i) { return static_cast<float>(Sd(i) - (2.0 * i + 1.0) / 8.0); }
};

// acc[j] += m * h[j] for the four columns, as two FFMA2 (column pairs;
// each lane rounds exactly as fmaf(m, h[j], acc[j])).
__device__ __forceinline__ void fma_pairs(float (&acc)[4], const float* h, float m) {
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const float2 a = __ffma2_rn(make_float2(h[2 * p], h[2 * p + 1]), make_float2(m, m),
                                    make_float2(acc[2 * p], acc[2 * p + 1]));
        acc[2 * p] = a.x;
        acc[2 * p + 1] = a.y;
    }
}

// Separated-form terms of one block octave (zg paper, ppc >= 8) in FFMA2
// pairs, each lane rounded as the scalar form:
//   C0[j] = fmaf(D[j], ay0, fmaf(S[j], dx, C0[j])), C1[j] = fmaf(D[j], ad, C1[j]),
//   R0[r] = fmaf(Sy[r], k0, R0[r]),                 R1[r] = fmaf(Sy[r], ad, R1[r]).
template <class SyLoad>
__device__ __forceinline__ void sep_terms(float (&C0)[4], float (&C1)[4], float (&R0)[kRPT], float (&R1)[kRPT],
                                          float4 sx, float4 dd, float dx, float ay0, float ad, float k0,
                                          SyLoad sy_load) {
    const float2 S2[2] = {make_float2(sx.x, sx.y), make_float2(sx.z, sx.w)};
    const float2 D2[2] = {make_float2(dd.x, dd.y), make_float2(dd.z, dd.w)};
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        float2 c0 = __ffma2_rn(S2[p], make_float2(dx, dx), make_float2(C0[2 * p], C0[2 * p + 1]));
        c0 = __ffma2_rn(D2[p], make_float2(ay0, ay0), c0);
        const float2 c1 = __ffma2_rn(D2[p], make_float2(ad, ad), make_float2(C1[2 * p], C1[2 * p + 1]));
        C0[2 * p] = c0.x, C0[2 * p + 1] = c0.y;
        C1[2 * p] = c1.x, C1[2 * p + 1] = c1.y;
    }
#pragma unroll
    for (int r4 = 0; r4 < kRPT; r4 += 4) {
        const float4 sy = sy_load(r4);
        const float2 Y2[2] = {make_float2(sy.x, sy.y), make_float2(sy.z, sy.w)};
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const int r = r4 + 2 * p;
            const float2 a = __ffma2_rn(Y2[p], make_float2(k0, k0), make_float2(R0[r], R0[r + 1]));
            const float2 b = __ffma2_rn(Y2[p], make_float2(ad, ad), make_float2(R1[r], R1[r + 1]));
            R0[r] = a.x, R0[r + 1] = a.y;
            R1[r] = b.x, R1[r + 1] = b.y;
        }
    }
}

// q*((h00 + h10) + (h01 + h11)) over a 4 x 8 pixel block whose corners are
// rows r = 0..8 of a 5-wide corner strip: x = y = 0.5 makes every zero-
// gradient kernel (S3 or S5, paper or separable) the mean of its 4 corners
// (q = amp/4, folded with the grid's 2^-63 height scale).
template <class Fetch>
__device__ __forceinline__ void ppc1_block(float (&acc)[kRPT][4], float q, Fetch fetch) {
    float h[5];
    fetch(0, h);
    float hs[4] = {h[0] + h[1], h[1] + h[2], h[2] + h[3], h[3] + h[4]};
#pragma unroll
    for (int r = 0; r < kRPT; ++r) {
        fetch(r + 1, h);
        const float ns[4] = {h[0] + h[1], h[1] + h[2], h[2] + h[3], h[3] + h[4]};
#pragma unroll
#if TG_F2_PPC1
        for (int p = 0; p < 2; ++p) {  // column pairs in FADD2 / FFMA2 (each lane as before)
            const float2 s = __fadd2_rn(make_float2(hs[2 * p], hs[2 * p + 1]), make_float2(ns[2 * p], ns[2 * p + 1]));
            const float2 a = __ffma2_rn(make_float2(q, q), s, make_float2(acc[r][2 * p], acc[r][2 * p + 1]));
            acc[r][2 * p] = a.x;
            acc[r][2 * p + 1] = a.y;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) hs[j] = ns[j];
#else
        for (int j = 0; j < 4; ++j) {
            acc[r][j] = fmaf(q, hs[j] + ns[j], acc[r][j]);
            hs[j] = ns[j];
        }
#endif
    }
}

// Corner grid of one aligned power-of-two octave (ppc = 2^SH <= 16) for a
// 128 x 64 tile: (Wm + 1) x (Hm + 1) corners, Wm = 128 >> SH, Hm = 64 >> SH.
// The Wm x Hm main block goes 4 consecutive corners per lane (four
// independent hash chains, keys advanced by +K3, one 16-byte store per
// channel), rows strided over the warps starting at warp `rot`; the last
// column and row go one corner per thread starting at thread 32 * rot.
template <int SH, int CH, bool SCALE = false, class GV>
__device__ __forceinline__ void fine_grid(float* g, int pitch, uint64_t p0, int warp, int lane, int tid, int rot,
                                          GV& grid_value, const OctDev& od, float scale = 1.0f) {
    constexpr int Wm = kTileW >> SH, Hm = kTileH >> SH;
    constexpr int LSH = 5 - SH;                   // log2(lanes per corner row) = log2(Wm / 4)
    constexpr int RSTEP = 8 << SH;                // corner rows per pass over the 8 warps
    constexpr int NIT = (Hm + RSTEP - 1) / RSTEP;  // passes
    const int wv = (warp - rot) & 7;
    const int cg = lane & ((1 << LSH) - 1), rs = lane >> LSH;
    const int cy0 = (wv << SH) + rs;
    // ppc >= 4: only the first Hm >> SH warps hold main-block rows (warp-uniform skip)
    if (Hm >= RSTEP || (wv << SH) < Hm) {
    uint64_t p = p0 + static_cast<uint64_t>(4 * cg) * kIxMul + static_cast<uint64_t>(static_cast<uint32_t>(cy0)) * kIyMul;
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
        const int cy = cy0 + it * RSTEP;
        if (Hm % RSTEP == 0 || cy < Hm) {
            float d[4][CH];
            if constexpr (CH == 1) {
                float h[4];
                map_height4(p, add64(p, kIxMul), add64(p, 2 * kIxMul), add64(p, 3 * kIxMul), h);
#pragma unroll
                for (int u = 0; u < 4; ++u) d[u][0] = SCALE ? scale * h[u] : h[u];
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) grid_value(add64(p, u * kIxMul), od, d[u]);
            }
#pragma unroll
            for (int c = 0; c < CH; ++c)
                *reinterpret_cast<float4*>(g + c * kGridCap + cy * pitch + 4 * cg) =
                    make_float4(d[0][c], d[1][c], d[2][c], d[3][c]);
        }
        if (it + 1 < NIT) p = add64(p, static_cast<uint64_t>(RSTEP) * kIyMul);
    }
    }
    constexpr int NE = Hm + 1 + Wm;  // last column (Hm + 1 corners) then last row (Wm)
    for (int i = (tid - 32 * rot) & (kThreads - 1); i < NE; i += kThreads) {
        const int cx = i <= Hm ? Wm : i - Hm - 1;
        const int cy = i <= Hm ? i : Hm;
        float d[CH];
        grid_value(p0 + static_cast<uint64_t>(static_cast<uint32_t>(cx)) * kIxMul +
                       static_cast<uint64_t>(static_cast<uint32_t>(cy)) * kIyMul,
                   od, d);
#pragma unroll
        for (int c = 0; c < CH; ++c) g[c * kGridCap + cy * pitch + cx] = SCALE ? scale * d[c] : d[c];
    }
}

// fine_grid with the shape decided at run time (same corner assignment).
template <int CH, class GV>
__device__ __forceinline__ void fine_grid_rt(int sh, float* g, int pitch, uint64_t p0, int warp, int lane, int tid,
                                          int rot, GV& grid_value, const OctDev& od) {
    const int Wm = kTileW >> sh, Hm = kTileH >> sh;
    const int lsh = 5 - sh, rstep = 8 << sh;
    const int wv = (warp - rot) & 7;
    const int cg = lane & ((1 << lsh) - 1), rs = lane >> lsh;
    const uint64_t px = p0 + static_cast<uint64_t>(4 * cg) * kIxMul;
    for (int cy = (wv << sh) + rs; cy < Hm; cy += rstep) {
        const uint64_t p = px + static_cast<uint64_t>(static_cast<uint32_t>(cy)) * kIyMul;
        float d[4][CH];
#pragma unroll
        for (int u = 0; u < 4; ++u) grid_value(add64(p, u * kIxMul), od, d[u]);
#pragma unroll
        for (int c = 0; c < CH; ++c)
            *reinterpret_cast<float4*>(g + c * kGridCap + cy * pitch + 4 * cg) =
                make_float4(d[0][c], d[1][c], d[2][c], d[3][c]);
    }
    for (int i = (tid - 32 * rot) & (kThreads - 1); i < Hm + 1 + Wm; i += kThreads) {
        const int cx = i <= Hm ? Wm : i - Hm - 1;
        const int cy = i <= Hm ? i : Hm;
        float d[CH];
        grid_value(p0 + static_cast<uint64_t>(static_cast<uint32_t>(cx)) * kIxMul +
                       static_cast<uint64_t>(static_cast<uint32_t>(cy)) * kIyMul,
                   od, d);
#pragma unroll
        for (int c = 0; c < CH; ++c) g[c * kGridCap + cy * pitch + cx] = d[c];
    }
}

// zero-gradient cell rows r_begin.. of one cell: c0 = h00 + sy*dy goes into
// the per-row accumulator (common to the 4 columns), the rest per pixel.
// Zero-gradient cell in column form: with the column features
// e1 = dy + a*x (paper) / dy + a*Sx (separable) and e2 = a*(Sx - x),
//   paper      v = (h00 + Sx*dx) + Sy*e1 + y*e2   -> 2 FFMA per pixel,
//   separable  v = (h00 + Sx*dx) + Sy*e1          -> 1 FFMA per pixel,
// the column-constant part accumulating in cacc[4] (4 registers instead of
// the 8 row accumulators) and h00 in one per-thread sum when the cell covers
// all the thread's rows (ONE_CELL); otherwise (ppc = 4, two cell rows) the
// column constant of this cell row is added per pixel.  Per row only
// (y, Sy) is loaded.
template <int KIND, int NR, bool ONE_CELL>
__device__ __forceinline__ void zg_cols(float (&acc)[kRPT][4], float (&cacc)[4], float& hsum, int r_begin,
                                        const float4* __restrict__ Ly, const float (&x)[4],
                                        const float (&sx)[4], const float (&smx)[4], float h00, float h10,
                                        float h01, float h11) {
    const float dx = h10 - h00, dy = h01 - h00, a = (h11 - h10) - dy;
    if constexpr (ONE_CELL) hsum += h00;
    float e0[4], e1[4], e2[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if constexpr (ONE_CELL) cacc[j] = fmaf(sx[j], dx, cacc[j]);
        else e0[j] = fmaf(sx[j], dx, h00);
        if constexpr (KIND == kZgPaper) {
            e1[j] = fmaf(a, x[j], dy);
            e2[j] = a * smx[j];
        } else {
            e1[j] = fmaf(a, sx[j], dy);
        }
    }
#pragma unroll
    for (int rr = 0; rr < NR; ++rr) {
        const int r = r_begin + rr;
        const float4 f = Ly[rr];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float base = ONE_CELL ? acc[r][j] : acc[r][j] + e0[j];
            if constexpr (KIND == kZgPaper) acc[r][j] = fmaf(f.x, e2[j], fmaf(f.y, e1[j], base));
            else acc[r][j] = fmaf(f.y, e1[j], base);
        }
    }
}

// Timing experiments only: TG_SKIP is a bit mask of octave lists to skip
// (1 fine grids, 2 lattice-point octaves, 4 per-thread block octaves, 8
// per-tile block octaves, 16 ppc-4, 32 ppc-2, 64 ppc-1); 0 in every build
// that produces maps.
#ifndef TG_SKIP
#define TG_SKIP 0
#endif
#define TG_NG(g, bit) ((TG_SKIP & (bit)) ? 0 : args.ngroup[g])

#ifndef TG_ZG_MIN_BLOCKS
#define TG_ZG_MIN_BLOCKS 3
#endif
#ifndef TG_ZG_LEAN_MIN_BLOCKS
#define TG_ZG_LEAN_MIN_BLOCKS 4
#endif
#ifndef TG_PDL
#define TG_PDL 1  // programmatic dependent launch of the 2D generation kernel
#endif
#ifndef TG_PPC2_WEIGHTS
#define TG_PPC2_WEIGHTS 1  // zero-gradient ppc-2 octaves as fixed corner blends
#endif
#ifndef TG_SUB_ROWS
#define TG_SUB_ROWS 2  // lattice-point octaves: pixel rows hashed per step (1, 2 or 4)
#endif
#ifndef TG_TMA_STORE
#define TG_TMA_STORE 1
#endif
#ifndef TG_GEN_MIN_BLOCKS
#define TG_GEN_MIN_BLOCKS 1
#endif

// LEAN: the plan has no general (non-dividing / fractional) octaves and no
// texture epilogue (decided on the host): that code and the sampling tables
// are compiled out.
template <int KIND, int ORDER, bool LEAN>
__global__ void __launch_bounds__(kThreads, (KIND == kZgPaper || KIND == kZgSeparable)
                                                ? (LEAN ? TG_ZG_LEAN_MIN_BLOCKS : TG_ZG_MIN_BLOCKS)
                                                : (KIND == kPerlin ? 2 : TG_GEN_MIN_BLOCKS))
fbm2d_kernel(const __grid_constant__ FbmArgs args, const __grid_constant__ CUtensorMap tmap,
             float* __restrict__ out) {
    constexpr int CH = Traits<KIND>::kCh;
    constexpr bool kZg = KIND == kZgPaper || KIND == kZgSeparable;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    TabSlot* tabs = reinterpret_cast<TabSlot*>(smem_raw);
    float* grid = reinterpret_cast<float*>(smem_raw + (LEAN ? 0 : sizeof(TabSlot) * kTabSlots));

    // let the next launch on the stream start filling SMs as this grid drains
    asm volatile("griddepcontrol.launch_dependents;");
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int64_t tx0 = args.tile_x0 + static_cast<int64_t>(blockIdx.x) * kTW;
    const int64_t ty0 = args.tile_y0 + static_cast<int64_t>(blockIdx.y) * kTH;
    const uint64_t seed_key = args.seed_key[blockIdx.z];
    const int c0 = lane * 4;
    const int r0 = warp * kRPT;

    // Grid contents: zero-gradient grids hold raw map_height() values (the
    // octave amplitude is folded in at evaluation); Perlin/generic grids hold
    // amplitude-scaled corner data.
    auto grid_value = [&](uint64_t p, const OctDev& od, float* d) {
        if constexpr (kZg) d[0] = map_height(p);
        else corner_data_packed<KIND>(p, od.amp, od.amp * kMapScale, od.w, d);
    };

    // ---- prologue: every octave's tile corners (and, for general octaves,
    // sampling tables) into shared memory; one barrier for the whole kernel.
    // (a) coarse aligned octaves (<= 32 corners): one warp per octave.
    for (int q = warp; q < args.ngroup[kGProCoarse]; q += kThreads / 32) {
        const OctDev& od = args.oct[args.group[kGProCoarse][q]];
        const int cy = (lane * od.cdiv) >> 16, cx = lane - cy * od.ncx;  // lane / ncx (lane < 32, ncx <= 32)
        if (KIND == kZgPaper && kRPT == 8 && od.cslot >= 0) {
            // kGBlkT octave: per cell (cx, cy) of the tile, the coefficients
            // of its column and row terms (see the per-tile block octaves
            // below) straight from the lanes' corners (lane = cy * ncx + cx):
            //   column  (h00, dx, a*yc, a/ppc),  row  (dy + a*xc, a/ppc)
            // with (xc, yc) the cell-local coordinate of the tile's pixel (0, 0).
            float h = map_height(pack_xy(seed_key + od.oct_key, (tx0 >> od.shift) + cx, (ty0 >> od.shift) + cy));
            h *= od.amp * kMapScale;
            const float h10 = __shfl_down_sync(0xffffffffu, h, 1);
            const float h01 = __shfl_down_sync(0xffffffffu, h, od.ncx);
            const float h11 = __shfl_down_sync(0xffffffffu, h, od.ncx + 1);
            if (cx < od.ncx - 1 && cy < od.ncy - 1) {
                const int mask = od.ppc - 1;
                const float xc = (static_cast<float>((static_cast<int>(tx0) & mask) - (cx << od.shift)) + 0.5f) * od.inv_ppc;
                const float yc = (static_cast<float>((static_cast<int>(ty0) & mask) - (cy << od.shift)) + 0.5f) * od.inv_ppc;
                const float dy = h01 - h, a = (h11 - h10) - dy, ai = a * od.inv_ppc;
                float* base = reinterpret_cast<float*>(smem_raw + smem_grid_end<KIND, LEAN>()) + 1024;
                const int cell = od.cslot * 8 + cy * (od.ncx - 1) + cx;
                reinterpret_cast<float4*>(base)[cell] = make_float4(h, h10 - h, a * yc, ai);
                reinterpret_cast<float2*>(base + 4 * 8 * kMaxCellSlots)[cell] = make_float2(fmaf(a, xc, dy), ai);
            }
        } else if (lane < od.ncx * od.ncy) {
            float d[CH];
            grid_value(pack_xy(seed_key + od.oct_key, (tx0 >> od.shift) + cx, (ty0 >> od.shift) + cy), od, d);
#pragma unroll
            for (int c = 0; c < CH; ++c) grid[c * kGridCap + od.goff + cy * od.pitch + cx] = d[c];
        }
    }
    // (b) aligned power-of-two grids, ppc = 1 .. 16: one slot per ppc with a
    // compile-time shape (FineDev, built by the host planner)
    auto fine_slot = [&](auto sh_c) {
        constexpr int SH = decltype(sh_c)::value;
        const FineDev& fd = args.fine[SH];
        if ((TG_SKIP & 1) || fd.goff < 0) return;
        // ppc >= 4: main block and edge list both sit on the first few warps
        // from fd.rot (rot == erot), the others skip the slot outright
        constexpr int Hm = kTH >> SH, NE = Hm + 1 + (kTW >> SH);
        constexpr int kMainW = Hm >= (8 << SH) ? 8 : (Hm + (1 << SH) - 1) >> SH;
        constexpr int kActW = kMainW > (NE + 31) / 32 ? kMainW : (NE + 31) / 32;
        if (kActW < 8 && ((warp - fd.rot) & 7) >= kActW) return;
        const uint64_t p0 = seed_key + fd.key0 + static_cast<uint64_t>(blockIdx.x) * fd.kx +
                            static_cast<uint64_t>(blockIdx.y) * fd.ky;
        float* g = grid + fd.goff;
        if constexpr (kZg && (SH == 1 || (KIND == kZgPaper && SH >= 2))) {
            // the ppc-2 grid (and the slot-evaluated ppc 4 / 8 / 16 grids) are
            // stored amplitude-scaled (their evaluation reads them as is)
            const float sc = (SH == 1 || fd.blk) ? args.oct[fd.oct].amp * kMapScale : 1.0f;
            fine_grid<SH, CH, true>(g, fd.pitch, p0, warp, lane, tid, fd.rot, grid_value, args.oct[fd.oct], sc);
        } else {
            fine_grid<SH, CH>(g, fd.pitch, p0, warp, lane, tid, fd.rot, grid_value, args.oct[fd.oct]);
        }
    };
    // (generic keeps its aligned grids in the list below: one runtime-shaped
    // copy of the 3-lane corner hash, two lanes with sincos — five
    // specialisations cost more than they save, 324 -> 398 us at config 3)
    if constexpr (KIND != kGeneric) {
        fine_slot(std::integral_constant<int, 0>{});
        fine_slot(std::integral_constant<int, 1>{});
        fine_slot(std::integral_constant<int, 2>{});
        fine_slot(std::integral_constant<int, 3>{});
        fine_slot(std::integral_constant<int, 4>{});
    }
    // (c) everything else with a grid
    for (int q = 0; q < TG_NG(kGProFine, 1); ++q) {
        const OctDev& od = args.oct[args.group[kGProFine][q]];
        const uint64_t base = seed_key + od.oct_key;
        const bool aligned = od.lut_off >= 0;  // power-of-two ppc on the aligned tile grid
        int64_t ix0, iy0;
        int ncx = od.ncx, ncy = od.ncy;
        if (aligned) {
            ix0 = tx0 >> od.shift;
            iy0 = ty0 >> od.shift;
        } else {
            int64_t ixe, iye;
            float t;
            axis_coord(od, args.R, tx0, &ix0, &t);
            axis_coord(od, args.R, ty0, &iy0, &t);
            axis_coord(od, args.R, tx0 + kTW - 1, &ixe, &t);
            axis_coord(od, args.R, ty0 + kTH - 1, &iye, &t);
            ncx = static_cast<int>(ixe - ix0 + 2);  // <= the planned bound
            ncy = static_cast<int>(iye - iy0 + 2);
        }
        if (!LEAN && od.mode == kModeGrid) {
            TabSlot& tb = tabs[od.tslot];
            if (tid < kTW) {
                int64_t i;
                float x;
                axis_coord(od, args.R, tx0 + tid, &i, &x);
                const float sx = smooth<ORDER>(x);
                tb.colI[tid] = static_cast<int32_t>(i - ix0);
                tb.colX[tid] = x;
                tb.colS[tid] = sx;
                tb.colXS[tid] = x * sx;
            } else if (tid < kTW + kTH) {
                const int r = tid - kTW;
                int64_t i;
                float y;
                axis_coord(od, args.R, ty0 + r, &i, &y);
                const float sy = smooth<ORDER>(y);
                tb.rowF[r] = make_float4(y, sy, sy - y, __int_as_float(static_cast<int32_t>(i - iy0)));
            }
        }
        const int pitch = od.pitch;
        float* g = grid + od.goff;
        if (KIND == kGeneric && aligned && od.shift <= 4) {
            const uint64_t p0 = seed_key + od.key0 + static_cast<uint64_t>(blockIdx.x) * od.kx +
                                static_cast<uint64_t>(blockIdx.y) * od.ky;
            fine_grid_rt<CH>(od.shift, g, pitch, p0, warp, lane, tid, q & 7, grid_value, od);
        } else {
            // Any other shape: flat corner list, four hash chains per thread.
            const uint64_t p0 = pack_xy(base, ix0, iy0);
            const int n = ncx * ncy;
            const float rcp = 1.0f / static_cast<float>(ncx);
            for (int i0 = tid; i0 < n; i0 += 4 * kThreads) {
                float d[4][CH];
                int dst[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = min(i0 + u * kThreads, n - 1);
                    const int cy = static_cast<int>((static_cast<float>(i) + 0.5f) * rcp);
                    const int cx = i - cy * ncx;
                    dst[u] = cy * pitch + cx;
                    grid_value(p0 + static_cast<uint64_t>(static_cast<uint32_t>(cx)) * kIxMul +
                                   static_cast<uint64_t>(static_cast<uint32_t>(cy)) * kIyMul,
                               od, d[u]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i0 + u * kThreads < n) {
#pragma unroll
                        for (int c = 0; c < CH; ++c) g[c * kGridCap + dst[u]] = d[u][c];
                    }
            }
        }
    }
    // Generic cells at the fixed in-cell positions of ppc 1 (x = y = 1/2) and
    // ppc 2 (x, y in {1/4, 3/4}): the cell value is linear in its 12 corner
    // values, so it is a fixed weighted sum — weights from the cell itself on
    // one-hot corners (class 0: ppc 1; 1 + 2 iy + ix: ppc 2).
    __shared__ float gwt[KIND == kGeneric ? 5 * 12 : 1];
    if constexpr (KIND == kGeneric) {
        if (tid < 5 * 12) {
            const int cls = tid / 12, k = tid - cls * 12;
            const float px = cls == 0 ? 0.5f : ((cls - 1) & 1) ? 0.75f : 0.25f;
            const float py = cls == 0 ? 0.5f : ((cls - 1) & 2) ? 0.75f : 0.25f;
            float k00[3], k10[3], k01[3], k11[3];  // the one-hot corner data (no local array)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                k00[c] = k == c ? 1.f : 0.f;
                k10[c] = k == 3 + c ? 1.f : 0.f;
                k01[c] = k == 6 + c ? 1.f : 0.f;
                k11[c] = k == 9 + c ? 1.f : 0.f;
            }
            Cell<kGeneric> cw;
            cw.make(k00, k10, k01, k11);
            gwt[tid] = Cell<kGeneric>::eval(cw.row(py, 0.f), px, 0.f, 0.f);
        }
    }
    __syncthreads();

    // ---- evaluation of the thread's 4 x 8 pixels (no barriers) --------------
    float acc[kRPT][4];
    float racc[kRPT];  // per-row terms common to the 4 columns (Perlin/generic block modes)
    // term common to all 32 pixels (zg block modes), starting from the
    // map_height offset of every octave (lattice.cuh)
    float hsum = kMapOffset && KIND != kPerlin ? kMapOffsetUnits * args.hoff : 0.f;
    float cacc[4] = {0.f, 0.f, 0.f, 0.f};  // per-column terms (zg block modes)
#pragma unroll
    for (int r = 0; r < kRPT; ++r) racc[r] = 0.f;

    if constexpr (KIND == kZgPaper) {
        // power-of-two ppc >= 8, all block octaves summed in separated form.
        // With x = x0 + c/ppc, y = y0 + r/ppc (c = 0..3, r = 0..7 the pixel's
        // place in the thread's block) the paper cell
        //   v = h00 + Sx*dx + Sy*(dy + a*x) + y*a*(Sx - x)
        // is  v = [h00 + Sx*dx + (a*y0)*(Sx - x)] + r*[(a/ppc)*(Sx - x)]
        //       + Sy*(dy + a*x0) + c*[Sy*(a/ppc)]
        // i.e. column terms C0(c), C1(c) and row terms R0(r), R1(r) that
        // add up over octaves; the pixels are formed once after the list:
        //   v(c, r) = C0(c) + R0(r) + c*R1(r) + r*C1(c).
        float C0[4] = {0.f, 0.f, 0.f, 0.f}, C1[4] = {0.f, 0.f, 0.f, 0.f}, R0[kRPT], R1[kRPT];
#pragma unroll
        for (int r = 0; r < kRPT; ++r) R0[r] = R1[r] = 0.f;
        const float* lutS = reinterpret_cast<const float*>(args.lut + kLutN4);  // S(x)
        const float* lutD = lutS + kLutN4;                                       // S(x) - x
        if constexpr (kRPT == 8) {
            if (TG_NG(kGBlkT, 8) > 0) {  // uniform per launch
                // ppc >= 32: a 128 x 64 tile spans at most 4 x 2 cells, so in
                // tile coordinates (X, Y) each octave is
                //   v = Cw(X, cr) + Y*C1(X, cr) + Rw(Y, cc) + X*R1(Y, cc)
                // with x = xc + X/ppc, y = yc + Y/ppc inside cell (cc, cr):
                //   Cw = h00 + Sx*dx + (a*yc)*(Sx - x), C1 = (a/ppc)*(Sx - x),
                //   Rw = Sy*(dy + a*xc),                R1 = (a/ppc)*Sy.
                // Cells nest, so every octave's (cc, cr) follows from the
                // ppc-32 cell; the entries are summed over the whole list.
                float* feat = reinterpret_cast<float*>(smem_raw + smem_grid_end<KIND, LEAN>());
                // Threads 0-127 build the column entries of X = tid for both
                // ppc-32 cell rows, threads 128-255 the row entries of
                // Y = tid % 64 for two ppc-32 cell columns; above ppc 32 the
                // two entries share their cell, so the term is computed once.
                // Per octave and entry: one LUT load, one shared load of the
                // cell's coefficients (coarse prologue), 2-3 FFMA.
                const float4* colp = reinterpret_cast<const float4*>(feat + 1024);
                const float2* rowp = reinterpret_cast<const float2*>(feat + 1024 + 4 * 8 * kMaxCellSlots);
                const int tlx = static_cast<int>(tx0), tly = static_cast<int>(ty0);  // (& mask: low bits)
                const int nq = args.ngroup[kGBlkT];
                if (tid < 128) {
                    const int X = tid;
                    float cwA = 0.f, cwB = 0.f, c1A = 0.f, c1B = 0.f;
#pragma unroll
                    for (int q = 0; q < kMaxCellSlots; ++q) {
                        if (q >= nq) break;
                        const BlkTDev& b = args.blkt[q];
                        const int sh = b.shift;
                        const float2 e = __ldg(b.sd + ((tlx + X) & b.mask));  // S, S - x
                        const float4 cp = colp[q * 8 + (X >> sh)];
                        const float tA = fmaf(cp.z, e.y, fmaf(e.x, cp.y, cp.x));
                        cwA += tA;
                        c1A = fmaf(cp.w, e.y, c1A);
                        if (sh == 5) {  // second ppc-32 cell row
                            const float4 cpB = colp[q * 8 + b.ncx1 + (X >> 5)];
                            cwB += fmaf(cpB.z, e.y, fmaf(e.x, cpB.y, cpB.x));
                            c1B = fmaf(cpB.w, e.y, c1B);
                        } else {
                            cwB += tA;
                            c1B = fmaf(cp.w, e.y, c1B);
                        }
                    }
                    feat[X] = cwA;
                    feat[128 + X] = cwB;
                    feat[256 + X] = c1A;
                    feat[384 + X] = c1B;
                } else {
                    const int u = tid - 128, Y = u & 63, ccA = (u >> 6) * 2;
                    float rwA = 0.f, rwB = 0.f, r1A = 0.f, r1B = 0.f;
#pragma unroll
                    for (int q = 0; q < kMaxCellSlots; ++q) {
                        if (q >= nq) break;
                        const BlkTDev& b = args.blkt[q];
                        const int sh = b.shift;
                        const float sy = __ldg(b.sd + ((tly + Y) & b.mask)).x;
                        const int cr = Y >> sh, cc = (ccA << 5) >> sh;
                        const float2 rp = rowp[q * 8 + cr * b.ncx1 + cc];
                        rwA = fmaf(sy, rp.x, rwA);
                        r1A = fmaf(rp.y, sy, r1A);
                        if (sh == 5) {  // second ppc-32 cell column
                            const float2 rpB = rowp[q * 8 + cr * b.ncx1 + cc + 1];
                            rwB = fmaf(sy, rpB.x, rwB);
                            r1B = fmaf(rpB.y, sy, r1B);
                        } else {
                            rwB = fmaf(sy, rp.x, rwB);
                            r1B = fmaf(rp.y, sy, r1B);
                        }
                    }
                    feat[512 + ccA * 64 + Y] = rwA;
                    feat[512 + (ccA + 1) * 64 + Y] = rwB;
                    feat[768 + ccA * 64 + Y] = r1A;
                    feat[768 + (ccA + 1) * 64 + Y] = r1B;
                }
                __syncthreads();
                // the thread's block: X = c0 + j, Y = r0 + r (block-local c = j, r = r)
                const float* fc = feat + (r0 >> 5) * 128 + c0;
                const float* fr = feat + 512 + (c0 >> 5) * 64 + r0;
                const float4 cw4 = *reinterpret_cast<const float4*>(fc);
                const float4 c14 = *reinterpret_cast<const float4*>(fc + 256);
                const float cwa[4] = {cw4.x, cw4.y, cw4.z, cw4.w}, c1a[4] = {c14.x, c14.y, c14.z, c14.w};
                const float fr0 = static_cast<float>(r0), fc0 = static_cast<float>(c0);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    C0[j] = fmaf(fr0, c1a[j], cwa[j]);
                    C1[j] = c1a[j];
                }
#pragma unroll
                for (int r4 = 0; r4 < kRPT; r4 += 4) {
                    const float4 rw4 = *reinterpret_cast<const float4*>(fr + r4);
                    const float4 r14 = *reinterpret_cast<const float4*>(fr + 256 + r4);
                    const float rwa[4] = {rw4.x, rw4.y, rw4.z, rw4.w}, r1a[4] = {r14.x, r14.y, r14.z, r14.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        R0[r4 + i] = fmaf(fc0, r1a[i], rwa[i]);
                        R1[r4 + i] = r1a[i];
                    }
                }
            }
        }
        // ppc 8 / 16 from their fine slots (compile-time shape, amplitude-
        // scaled grids): the same separated-form terms as the list below.
        // Tiles are 128 x 64 aligned, so the thread's block starts at cell
        // offset (c0 & (PPC - 1), r0 & (PPC - 1)).
        auto blk_slot = [&](auto sh_c) {
            constexpr int SH = decltype(sh_c)::value, PPC = 1 << SH;
            constexpr float inv = 1.0f / PPC;
            const FineDev& fd = args.fine[SH];
            if ((TG_SKIP & 4) || !fd.blk) return;
            const int mx = c0 & (PPC - 1), my = r0 & (PPC - 1);
            const float* g = grid + fd.goff + (r0 >> SH) * fd.pitch + (c0 >> SH);
            const float h00 = g[0], h10 = g[1], h01 = g[fd.pitch], h11 = g[fd.pitch + 1];
            const float dx = h10 - h00, dy = h01 - h00, a = (h11 - h10) - dy;
            const float x0 = (static_cast<float>(mx) + 0.5f) * inv, y0 = (static_cast<float>(my) + 0.5f) * inv;
            const float4 sx = __ldg(reinterpret_cast<const float4*>(lutS + PPC + mx));
            const float4 dd = __ldg(reinterpret_cast<const float4*>(lutD + PPC + mx));
            const float sxa[4] = {sx.x, sx.y, sx.z, sx.w}, dda[4] = {dd.x, dd.y, dd.z, dd.w};
            const float ay0 = a * y0, ad = a * inv, k0 = fmaf(a, x0, dy);
            hsum += h00;
#if TG_F2_BLK
            sep_terms(C0, C1, R0, R1, sx, dd, dx, ay0, ad, k0, [&](int r4) {
                return __ldg(reinterpret_cast<const float4*>(lutS + PPC + my + r4));
            });
#else
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                C0[j] = fmaf(dda[j], ay0, fmaf(sxa[j], dx, C0[j]));
                C1[j] = fmaf(dda[j], ad, C1[j]);
            }
#pragma unroll
            for (int r4 = 0; r4 < kRPT; r4 += 4) {
                const float4 sy = __ldg(reinterpret_cast<const float4*>(lutS + PPC + my + r4));
                const float sya[4] = {sy.x, sy.y, sy.z, sy.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    R0[r4 + i] = fmaf(sya[i], k0, R0[r4 + i]);
                    R1[r4 + i] = fmaf(sya[i], ad, R1[r4 + i]);
                }
            }
#endif
        };
        blk_slot(std::integral_constant<int, 4>{});
        blk_slot(std::integral_constant<int, 3>{});
        for (int q = 0; q < TG_NG(kGBlk8, 4); ++q) {
            const OctDev& od = args.oct[args.group[kGBlk8][q]];
            const int sh = od.shift, mask = od.ppc - 1;
            const int xo = static_cast<int>(tx0 & mask) + c0;
            const int yo = static_cast<int>(ty0 & mask) + r0;
            const int mx = xo & mask, my = yo & mask;  // multiples of 4 and 8
            const float* g = grid + od.goff + (yo >> sh) * od.pitch + (xo >> sh);
            const float amp = od.amp * kMapScale;
            const float h00 = amp * g[0], h10 = amp * g[1], h01 = amp * g[od.pitch], h11 = amp * g[od.pitch + 1];
            const float dx = h10 - h00, dy = h01 - h00, a = (h11 - h10) - dy;
            const float inv = od.inv_ppc;  // exact power of two
            const float x0 = (static_cast<float>(mx) + 0.5f) * inv, y0 = (static_cast<float>(my) + 0.5f) * inv;
            const float4 sx = __ldg(reinterpret_cast<const float4*>(lutS + od.ppc + mx));
            const float4 dd = __ldg(reinterpret_cast<const float4*>(lutD + od.ppc + mx));
            const float sxa[4] = {sx.x, sx.y, sx.z, sx.w}, dda[4] = {dd.x, dd.y, dd.z, dd.w};
            const float ay0 = a * y0, ad = a * inv, k0 = fmaf(a, x0, dy);
            hsum += h00;
#if TG_F2_BLK
            sep_terms(C0, C1, R0, R1, sx, dd, dx, ay0, ad, k0, [&](int r4) {
                return __ldg(reinterpret_cast<const float4*>(lutS + od.ppc + my + r4));
            });
#else
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                C0[j] = fmaf(dda[j], ay0, fmaf(sxa[j], dx, C0[j]));
                C1[j] = fmaf(dda[j], ad, C1[j]);
            }
#pragma unroll
            for (int r4 = 0; r4 < kRPT; r4 += 4) {
                const float4 sy = __ldg(reinterpret_cast<const float4*>(lutS + od.ppc + my + r4));
                const float sya[4] = {sy.x, sy.y, sy.z, sy.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    R0[r4 + i] = fmaf(sya[i], k0, R0[r4 + i]);
                    R1[r4 + i] = fmaf(sya[i], ad, R1[r4 + i]);
                }
            }
#endif
        }
        // ppc == 4 in the same separated form.  The thread's 4 columns are one
        // cell (x = 1/8 + c/4); rows 0-3 lie in cell row A, rows 4-7 in B
        // (y = 1/8 + r/4 in A, -7/8 + r/4 in B).  The row terms take each
        // half's own cell; the column terms of B differ from A's by D0, D1,
        // added to rows 4-7 only.
        float D0[4] = {0.f, 0.f, 0.f, 0.f}, D1[4] = {0.f, 0.f, 0.f, 0.f};
        static_assert(kRPT == 8, "ppc-4 blocks assume 8 rows per thread (two cell rows)");
        // slot-evaluated ppc 4 (amplitude-scaled grid, x = 1/8 + c/4: S(x)
        // and S(x) - x as compile-time constants)
        if (!(TG_SKIP & 16) && args.fine[2].blk) {
            const FineDev& fd = args.fine[2];
            const int pitch = fd.pitch;
            const float* g = grid + fd.goff + (r0 >> 2) * pitch + (c0 >> 2);
            const float a0 = g[0], a1 = g[1], b0 = g[pitch], b1 = g[pitch + 1];
            const float e0 = g[2 * pitch], e1 = g[2 * pitch + 1];
            const float dyA = b0 - a0, aA = (b1 - a1) - dyA, dxA = a1 - a0;
            const float dyB = e0 - b0, aB = (e1 - b1) - dyB, dxB = b1 - b0;
            const float qA = 0.25f * aA, qB = 0.25f * aB;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float sj = Ppc4S<ORDER>::S(j), dj = Ppc4S<ORDER>::D(j);
                const float cA = fmaf(0.125f * aA, dj, fmaf(sj, dxA, a0));
                const float cB = fmaf(-0.875f * aB, dj, fmaf(sj, dxB, b0));
                C0[j] += cA;
                D0[j] += cB - cA;
                C1[j] = fmaf(qA, dj, C1[j]);
                D1[j] = fmaf(qB - qA, dj, D1[j]);
            }
            const float kA = fmaf(0.125f, aA, dyA), kB = fmaf(0.125f, aB, dyB);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const float sr = Ppc4S<ORDER>::S(r);
                R0[r] = fmaf(sr, kA, R0[r]);
                R1[r] = fmaf(sr, qA, R1[r]);
                R0[r + 4] = fmaf(sr, kB, R0[r + 4]);
                R1[r + 4] = fmaf(sr, qB, R1[r + 4]);
            }
        }
        for (int q = 0; q < TG_NG(kGBlk4, 16); ++q) {
            const OctDev& od = args.oct[args.group[kGBlk4][q]];
            const float4* L = args.lut + od.lut_off;  // 4 entries: x = 1/8, 3/8, 5/8, 7/8
            const int pitch = od.pitch;
            const float* g = grid + od.goff + (r0 >> 2) * pitch + (c0 >> 2);
            const float amp = od.amp * kMapScale;
            const float a0 = amp * g[0], a1 = amp * g[1];
            const float b0 = amp * g[pitch], b1 = amp * g[pitch + 1];
            const float e0 = amp * g[2 * pitch], e1 = amp * g[2 * pitch + 1];
            const float dyA = b0 - a0, aA = (b1 - a1) - dyA, dxA = a1 - a0;
            const float dyB = e0 - b0, aB = (e1 - b1) - dyB, dxB = b1 - b0;
            const float qA = 0.25f * aA, qB = 0.25f * aB;
            float sv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float4 e = L[j];
                sv[j] = e.y;
                const float cA = fmaf(0.125f * aA, e.z, fmaf(e.y, dxA, a0));
                const float cB = fmaf(-0.875f * aB, e.z, fmaf(e.y, dxB, b0));
                C0[j] += cA;
                D0[j] += cB - cA;
                C1[j] = fmaf(qA, e.z, C1[j]);
                D1[j] = fmaf(qB - qA, e.z, D1[j]);
            }
            const float kA = fmaf(0.125f, aA, dyA), kB = fmaf(0.125f, aB, dyB);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                R0[r] = fmaf(sv[r], kA, R0[r]);
                R1[r] = fmaf(sv[r], qA, R1[r]);
                R0[r + 4] = fmaf(sv[r], kB, R0[r + 4]);
                R1[r + 4] = fmaf(sv[r], qB, R1[r + 4]);
            }
        }
        // column constants of the two cell-row halves, the common term folded in
        float CA[4], CB[4], C1B[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            CA[j] = C0[j] + hsum;
            CB[j] = CA[j] + D0[j];
            C1B[j] = C1[j] + D1[j];
        }
#if TG_F2_FORM
#pragma unroll
        for (int r = 0; r < kRPT; ++r) {
#pragma unroll
            for (int p = 0; p < 2; ++p) {  // column pairs (2p, 2p + 1) in FADD2 / FFMA2
                const float* cc = r >= 4 ? CB : CA;
                const float* c1 = r >= 4 ? C1B : C1;
                float2 v = __fadd2_rn(make_float2(cc[2 * p], cc[2 * p + 1]), make_float2(R0[r], R0[r]));
                if (r) v = __ffma2_rn(make_float2(static_cast<float>(r), static_cast<float>(r)),
                                      make_float2(c1[2 * p], c1[2 * p + 1]), v);
                // column 0 adds 0 * R1 (= v up to the sign of a zero)
                v = __ffma2_rn(make_float2(static_cast<float>(2 * p), static_cast<float>(2 * p + 1)),
                               make_float2(R1[r], R1[r]), v);
                acc[r][2 * p] = v.x;
                acc[r][2 * p + 1] = v.y;
            }
        }
#else
#pragma unroll
        for (int r = 0; r < kRPT; ++r) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float v = (r >= 4 ? CB[j] : CA[j]) + R0[r];
                if (r) v = fmaf(static_cast<float>(r), r >= 4 ? C1B[j] : C1[j], v);
                if (j) v = fmaf(static_cast<float>(j), R1[r], v);
                acc[r][j] = v;
            }
        }
#endif
    } else {
        const float init = KIND == kGeneric ? hsum : 0.f;  // zg separable folds hsum later
#pragma unroll
        for (int r = 0; r < kRPT; ++r)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[r][j] = init;
    }

    if constexpr (KIND == kZgSeparable) {
        // power-of-two ppc >= 8: the 4 x 8 block lies in one cell
        for (int q = 0; q < TG_NG(kGBlk8, 4); ++q) {
            const OctDev& od = args.oct[args.group[kGBlk8][q]];
            const int sh = od.shift, mask = od.ppc - 1;
            const float4* L = args.lut + od.lut_off;
            const int xo = static_cast<int>(tx0 & mask) + c0;
            const int yo = static_cast<int>(ty0 & mask) + r0;
            const float* g = grid + od.goff + (yo >> sh) * od.pitch + (xo >> sh);
            const float amp = od.amp * kMapScale;
            float x[4], sx[4], smx[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float4 e = L[(xo & mask) + j];
                x[j] = e.x;
                sx[j] = e.y;
                smx[j] = e.z;
            }
            zg_cols<KIND, kRPT, true>(acc, cacc, hsum, 0, L + (yo & mask), x, sx, smx, amp * g[0], amp * g[1],
                                      amp * g[od.pitch], amp * g[od.pitch + 1]);
        }
    }
    if constexpr (KIND == kZgSeparable) {
        // ppc == 4: the thread's 4 columns are one cell; rows 0-3 / 4-7 two cell rows
        for (int q = 0; q < TG_NG(kGBlk4, 16); ++q) {
            const OctDev& od = args.oct[args.group[kGBlk4][q]];
            const float4* L = args.lut + od.lut_off;  // 4 entries: x = 1/8, 3/8, 5/8, 7/8
            const int pitch = od.pitch;
            const float* g = grid + od.goff + (r0 >> 2) * pitch + (c0 >> 2);
            const float amp = od.amp * kMapScale;
            float x[4], sx[4], smx[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float4 e = L[j];
                x[j] = e.x;
                sx[j] = e.y;
                smx[j] = e.z;
            }
            const float a0 = amp * g[0], a1 = amp * g[1];
            const float b0 = amp * g[pitch], b1 = amp * g[pitch + 1];
            static_assert(kRPT == 8, "ppc-4 blocks assume 8 rows per thread (two cell rows)");
            const float e0 = amp * g[2 * pitch], e1 = amp * g[2 * pitch + 1];
            zg_cols<KIND, 4, false>(acc, cacc, hsum, 0, L, x, sx, smx, a0, a1, b0, b1);
            zg_cols<KIND, 4, false>(acc, cacc, hsum, 4, L, x, sx, smx, b0, b1, e0, e1);
        }
    }
    if constexpr (KIND == kZgSeparable) {
        // the column and per-thread terms are complete: fold them in so those
        // registers are free for the hashing phases
#pragma unroll
        for (int r = 0; r < kRPT; ++r)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[r][j] += hsum + cacc[j];
    }

    // ppc == 2: columns (0,1) | (2,3) are two cells at x = 0.25, 0.75; rows
    // pair up the same way; 3 corners per corner row.
#if TG_PPC2_WEIGHTS
    // Zero-gradient kinds: every pixel sits at one of the 4 cell positions
    // (x, y) in {1/4, 3/4}^2, so it is a fixed blend of its 4 corners,
    //   v = w00*h00 + w10*h10 + w01*h01 + w11*h11,
    // with compile-time weights (S(1/4), S(3/4) and x*y exact in fp32):
    // 4 FFMA per pixel from the (amp-scaled) corners, no per-cell set-up.
    if constexpr (kZg) {
        for (int q = 0; q < TG_NG(kGBlk2, 32); ++q) {
            const OctDev& od = args.oct[args.group[kGBlk2][q]];
            const int pitch = od.pitch;
            // the grid holds amplitude-scaled heights (fine slot 1)
            const float* g = grid + od.goff + (r0 >> 1) * pitch + (c0 >> 1);
            float t[3];
#pragma unroll
            for (int u = 0; u < 3; ++u) t[u] = g[u];
#pragma unroll
            for (int k = 0; k < kRPT / 2; ++k) {
                const float* gn = g + (k + 1) * pitch;
                float b[3];
#pragma unroll
                for (int u = 0; u < 3; ++u) b[u] = gn[u];
#pragma unroll
#if TG_F2_PPC2
                for (int iy = 0; iy < 2; ++iy)
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        // pixel pair (2 cc, 2 cc + 1) = cell positions ix = 0, 1:
                        // per-lane weights, shared corner (FFMA2, each lane as fmaf)
                        using W = Ppc2W<KIND, ORDER>;
                        float2 a = make_float2(acc[2 * k + iy][2 * cc], acc[2 * k + iy][2 * cc + 1]);
                        a = __ffma2_rn(make_float2(W::w(0, iy, 3), W::w(1, iy, 3)), make_float2(b[cc + 1], b[cc + 1]), a);
                        a = __ffma2_rn(make_float2(W::w(0, iy, 2), W::w(1, iy, 2)), make_float2(b[cc], b[cc]), a);
                        a = __ffma2_rn(make_float2(W::w(0, iy, 1), W::w(1, iy, 1)), make_float2(t[cc + 1], t[cc + 1]), a);
                        a = __ffma2_rn(make_float2(W::w(0, iy, 0), W::w(1, iy, 0)), make_float2(t[cc], t[cc]), a);
                        acc[2 * k + iy][2 * cc] = a.x;
                        acc[2 * k + iy][2 * cc + 1] = a.y;
                    }
#else
                for (int iy = 0; iy < 2; ++iy)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int cc = j >> 1, ix = j & 1;
                        float& a = acc[2 * k + iy][j];
                        a = fmaf(Ppc2W<KIND, ORDER>::w(ix, iy, 3), b[cc + 1], a);
                        a = fmaf(Ppc2W<KIND, ORDER>::w(ix, iy, 2), b[cc], a);
                        a = fmaf(Ppc2W<KIND, ORDER>::w(ix, iy, 1), t[cc + 1], a);
                        a = fmaf(Ppc2W<KIND, ORDER>::w(ix, iy, 0), t[cc], a);
                    }
#endif
#pragma unroll
                for (int u = 0; u < 3; ++u) t[u] = b[u];
            }
        }
    }
    for (int q = 0; q < (kZg ? 0 : TG_NG(kGBlk2, 32)); ++q) {
#else
    for (int q = 0; q < TG_NG(kGBlk2, 32); ++q) {
#endif
        const OctDev& od = args.oct[args.group[kGBlk2][q]];
        const float4 e0 = args.lut[od.lut_off], e1 = args.lut[od.lut_off + 1];
        const int pitch = od.pitch;
        const float sc = kZg ? od.amp * kMapScale : 1.0f;
        const float* g = grid + od.goff + (r0 >> 1) * pitch + (c0 >> 1);
        float t[3][CH];
#pragma unroll
        for (int u = 0; u < 3; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c) t[u][c] = sc * g[c * kGridCap + u];
#pragma unroll
        for (int k = 0; k < kRPT / 2; ++k) {
            const float* gn = g + (k + 1) * pitch;
            float b[3][CH];
#pragma unroll
            for (int u = 0; u < 3; ++u)
#pragma unroll
                for (int c = 0; c < CH; ++c) b[u][c] = sc * gn[c * kGridCap + u];
            Cell<KIND> ca, cb;
            ca.make(t[0], t[1], b[0], b[1]);
            cb.make(t[1], t[2], b[1], b[2]);
#pragma unroll
            for (int rr = 0; rr < 2; ++rr) {
                const float4 f = rr ? e1 : e0;
                const auto ra = ca.row(f.x, f.y);
                const auto rb = cb.row(f.x, f.y);
                const int r = 2 * k + rr;
                acc[r][0] += Cell<KIND>::eval(ra, e0.x, e0.y, e0.w);
                acc[r][1] += Cell<KIND>::eval(ra, e1.x, e1.y, e1.w);
                acc[r][2] += Cell<KIND>::eval(rb, e0.x, e0.y, e0.w);
                acc[r][3] += Cell<KIND>::eval(rb, e1.x, e1.y, e1.w);
            }
#pragma unroll
            for (int u = 0; u < 3; ++u)
#pragma unroll
                for (int c = 0; c < CH; ++c) t[u][c] = b[u][c];
        }
    }
    // ppc == 1 (x = y = 1/2)
    for (int q = 0; q < TG_NG(kGPpc1, 64); ++q) {
        const OctDev& od = args.oct[args.group[kGPpc1][q]];
        const int pitch = od.pitch;
        const float* g = grid + od.goff + r0 * pitch + c0;
        if constexpr (kZg) {
            // every zero-gradient kernel is the mean of its 4 corners
            ppc1_block(acc, 0.25f * (od.amp * kMapScale), [&](int r, float (&h)[5]) {
                const float4 v = *reinterpret_cast<const float4*>(g + r * pitch);
                h[0] = v.x;
                h[1] = v.y;
                h[2] = v.z;
                h[3] = v.w;
                h[4] = g[r * pitch + 4];
            });
        } else if constexpr (KIND == kPerlin) {
            // Perlin at the cell centre: v = (a00 + b10 - b01 - a11)/8 with
            // a = f + g, b = g - f per corner (kernels2d.hpp:163-173 at 1/2)
            auto load = [&](int r, float (&av)[5], float (&bv)[5]) {
                const float* gf = g + r * pitch;
                const float* gg = gf + kGridCap;
                const float4 f4 = *reinterpret_cast<const float4*>(gf);
                const float4 g4 = *reinterpret_cast<const float4*>(gg);
                const float fv[5] = {f4.x, f4.y, f4.z, f4.w, gf[4]};
                const float gv[5] = {g4.x, g4.y, g4.z, g4.w, gg[4]};
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    av[k] = fv[k] + gv[k];
                    bv[k] = gv[k] - fv[k];
                }
            };
            float at[5], bt[5];
            load(0, at, bt);
#pragma unroll
            for (int r = 0; r < kRPT; ++r) {
                float ab[5], bb[5];
                load(r + 1, ab, bb);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    acc[r][j] = fmaf(0.125f, (at[j] + bt[j + 1]) - (bb[j] + ab[j + 1]), acc[r][j]);
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    at[k] = ab[k];
                    bt[k] = bb[k];
                }
            }
        }
    }

    // lattice-point octaves: zg and generic contribute h(ix, iy) exactly,
    // Perlin exactly 0 (SURVEY §8c "exact shortcuts")
    if constexpr (KIND != kPerlin) {
        for (int q = 0; q < TG_NG(kGSub, 2); ++q) {
            const OctDev& od = args.oct[args.group[kGSub][q]];
            const float amp = od.amp * kMapScale;  // exact power-of-two rescale
            // key(gx, gy) = seed*K1 + oct*K2 + (gx*k + k/2)*K3 + (gy*k + k/2)*K4,
            // tile / thread offsets as 32-bit multiples of the per-launch steps
#if TG_SUB_ROWS == 1
            uint64_t X[4];
            X[0] = static_cast<uint64_t>(blockIdx.x * kTW + c0) * od.kx;
#pragma unroll
            for (int j = 1; j < 4; ++j) X[j] = add64(X[j - 1], od.kx);
            uint64_t Y = seed_key + od.key0 + static_cast<uint64_t>(blockIdx.y * kTH + r0) * od.ky;
            const uint64_t dY = od.ky;
#pragma unroll
            for (int r = 0; r < kRPT; ++r) {
                float h[4];
                map_height4(add64(X[0], Y), add64(X[1], Y), add64(X[2], Y), add64(X[3], Y), h);
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[r][j] = fmaf(amp, h[j], acc[r][j]);
                Y = add64(Y, dY);
            }
#else
            // TG_SUB_ROWS rows per step: 4 * TG_SUB_ROWS independent hash
            // chains (the 4-chain form stalls on the IMAD dependency latency)
            const uint64_t kx = od.kx, ky = od.ky;
            uint64_t K = seed_key + od.key0 + static_cast<uint64_t>(blockIdx.y * kTH + r0) * ky +
                         static_cast<uint64_t>(blockIdx.x * kTW + c0) * kx;  // (row r0, column c0)
#pragma unroll
            for (int r = 0; r < kRPT; r += TG_SUB_ROWS) {
                uint64_t p[4 * TG_SUB_ROWS];
#pragma unroll
                for (int i = 0; i < TG_SUB_ROWS; ++i) {
                    p[4 * i] = i ? add64(p[4 * (i - 1)], ky) : K;
#pragma unroll
                    for (int j = 1; j < 4; ++j) p[4 * i + j] = add64(p[4 * i + j - 1], kx);
                }
                float h[4 * TG_SUB_ROWS];
                map_heightN<4 * TG_SUB_ROWS>(p, h);
#pragma unroll
#if TG_F2_SUB
                for (int i = 0; i < TG_SUB_ROWS; ++i) fma_pairs(acc[r + i], h + 4 * i, amp);
#else
                for (int i = 0; i < TG_SUB_ROWS; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[r + i][j] = fmaf(amp, h[4 * i + j], acc[r + i][j]);
#endif
                if (r + TG_SUB_ROWS < kRPT) K = add64(p[4 * (TG_SUB_ROWS - 1)], ky);
            }
#endif
        }
    }

    // everything else: Perlin/generic cells, general (non-dividing/fractional) octaves
    for (int q = 0; q < (LEAN ? 0 : args.ngroup[kGGen]); ++q) {
        const OctDev& od = args.oct[args.group[kGGen][q]];
        const int mode = od.mode;
        const uint64_t base = seed_key + od.oct_key;
        // grids of zg octaves hold raw heights: scale at load
        const float gscale = kZg ? od.amp * kMapScale : 1.0f;

        if (mode == kModeBlock) {
            // Perlin/generic, power-of-two ppc >= 4: 4 columns share one cell
            const int sh = od.shift, mask = od.ppc - 1;
            const float4* L = args.lut + od.lut_off;
            const int xo = static_cast<int>(tx0 & mask) + c0;
            const int yo = static_cast<int>(ty0 & mask) + r0;
            const int pitch = od.pitch;
            const float* g = grid + od.goff + (xo >> sh);
            float x[4], sx[4], xs[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float4 e = L[(xo & mask) + j];
                x[j] = e.x;
                sx[j] = e.y;
                xs[j] = e.w;
            }
            // row terms: the column-independent one to the row accumulator,
            // the rest 3 FFMA per pixel (Perlin {x, sx, xs}, generic Horner in x)
            // column pairs (0, 1), (2, 3) in packed fp32x2 (FFMA2: one issue slot
            // per pair, each lane rounded as fmaf — bit-identical)
            const float2 x2[2] = {make_float2(x[0], x[1]), make_float2(x[2], x[3])};
            const float2 sx2[2] = {make_float2(sx[0], sx[1]), make_float2(sx[2], sx[3])};
            const float2 xs2[2] = {make_float2(xs[0], xs[1]), make_float2(xs[2], xs[3])};
            auto accum = [&](int r, const typename Cell<KIND>::Row& row) {
                if constexpr (KIND == kPerlin) {
                    racc[r] += row.a0;
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        float2 a = make_float2(acc[r][2 * p], acc[r][2 * p + 1]);
                        a = __ffma2_rn(x2[p], make_float2(row.a1, row.a1), a);
                        a = __ffma2_rn(sx2[p], make_float2(row.a2, row.a2), a);
                        a = __ffma2_rn(xs2[p], make_float2(row.a3, row.a3), a);
                        acc[r][2 * p] = a.x;
                        acc[r][2 * p + 1] = a.y;
                    }
                } else if constexpr (KIND == kGeneric) {
                    racc[r] += row.r0;
#pragma unroll
                    for (int p = 0; p < 2; ++p) {
                        float2 t = __ffma2_rn(make_float2(row.r3, row.r3), x2[p], make_float2(row.r2, row.r2));
                        t = __ffma2_rn(t, x2[p], make_float2(row.r1, row.r1));
                        const float2 a = __ffma2_rn(t, x2[p], make_float2(acc[r][2 * p], acc[r][2 * p + 1]));
                        acc[r][2 * p] = a.x;
                        acc[r][2 * p + 1] = a.y;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[r][j] += Cell<KIND>::eval(row, x[j], sx[j], xs[j]);
                }
            };
            auto load_cell = [&](Cell<KIND>& cell, int ry) {
                const int key = ry * pitch;
                float k00[CH], k10[CH], k01[CH], k11[CH];
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    k00[c] = gscale * g[c * kGridCap + key];
                    k10[c] = gscale * g[c * kGridCap + key + 1];
                    k01[c] = gscale * g[c * kGridCap + key + pitch];
                    k11[c] = gscale * g[c * kGridCap + key + pitch + 1];
                }
                cell.make(k00, k10, k01, k11);
            };
            Cell<KIND> cell;
            if (od.ppc >= kRPT) {
                // the thread's rows lie in one cell: corners once per octave;
                // its rows are LUT entries (yo & mask) + r without wrap-around
                load_cell(cell, yo >> sh);
                const float4* Ly = L + (yo & mask);
#pragma unroll
                for (int r = 0; r < kRPT; ++r) {
                    const float4 f = Ly[r];
                    accum(r, cell.row(f.x, f.y));
                }
            } else {
                int last = -1;
#pragma unroll
                for (int r = 0; r < kRPT; ++r) {
                    const int yr = yo + r;
                    const int ry = yr >> sh;
                    const float4 f = L[yr & mask];
                    if (ry != last) {
                        load_cell(cell, ry);
                        last = ry;
                    }
                    accum(r, cell.row(f.x, f.y));
                }
            }
            continue;
        }

        if (mode == kModeGrid) {
            const TabSlot& tb = tabs[od.tslot];
            const float* g = grid + od.goff;
            const int pitch = od.pitch;
            if constexpr (KIND == kGeneric) {
                if (od.cls == kClsFast && (od.shift == 0 || od.shift == 1)) {
                    // fixed positions: value = sum of the 12 corner values with the
                    // class weights (gwt), no per-pixel cell set-up.  The thread's
                    // corner rows are swept top to bottom (each corner value read
                    // once per thread: 12 scattered loads per pixel were 4-way
                    // bank-conflicted and saturated the shared-memory pipe).
                    const int cx0 = tb.colI[c0];
                    const int cy0 = __float_as_int(tb.rowF[r0].w);
                    if (od.shift == 0) {
                        float w[12];
#pragma unroll
                        for (int k = 0; k < 12; ++k) w[k] = gwt[k] * gscale;
                        // corners (cx0 .. cx0 + 4) of a row, 3 channels
                        auto load_row = [&](int cy, float (&v)[3][5]) {
                            const int key = cy * pitch + cx0;
#pragma unroll
                            for (int c = 0; c < 3; ++c) {
                                const float* q = g + c * kGridCap + key;
                                const float4 t = *reinterpret_cast<const float4*>(q);  // cx0 % 4 == 0
                                v[c][0] = t.x, v[c][1] = t.y, v[c][2] = t.z, v[c][3] = t.w;
                                v[c][4] = q[4];
                            }
                        };
                        float top[3][5], bot[3][5];
                        load_row(cy0, top);
#pragma unroll
                        for (int r = 0; r < kRPT; ++r) {
                            load_row(cy0 + r + 1, bot);
                            // v_j = A_j + B_(j+1): A_i = sum_c w_c top_c[i] + w_(6+c) bot_c[i] (corner
                            // column i as a cell's left corners), B_i the same with w_(3+c), w_(9+c)
                            // (as its right corners); column pairs (0, 1), (2, 3) in FFMA2
                            float2 A[2], B[2];
                            float B4 = 0.f;
#pragma unroll
                            for (int p = 0; p < 2; ++p) {
                                A[p] = B[p] = make_float2(0.f, 0.f);
#pragma unroll
                                for (int c = 0; c < 3; ++c) {
                                    const float2 tp = make_float2(top[c][2 * p], top[c][2 * p + 1]);
                                    const float2 bp = make_float2(bot[c][2 * p], bot[c][2 * p + 1]);
                                    A[p] = __ffma2_rn(make_float2(w[c], w[c]), tp, A[p]);
                                    A[p] = __ffma2_rn(make_float2(w[6 + c], w[6 + c]), bp, A[p]);
                                    B[p] = __ffma2_rn(make_float2(w[3 + c], w[3 + c]), tp, B[p]);
                                    B[p] = __ffma2_rn(make_float2(w[9 + c], w[9 + c]), bp, B[p]);
                                }
                            }
#pragma unroll
                            for (int c = 0; c < 3; ++c) {
                                B4 = fmaf(w[3 + c], top[c][4], B4);
                                B4 = fmaf(w[9 + c], bot[c][4], B4);
                            }
                            const float Bn[4] = {B[0].y, B[1].x, B[1].y, B4};
#pragma unroll
                            for (int p = 0; p < 2; ++p) {
                                const float2 a = __fadd2_rn(make_float2(acc[r][2 * p], acc[r][2 * p + 1]), A[p]);
                                acc[r][2 * p] = a.x + Bn[2 * p];
                                acc[r][2 * p + 1] = a.y + Bn[2 * p + 1];
                            }
#pragma unroll
                            for (int c = 0; c < 3; ++c)
#pragma unroll
                                for (int i = 0; i < 5; ++i) top[c][i] = bot[c][i];
                        }
                    } else {
                        // ppc 2: corner columns cx0 .. cx0 + 2, cell rows of 2 pixel rows;
                        // the pixel's class is its parity in the cell (even origins)
                        auto load_row = [&](int cy, float (&v)[3][3]) {
                            const int key = cy * pitch + cx0;
#pragma unroll
                            for (int c = 0; c < 3; ++c)
#pragma unroll
                                for (int i = 0; i < 3; ++i) v[c][i] = gscale * g[c * kGridCap + key + i];
                        };
                        float top[3][3], bot[3][3];
                        load_row(cy0, top);
#pragma unroll
                        for (int cr = 0; cr < kRPT / 2; ++cr) {
                            load_row(cy0 + cr + 1, bot);
#pragma unroll
                            for (int rr = 0; rr < 2; ++rr)
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    const float* w = gwt + 12 * (1 + 2 * rr + (j & 1));
                                    const int cx = j >> 1;
                                    float v = 0.f;
#pragma unroll
                                    for (int c = 0; c < 3; ++c) {
                                        v = fmaf(w[c], top[c][cx], v);
                                        v = fmaf(w[3 + c], top[c][cx + 1], v);
                                        v = fmaf(w[6 + c], bot[c][cx], v);
                                        v = fmaf(w[9 + c], bot[c][cx + 1], v);
                                    }
                                    acc[2 * cr + rr][j] += v;
                                }
#pragma unroll
                            for (int c = 0; c < 3; ++c)
#pragma unroll
                                for (int i = 0; i < 3; ++i) top[c][i] = bot[c][i];
                        }
                    }
                    continue;
                }
            }
            float x[4], sx[4], xs[4];
            int cxi[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                x[j] = tb.colX[c0 + j];
                sx[j] = tb.colS[c0 + j];
                xs[j] = tb.colXS[c0 + j];
                cxi[j] = tb.colI[c0 + j];
            }
            const bool one_cell = cxi[0] == cxi[3];
            int last_key = -1;
            Cell<KIND> cell;
#pragma unroll
            for (int r = 0; r < kRPT; ++r) {
                const float4 f = tb.rowF[r0 + r];
                const float y = f.x, sy = f.y;
                const int ry = __float_as_int(f.w) * pitch;
                if (one_cell) {
                    const int key = ry + cxi[0];
                    if (key != last_key) {
                        float k00[CH], k10[CH], k01[CH], k11[CH];
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            k00[c] = gscale * g[c * kGridCap + key];
                            k10[c] = gscale * g[c * kGridCap + key + 1];
                            k01[c] = gscale * g[c * kGridCap + key + pitch];
                            k11[c] = gscale * g[c * kGridCap + key + pitch + 1];
                        }
                        cell.make(k00, k10, k01, k11);
                        last_key = key;
                    }
                    const auto row = cell.row(y, sy);
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[r][j] += Cell<KIND>::eval(row, x[j], sx[j], xs[j]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int key = ry + cxi[j];
                        float k00[CH], k10[CH], k01[CH], k11[CH];
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            k00[c] = gscale * g[c * kGridCap + key];
                            k10[c] = gscale * g[c * kGridCap + key + 1];
                            k01[c] = gscale * g[c * kGridCap + key + pitch];
                            k11[c] = gscale * g[c * kGridCap + key + pitch + 1];
                        }
                        Cell<KIND> cj;
                        cj.make(k00, k10, k01, k11);
                        acc[r][j] += Cell<KIND>::eval(cj.row(y, sy), x[j], sx[j], xs[j]);
                    }
                }
            }
            continue;
        }

        // kModeDirect: corners hashed per pixel, coordinates per thread.
        const float amp = od.amp;
        if constexpr (kZg) {
            if (od.cls == kClsFast && od.ppc == 1) {
                ppc1_block(acc, 0.25f, [&](int r, float (&h)[5]) {
#pragma unroll
                    for (int k = 0; k < 5; ++k)
                        corner_data<KIND>(base, tx0 + c0 + k, ty0 + r0 + r, amp, od.w, &h[k]);
                });
                continue;
            }
        }
        {
            int64_t cxi[4];
            float x[4], sx[4], xs[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                axis_coord(od, args.R, tx0 + c0 + j, &cxi[j], &x[j]);
                sx[j] = smooth<ORDER>(x[j]);
                xs[j] = x[j] * sx[j];
            }
#pragma unroll 1
            for (int r = 0; r < kRPT; ++r) {
                int64_t iy;
                float y;
                axis_coord(od, args.R, ty0 + r0 + r, &iy, &y);
                const float sy = smooth<ORDER>(y);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float k00[CH], k10[CH], k01[CH], k11[CH];
                    corner_data<KIND>(base, cxi[j], iy, amp, od.w, k00);
                    corner_data<KIND>(base, cxi[j] + 1, iy, amp, od.w, k10);
                    corner_data<KIND>(base, cxi[j], iy + 1, amp, od.w, k01);
                    corner_data<KIND>(base, cxi[j] + 1, iy + 1, amp, od.w, k11);
                    Cell<KIND> cj;
                    cj.make(k00, k10, k01, k11);
                    const float v = Cell<KIND>::eval(cj.row(y, sy), x[j], sx[j], xs[j]);
#pragma unroll
                    for (int rr = 0; rr < kRPT; ++rr)
                        if (rr == r) acc[rr][j] += v;
                }
            }
        }
    }

    // ---- single fp32 store of the finished tile ----------------------------
    // Programmatic dependent launch: this grid may have started while the
    // previous kernel on the stream was finishing (the hashing above touches no
    // global memory but the immutable row LUT); wait for it to complete before
    // writing the output (write-after-write / write-after-read on `out`).
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t lx0 = tx0 + c0 - args.ox;
    const int64_t ly0 = ty0 + r0 - args.oy;
#if TG_TMA_STORE
    // Every tile (right / bottom edge tiles included: the tensor copy clips
    // rows and columns outside the window) is staged in shared memory (the corner grids are
    // dead by now) and written by the TMA engine, one 128 x 8 box per warp
    // (cp.async.bulk.tensor, SASS UTMASTG) from the host-encoded tensor map of
    // the output window.
    // Box start coordinates must be non-negative (negative ones fault), so a
    // warp whose rows start left of / above the window stores directly.
    const bool tma_warp = args.tma && tx0 >= args.ox && ty0 + r0 >= args.oy;
    if (args.tma) {  // uniform per launch
        if (args.stage_pairs) {
            // warp w stages over ppc-1 corner rows 7.76w .. 7.76w + 7.75 (pitch
            // 132): only warps w-1 and w read those, so w waits for w-1 alone
            if (warp < kThreads / 32 - 1) asm volatile("bar.arrive %0, 64;" ::"r"(warp + 1) : "memory");
            if (warp > 0) asm volatile("bar.sync %0, 64;" ::"r"(warp) : "memory");
        } else {
            __syncthreads();  // every warp is done reading the corner grids
        }
    }
    if (tma_warp) {
        float* stage = grid + r0 * kTW;
#pragma unroll
        for (int r = 0; r < kRPT; ++r) {
            const float rr_ = kZg ? 0.f : racc[r];  // zg never uses the row accumulators
            float w[4] = {acc[r][0], acc[r][1], acc[r][2], acc[r][3]};
            if constexpr (!kZg)
#pragma unroll
                for (int j = 0; j < 4; ++j) w[j] += rr_;
            if (!LEAN && args.epilogue) {
                const float invR = static_cast<float>(1.0 / args.R);
                const float vv = (static_cast<float>(ty0 + r0 + r) + 0.5f) * invR;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float u = (static_cast<float>(tx0 + c0 + j) + 0.5f) * invR;
                    const float phase =
                        args.epilogue == 1 ? u : sqrtf((u - 0.5f) * (u - 0.5f) + (vv - 0.5f) * (vv - 0.5f));
                    w[j] = sinf(fmaf(args.tex_freq2pi, phase, args.tex_gain * w[j]));
                }
            }
            *reinterpret_cast<float4*>(stage + r * kTW + c0) = make_float4(w[0], w[1], w[2], w[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
            const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                    reinterpret_cast<uint64_t>(&tmap)),
                "r"(static_cast<int32_t>(tx0 - args.ox)), "r"(static_cast<int32_t>(ty0 + r0 - args.oy)),
                "r"(static_cast<int32_t>(blockIdx.z)), "r"(sa)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        return;
    }
#endif
    float* row = out + static_cast<int64_t>(blockIdx.z) * args.map_stride + ly0 * args.ld + lx0;
    const bool vec_ok = ((lx0 & 3) == 0) && ((args.ld & 3) == 0) && ((args.map_stride & 3) == 0) &&
                        ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && lx0 >= 0 &&
                        lx0 + 4 <= args.width;
#pragma unroll
    for (int r = 0; r < kRPT; ++r, row += args.ld) {
        const int64_t ly = ly0 + r;
        if (ly < 0 || ly >= args.height) continue;
        float v0 = acc[r][0], v1 = acc[r][1], v2 = acc[r][2], v3 = acc[r][3];
        if constexpr (!kZg) {  // zg never uses the row accumulators
            v0 += racc[r];
            v1 += racc[r];
            v2 += racc[r];
            v3 += racc[r];
        }
        if (!LEAN && args.epilogue) {
            // texture::render (texture.hpp:57-68) fused into the store:
            // sin(2 pi f phase + gain * noise), (u, v) pixel centres in [0, 1)
            const float invR = static_cast<float>(1.0 / args.R);
            const float vv = (static_cast<float>(ty0 + r0 + r) + 0.5f) * invR;
            float w[4] = {v0, v1, v2, v3};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float u = (static_cast<float>(tx0 + c0 + j) + 0.5f) * invR;
                const float phase = args.epilogue == 1 ? u : sqrtf((u - 0.5f) * (u - 0.5f) + (vv - 0.5f) * (vv - 0.5f));
                w[j] = sinf(fmaf(args.tex_freq2pi, phase, args.tex_gain * w[j]));
            }
            v0 = w[0];
            v1 = w[1];
            v2 = w[2];
            v3 = w[3];
        }
        if (vec_ok) {
            *reinterpret_cast<float4*>(row) = make_float4(v0, v1, v2, v3);
        } else {
            const float v[4] = {v0, v1, v2, v3};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t lx = lx0 + j;
                if (lx >= 0 && lx < args.width) row[j] = v[j];
            }
        }
    }
}

// ---- launch ------------------------------------------------------------------

// Tensor map of the output window for the TMA tile store: dims (width,
// height, maps), fp32, box 128 x 8 x 1 (one warp's rows).  Needs a 16-byte
// aligned base and row / map strides that are multiples of 16 bytes; the
// caller falls back to vector stores otherwise.
static bool encode_out_map(const FbmArgs& a, float* out, CUtensorMap* m) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    if (!encode) return false;
    if ((reinterpret_cast<uintptr_t>(out) & 15) || (a.ld & 3) || a.width < 1 || a.height < 1 ||
        a.width > (int64_t(1) << 31) || a.height > (int64_t(1) << 31) || a.ld < a.width)
        return false;
    const int64_t mstride = a.n_maps > 1 ? a.map_stride : a.ld * a.height;
    if ((mstride & 3) || mstride < a.ld * a.height) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(a.width), static_cast<cuuint64_t>(a.height),
                                static_cast<cuuint64_t>(a.n_maps)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(a.ld) * 4, static_cast<cuuint64_t>(mstride) * 4};
    const cuuint32_t box[3] = {kTW, kRPT, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, out, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int KIND, int ORDER, bool LEAN>
static cudaError_t launch_v(const FbmArgs& a0, float* out, cudaStream_t st) {
    constexpr size_t smem = smem_bytes<KIND, LEAN>();
    auto kern = fbm2d_kernel<KIND, ORDER, LEAN>;
    static PerDeviceOnce configured;
    cudaError_t e = configured.run([&] {
        return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    });
    if (e != cudaSuccess) return e;
    FbmArgs a = a0;
    CUtensorMap m;
    a.tma = TG_TMA_STORE && encode_out_map(a, out, &m) ? 1 : 0;
    if (!a.tma) memset(&m, 0, sizeof(m));
    constexpr int TH = kTH;
    const int64_t tiles_x = (a.ox + a.width - a.tile_x0 + kTW - 1) / kTW;
    const int64_t tiles_y = (a.oy + a.height - a.tile_y0 + TH - 1) / TH;
    dim3 grid(static_cast<unsigned>(tiles_x), static_cast<unsigned>(tiles_y),
              static_cast<unsigned>(a.n_maps));
#if TG_PDL
    // programmatic stream serialisation: consecutive generation launches
    // overlap one grid's tail with the next grid's compute (the kernel waits
    // on the previous grid before its stores)
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, kern, a, m, out);
#else
    kern<<<grid, kThreads, smem, st>>>(a, m, out);
    return cudaGetLastError();
#endif
}

template <int KIND, int ORDER>
static cudaError_t launch_t(const FbmArgs& a, float* out, cudaStream_t st) {
    // Zero-gradient kinds take the lean kernel at 4 CTAs/SM (64 registers)
    // whenever the plan allows: measured 90.5 -> 84.0 us (separable) and
    // 100.9 -> 94.5 us (paper) at the config-2 shape.
    if constexpr (KIND == kZgSeparable || KIND == kZgPaper)
        if (a.epilogue == 0 && a.ngroup[kGGen] == 0) return launch_v<KIND, ORDER, true>(a, out, st);
    return launch_v<KIND, ORDER, false>(a, out, st);
}

int fbm2d_tile_h() { return kTH; }

cudaError_t simplex2d_launch(const FbmArgs& a, float* out, cudaStream_t st);
cudaError_t perm2d_launch(int order, const FbmArgs& a, float* out, cudaStream_t st);

cudaError_t fbm2d_launch(int kind, int order, const FbmArgs& a, float* out, cudaStream_t st) {
    if (kind == kOpenSimplex) return simplex2d_launch(a, out, st);
    if (kind == kPerlinPerm) return perm2d_launch(order, a, out, st);
    if (order == 5) {
        switch (kind) {
            case kZgPaper: return launch_t<kZgPaper, 5>(a, out, st);
            case kZgSeparable: return launch_t<kZgSeparable, 5>(a, out, st);
            case kGeneric: return launch_t<kGeneric, 5>(a, out, st);
            default: return launch_t<kPerlin, 5>(a, out, st);
        }
    }
    switch (kind) {
        case kZgPaper: return launch_t<kZgPaper, 3>(a, out, st);
        case kZgSeparable: return launch_t<kZgSeparable, 3>(a, out, st);
        case kGeneric: return launch_t<kGeneric, 3>(a, out, st);
        default: return launch_t<kPerlin, 3>(a, out, st);
    }
}

}  // namespace tg
