// fbm2d.cu — fused-octave 2D fBm kernel for sm_100a.
//
// Replaces the octave loop of generate_into_with_source
// (terrain/fbm.hpp:541-628) and its render paths render_zg_fast (231-312),
// render_generic_fast (321-379), render_perlin_fast (384-455) and
// render_general (460-527).  One CTA owns a 128 x TH pixel tile whose
// accumulators stay in registers across ALL octaves; the map is written once
// (4 B/pixel) instead of the reference's read-modify-write of a double buffer
// per octave (fbm.hpp:187,193).
//
// Per octave the CTA
//   (A) builds column/row sampling tables (cell index, x, S(x)) and hashes the
//       tile's unique lattice corners once into shared memory;
//   (B) every thread evaluates its 4 x RPT pixels from the shared corners with
//       the cell polynomial factorised per (cell, row):
//         zg paper     v = c0 + sx*c1 + x*c2      (kernels2d.hpp:62-76)
//         zg separable v = c0 + sx*c1
//         perlin       v = a0 + x*a1 + sx*a2 + x*sx*a3   (kernels2d.hpp:163-173)
//         generic      v = ((r3*x + r2)*x + r1)*x + r0    (kernels2d.hpp:124-134)
// Octaves whose samples sit exactly on lattice points (kClsSubInt) skip the
// tables: each pixel hashes its one corner in registers.
//
// Every pixel's arithmetic is a function of (config, global pixel) only, so
// any window / tile decomposition reproduces the same bits (fbm.hpp:7-8).
#include <cuda_runtime.h>

#include "fbm_params.h"
#include "lattice.cuh"

namespace tg {

constexpr int kThreads = 256;
constexpr int kTW = 128;  // 32 lanes x 4 columns

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

// Corner data of one lattice point, already scaled like the reference's
// render paths: zg/generic heights x amp (fbm.hpp:270,349), Perlin unit
// gradients x amp (409-420), generic gradients unscaled (348).
template <int KIND>
__device__ __forceinline__ void corner_data(uint64_t base, int64_t ix, int64_t iy, float amp,
                                            float w, int zero, float* d) {
    if (zero) {
#pragma unroll
        for (int c = 0; c < Traits<KIND>::kCh; ++c) d[c] = 0.f;
        return;
    }
    if constexpr (KIND == kZgPaper || KIND == kZgSeparable) {
        d[0] = amp * corner_height(base, ix, iy);
    } else if constexpr (KIND == kPerlin) {
        float c, s;
        corner_unit_gradient(base, ix, iy, &c, &s);
        d[0] = amp * c;
        d[1] = amp * s;
    } else {
        d[0] = amp * corner_height(base, ix, iy);
        corner_gradient(base, ix, iy, w, &d[1], &d[2]);
    }
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
    float f0, g0, f1, g1, f2, g2, f3, g3;  // corners 00, 10, 01, 11
    __device__ __forceinline__ void make(const float* k00, const float* k10, const float* k01,
                                         const float* k11) {
        f0 = k00[0]; g0 = k00[1];
        f1 = k10[0]; g1 = k10[1];
        f2 = k01[0]; g2 = k01[1];
        f3 = k11[0]; g3 = k11[1];
    }
    struct Row { float a0, a1, a2, a3; };
    __device__ __forceinline__ Row row(float y, float sy) const {
        // lerp_y of the two x-lerped ramps (kernels2d.hpp:163-173), expanded in
        // the column features {1, x, sx, x*sx}.
        const float ym = y - 1.f;
        const float p0 = g0 * y, p1 = f0, p2 = fmaf(g1 - g0, y, -f1), p3 = f1 - f0;
        const float q0 = g2 * ym, q1 = f2, q2 = fmaf(g3 - g2, ym, -f3), q3 = f3 - f2;
        return {fmaf(sy, q0 - p0, p0), fmaf(sy, q1 - p1, p1), fmaf(sy, q2 - p2, p2),
                fmaf(sy, q3 - p3, p3)};
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

template <int RPT>
struct SmemFixed {
    float colX[kTW], colS[kTW], colXS[kTW];
    int64_t colI[kTW];
    float rowY[8 * RPT], rowS[8 * RPT];
    int64_t rowI[8 * RPT];
};

template <int RPT>
constexpr int grid_capacity() {
    return ((kTW + 2) * (8 * RPT + 2) + 63) / 64 * 64;
}

template <int KIND, int RPT>
constexpr size_t smem_bytes() {
    return sizeof(SmemFixed<RPT>) + sizeof(float) * Traits<KIND>::kCh * grid_capacity<RPT>();
}

template <int KIND, int ORDER, int RPT>
__global__ void __launch_bounds__(kThreads)
fbm2d_kernel(const __grid_constant__ FbmArgs args, float* __restrict__ out) {
    constexpr int TH = 8 * RPT;
    constexpr int CH = Traits<KIND>::kCh;
    constexpr int CAP = grid_capacity<RPT>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SmemFixed<RPT>& S = *reinterpret_cast<SmemFixed<RPT>*>(smem_raw);
    float* grid = reinterpret_cast<float*>(smem_raw + sizeof(SmemFixed<RPT>));

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int64_t tx0 = args.tile_x0 + static_cast<int64_t>(blockIdx.x) * kTW;
    const int64_t ty0 = args.tile_y0 + static_cast<int64_t>(blockIdx.y) * TH;
    const int map = blockIdx.z;
    const uint64_t seed_key = args.seed_key[map];
    const int c0 = lane * 4;
    const int r0 = warp * RPT;

    float acc[RPT][4];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[r][j] = 0.f;

    for (int o = 0; o < args.octaves; ++o) {
        const OctDev& od = args.oct[o];
        const uint64_t base = seed_key + od.oct_key;
        const float amp = od.amp;

        if (od.cls == kClsSubInt) {
            // Samples on lattice points: zg and generic contribute h(ix, iy)
            // exactly, Perlin exactly 0 (SURVEY §8c "exact shortcuts").
            if (KIND == kPerlin || args.zero) continue;
            const int64_t k = od.k, half = od.k >> 1;
            uint64_t X[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                X[j] = static_cast<uint64_t>((tx0 + c0 + j) * k + half) * kIxMul;
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                const uint64_t Y =
                    base + static_cast<uint64_t>((ty0 + r0 + r) * k + half) * kIyMul;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    acc[r][j] = fmaf(amp, height_from_hash(mix64(X[j] + Y)), acc[r][j]);
            }
            continue;
        }

        // ---- (A) sampling tables + unique corners of this tile -------------
        __syncthreads();  // previous octave finished reading shared memory
        if (tid < kTW) {
            int64_t i;
            float t;
            axis_coord(od, args.R, tx0 + tid, &i, &t);
            const float s = smooth<ORDER>(t);
            S.colI[tid] = i;
            S.colX[tid] = t;
            S.colS[tid] = s;
            S.colXS[tid] = t * s;
        } else if (tid - kTW < TH) {
            const int r = tid - kTW;
            int64_t i;
            float t;
            axis_coord(od, args.R, ty0 + r, &i, &t);
            S.rowI[r] = i;
            S.rowY[r] = t;
            S.rowS[r] = smooth<ORDER>(t);
        }
        int64_t ix0, iy0, ixe, iye;
        float dummy;
        axis_coord(od, args.R, tx0, &ix0, &dummy);
        axis_coord(od, args.R, tx0 + kTW - 1, &ixe, &dummy);
        axis_coord(od, args.R, ty0, &iy0, &dummy);
        axis_coord(od, args.R, ty0 + TH - 1, &iye, &dummy);
        const int64_t ncx64 = ixe - ix0 + 2, ncy64 = iye - iy0 + 2;
        const bool direct = ncx64 * ncy64 > CAP;
        const int ncx = static_cast<int>(ncx64), ncy = static_cast<int>(ncy64);
        if (!direct) {
            for (int cy = warp; cy < ncy; cy += kThreads / 32)
                for (int cx = lane; cx < ncx; cx += 32) {
                    float d[CH];
                    corner_data<KIND>(base, ix0 + cx, iy0 + cy, amp, od.w, args.zero, d);
#pragma unroll
                    for (int c = 0; c < CH; ++c) grid[c * CAP + cy * ncx + cx] = d[c];
                }
        }
        __syncthreads();

        // ---- (B) evaluate the thread's 4 x RPT pixels ----------------------
        float x[4], sx[4], xs[4];
        int64_t cxi[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            x[j] = S.colX[c0 + j];
            sx[j] = S.colS[c0 + j];
            xs[j] = S.colXS[c0 + j];
            cxi[j] = S.colI[c0 + j];
        }
        const bool one_cell = cxi[0] == cxi[3];
        int last_key = -1;
        Cell<KIND> cell;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const float y = S.rowY[r0 + r];
            const float sy = S.rowS[r0 + r];
            const int64_t iy = S.rowI[r0 + r];
            if (!direct) {
                const int ry = static_cast<int>(iy - iy0);
                if (one_cell) {
                    const int key = ry * ncx + static_cast<int>(cxi[0] - ix0);
                    if (key != last_key) {
                        float k00[CH], k10[CH], k01[CH], k11[CH];
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            k00[c] = grid[c * CAP + key];
                            k10[c] = grid[c * CAP + key + 1];
                            k01[c] = grid[c * CAP + key + ncx];
                            k11[c] = grid[c * CAP + key + ncx + 1];
                        }
                        cell.make(k00, k10, k01, k11);
                        last_key = key;
                    }
                    const auto row = cell.row(y, sy);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        acc[r][j] += Cell<KIND>::eval(row, x[j], sx[j], xs[j]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int key = ry * ncx + static_cast<int>(cxi[j] - ix0);
                        float k00[CH], k10[CH], k01[CH], k11[CH];
#pragma unroll
                        for (int c = 0; c < CH; ++c) {
                            k00[c] = grid[c * CAP + key];
                            k10[c] = grid[c * CAP + key + 1];
                            k01[c] = grid[c * CAP + key + ncx];
                            k11[c] = grid[c * CAP + key + ncx + 1];
                        }
                        Cell<KIND> cj;
                        cj.make(k00, k10, k01, k11);
                        acc[r][j] += Cell<KIND>::eval(cj.row(y, sy), x[j], sx[j], xs[j]);
                    }
                }
            } else {
                // Cells too spread out for the shared grid (sub-pixel general
                // octaves): hash the four corners per pixel.
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float k00[CH], k10[CH], k01[CH], k11[CH];
                    corner_data<KIND>(base, cxi[j], iy, amp, od.w, args.zero, k00);
                    corner_data<KIND>(base, cxi[j] + 1, iy, amp, od.w, args.zero, k10);
                    corner_data<KIND>(base, cxi[j], iy + 1, amp, od.w, args.zero, k01);
                    corner_data<KIND>(base, cxi[j] + 1, iy + 1, amp, od.w, args.zero, k11);
                    Cell<KIND> cj;
                    cj.make(k00, k10, k01, k11);
                    acc[r][j] += Cell<KIND>::eval(cj.row(y, sy), x[j], sx[j], xs[j]);
                }
            }
        }
    }

    // ---- single fp32 store of the finished tile ----------------------------
    float* base_out = out + static_cast<int64_t>(map) * args.map_stride;
    const int64_t gx0 = tx0 + c0;
    const int64_t lx0 = gx0 - args.ox;
    const bool vec_ok = ((lx0 & 3) == 0) && ((args.ld & 3) == 0) &&
                        ((reinterpret_cast<uintptr_t>(base_out) & 15) == 0) && lx0 >= 0 &&
                        lx0 + 4 <= args.width;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int64_t ly = ty0 + r0 + r - args.oy;
        if (ly < 0 || ly >= args.height) continue;
        float* row = base_out + ly * args.ld;
        if (vec_ok) {
            __stcs(reinterpret_cast<float4*>(row + lx0),
                   make_float4(acc[r][0], acc[r][1], acc[r][2], acc[r][3]));
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t lx = lx0 + j;
                if (lx >= 0 && lx < args.width) row[lx] = acc[r][j];
            }
        }
    }
}

// ---- launch ------------------------------------------------------------------

template <int KIND, int ORDER, int RPT>
static cudaError_t launch_t(const FbmArgs& a, float* out, cudaStream_t st) {
    constexpr size_t smem = smem_bytes<KIND, RPT>();
    auto kern = fbm2d_kernel<KIND, ORDER, RPT>;
    static bool configured = false;  // benign race: idempotent attribute set
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    constexpr int TH = 8 * RPT;
    const int64_t tiles_x = (a.ox + a.width - a.tile_x0 + kTW - 1) / kTW;
    const int64_t tiles_y = (a.oy + a.height - a.tile_y0 + TH - 1) / TH;
    dim3 grid(static_cast<unsigned>(tiles_x), static_cast<unsigned>(tiles_y),
              static_cast<unsigned>(a.n_maps));
    kern<<<grid, kThreads, smem, st>>>(a, out);
    return cudaGetLastError();
}

int fbm2d_tile_h() { return 64; }

cudaError_t fbm2d_launch(int kind, int order, const FbmArgs& a, float* out, cudaStream_t st) {
    constexpr int RPT = 8;
    if (order == 5) {
        switch (kind) {
            case kZgPaper: return launch_t<kZgPaper, 5, RPT>(a, out, st);
            case kZgSeparable: return launch_t<kZgSeparable, 5, RPT>(a, out, st);
            case kGeneric: return launch_t<kGeneric, 5, RPT>(a, out, st);
            default: return launch_t<kPerlin, 5, RPT>(a, out, st);
        }
    }
    switch (kind) {
        case kZgPaper: return launch_t<kZgPaper, 3, RPT>(a, out, st);
        case kZgSeparable: return launch_t<kZgSeparable, 3, RPT>(a, out, st);
        case kGeneric: return launch_t<kGeneric, 3, RPT>(a, out, st);
        default: return launch_t<kPerlin, 3, RPT>(a, out, st);
    }
}

}  // namespace tg
