// simplex2d.cu — OpenSimplex 2D fBm (the paper's third comparison baseline,
// PAPER.md:234-236; absent from the reference: parity unpinned,
// checked against the restated oracle/oracle.c or_opensimplex).
//
// Geometry of the 2014 OpenSimplex algorithm: stretch (x, y) by
// (x + y)(1/sqrt(3) - 1)/2 onto a square lattice, split the rhombus into two
// triangles, sum (2 - d^2)^4 (g . d) over the two shared vertices, the
// triangle's own corner and one extra vertex, divide by 47.  Gradients are
// the 8 vectors (+-5, +-2), (+-2, +-5) chosen by the lattice hash (lane
// TG_LANE_SIMPLEX), so chunks stay stateless like every other method.  Sample
// positions are u = (g + 0.5) * (freq / R) (render_general's position,
// fbm.hpp:468, with the ratio formed once per octave).
// Lattice selection (skew, floors, region) in fp64 with the oracle's
// operations, the four contributions in fp32.  256 threads x 4 x 8 pixels,
// octaves outermost, one fp32 store per pixel.
// Coarse octaves read gradient indices from a per-CTA shared-memory table of
// every vertex the tile can touch (hashed once per CTA); fine octaves hash
// per lookup.  Both give the same index, so the choice never changes a pixel.
#include <cuda_runtime.h>

#include "devattr.h"
#include "fbm_params.h"
#include "lattice.cuh"

namespace tg {
namespace {

constexpr uint64_t kSimplexLane = 0x8EBC6AF09C88C6E3ULL;
constexpr double kStretch = -0.211324865405187117745425609749;  // (1/sqrt(3) - 1)/2
constexpr double kSquish = 0.366025403784438646763723170753;    // (sqrt(3) - 1)/2

// Gradient index of lattice vertex (xsv, ysv) = top 3 bits of its hash
// (the final fmix64 xorshift leaves the high word alone).
__device__ __forceinline__ uint32_t grad_index(uint64_t base, int64_t xsv, int64_t ysv) {
    uint32_t lo, hi;
    mix64_pre(pack_xy(base, xsv, ysv) ^ kMapLane(kSimplexLane), lo, hi);
    return hi >> 29;
}

// integral v, |v| < 2^31: the integer sits in the low mantissa word of v + 1.5*2^52
__device__ __forceinline__ int exact_int32(double v) {
    return __double2loint(v + 6755399441055744.0);
}

// (2 - d^2)^4 (g . d) of one vertex, d = d0 - (a + (a + b) S, b + (a + b) S)
// with the displacement offsets given and gi its gradient index (table or
// hash); the radial term clamps at zero, so the gradient is always read.
__device__ __forceinline__ float contrib_at(const float2* gv, uint32_t gi, float ox, float oy, float dx0, float dy0,
                                            float v) {
    const float dx = dx0 - ox, dy = dy0 - oy;
    float attn = fmaxf(fmaf(-dy, dy, fmaf(-dx, dx, 2.0f)), 0.0f);
    const float2 g = gv[gi];
    attn *= attn;
    return fmaf(attn * attn, fmaf(g.x, dx, g.y * dy), v);
}

// The six extra vertices of the region logic (OpenSimplex 2014): upper edge
// (2,0) / (0,2), upper interior (0,0), lower edge (1,-1) / (-1,1), lower
// interior (1,1) — displacement offsets and the integer offsets.
struct ExtraCase {
    float ox, oy;
    int a, b;
};

constexpr int kTW = 128, kTH = 64, kThreads = 256;
constexpr int kTableMargin = 6;           // vertices beyond the tile's stretched range
constexpr int kTableMaxBytes = 96 * 1024;  // per CTA, all table octaves together

// Stretched-coordinate range of a tile: xs = u + (u + v) * kStretch with
// kStretch < 0, so xs is largest at (u1, v0) and smallest at (u0, v1); ys
// symmetric.  Table size bound: spans + margin (host and device agree).
__host__ __device__ inline void table_dims(double fr, int* nx, int* ny) {
    const double a = 1.0 + kStretch, b = -kStretch;  // 0.7887, 0.2113
    *nx = static_cast<int>(ceil((kTW * a + kTH * b) * fr)) + 2 * kTableMargin;
    *ny = static_cast<int>(ceil((kTH * a + kTW * b) * fr)) + 2 * kTableMargin;
}

struct TabPlan {
    double bx, by;  // table origin (integral)
};

// One octave for 4 consecutive pixels of a row (rows and octaves are rolled
// loops around it: one unrolled body per mode keeps the kernel small — the
// fully unrolled 4 x 8 body stalled 44 % on instruction fetch).
// Lattice selection in fp64 with the oracle's operations (u, v, the skew, the
// two floors, xins / yins / in_sum and the region comparisons), so every pixel
// picks the oracle's vertices; the offsets from the cell origin in fp32 via
// dx0 = xins + in_sum * squish (the oracle's x - (xsb + (xsb + ysb) squish)).
template <bool kTable>
__device__ __forceinline__ void os_octave4(float (&acc)[4], const float2* gv, const ExtraCase* ext, double fr, float amp,
                                           const uint8_t* tab, int nx, double bx, double by, uint64_t base,
                                           const double (&gx)[4], double gy) {
    constexpr float S = static_cast<float>(kSquish);
    const double v = __dmul_rn(gy, fr);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const double u = __dmul_rn(gx[j], fr);
        const double so = (u + v) * kStretch;
        const double xs = u + so, ys = v + so;
        const double xb = floor(xs), yb = floor(ys);
        const double xins = xs - xb, yins = ys - yb;
        const double in_sum = xins + yins;
        const bool upper = in_sum > 1.0;
        const double zins = (upper ? 2.0 : 1.0) - in_sum;
        // branch-free region: the four comparisons, then one case index (a
        // divergent branch per pixel cost both paths; per-value selects ~23
        // instructions): the extra vertex's offsets come from a shared table
        const bool edge = upper ? (zins < xins || zins < yins) : (zins > xins || zins > yins);
        const bool xgt = xins > yins;
        const int cs = (upper ? 0 : 3) + (edge ? (xgt ? 0 : 1) : 2);
        const ExtraCase ec = ext[cs];
        constexpr float C1 = 1.0f + 2.0f * S;
        const float fc = upper ? C1 : 0.0f;  // (c, c) vertex displacement
        const float xf = static_cast<float>(xins), yf = static_cast<float>(yins);
        const float sf = (xf + yf) * S;
        const float dx0 = xf + sf, dy0 = yf + sf;
        float nv;
        if (kTable) {
            const uint8_t* r0 = tab + exact_int32(yb - by) * nx + exact_int32(xb - bx);
            nv = contrib_at(gv, r0[1], 1.0f + S, S, dx0, dy0, 0.0f);
            nv = contrib_at(gv, r0[nx], S, 1.0f + S, dx0, dy0, nv);
            nv = contrib_at(gv, r0[upper ? nx + 1 : 0], fc, fc, dx0, dy0, nv);
            nv = contrib_at(gv, r0[ec.b * nx + ec.a], ec.ox, ec.oy, dx0, dy0, nv);
        } else {
            const int64_t xi = __double2ll_rd(xb), yi = __double2ll_rd(yb);
            const int c = upper ? 1 : 0;
            nv = contrib_at(gv, grad_index(base, xi + 1, yi), 1.0f + S, S, dx0, dy0, 0.0f);
            nv = contrib_at(gv, grad_index(base, xi, yi + 1), S, 1.0f + S, dx0, dy0, nv);
            nv = contrib_at(gv, grad_index(base, xi + c, yi + c), fc, fc, dx0, dy0, nv);
            nv = contrib_at(gv, grad_index(base, xi + ec.a, yi + ec.b), ec.ox, ec.oy, dx0, dy0, nv);
        }
        acc[j] = fmaf(amp, nv * (1.0f / 47.0f), acc[j]);
    }
}

__global__ void __launch_bounds__(kThreads)
simplex2d_kernel(const __grid_constant__ FbmArgs args, float* __restrict__ out) {
    extern __shared__ uint8_t gtab[];
    __shared__ TabPlan plan[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t tx0 = args.tile_x0 + static_cast<int64_t>(blockIdx.x) * kTW;
    const int64_t ty0 = args.tile_y0 + static_cast<int64_t>(blockIdx.y) * kTH;
    const uint64_t seed_key = args.seed_key[blockIdx.z];
    // table octaves (host plan: oct[o].mode != 0, goff = byte offset, ncx/ncy)
    if (threadIdx.x < args.octaves && args.oct[threadIdx.x].mode) {
        const OctDev& od = args.oct[threadIdx.x];
        const double fr = od.ratio;
        const double u0 = __dmul_rn(__dadd_rn(static_cast<double>(tx0), 0.5), fr);
        const double v0 = __dmul_rn(__dadd_rn(static_cast<double>(ty0), 0.5), fr);
        const double xs_min = u0 + (u0 + (v0 + kTH * fr)) * kStretch;
        const double ys_min = v0 + ((u0 + kTW * fr) + v0) * kStretch;
        plan[threadIdx.x] = {floor(xs_min) - kTableMargin, floor(ys_min) - kTableMargin};
    }
    __shared__ ExtraCase ext[6];
    if (threadIdx.x < 6) {
        constexpr int ea[6] = {2, 0, 0, 1, -1, 1}, eb[6] = {0, 2, 0, -1, 1, 1};
        const int i = threadIdx.x;
        const float s = static_cast<float>(ea[i] + eb[i]) * static_cast<float>(kSquish);
        ext[i] = {static_cast<float>(ea[i]) + s, static_cast<float>(eb[i]) + s, ea[i], eb[i]};
    }
    __shared__ float2 gv[8];  // (+-5, +-2) / (+-2, +-5): bit 0 swaps, bits 1 / 2 negate x / y
    if (threadIdx.x < 8) {
        const int i = threadIdx.x;
        const float gxv = (i & 1) ? 2.0f : 5.0f, gyv = (i & 1) ? 5.0f : 2.0f;
        gv[i] = make_float2((i & 2) ? -gxv : gxv, (i & 4) ? -gyv : gyv);
    }
    __syncthreads();
    for (int o = 0; o < args.octaves; ++o) {
        const OctDev& od = args.oct[o];
        if (!od.mode) continue;
        const uint64_t base = seed_key + od.oct_key;
        uint8_t* t = gtab + od.goff;
        const int64_t bx = __double2ll_rd(plan[o].bx), by = __double2ll_rd(plan[o].by);
        for (int j = warp; j < od.ncy; j += kThreads / 32)  // one warp per table row
            for (int i = lane; i < od.ncx; i += 32)
                t[j * od.ncx + i] = static_cast<uint8_t>(grad_index(base, bx + i, by + j));
    }
    __syncthreads();
    const int c0 = lane * 4, r0 = warp * 8;
    double gx[4];  // pixel centres g + 0.5 (exact)
#pragma unroll
    for (int j = 0; j < 4; ++j) gx[j] = static_cast<double>(tx0 + c0 + j) + 0.5;
    const int64_t lx0 = tx0 + c0 - args.ox;
    float* out_map = out + static_cast<int64_t>(blockIdx.z) * args.map_stride;
#pragma unroll 1
    for (int r = 0; r < 8; ++r) {
        const double gy = static_cast<double>(ty0 + r0 + r) + 0.5;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
        for (int o = 0; o < args.octaves; ++o) {
            const OctDev& od = args.oct[o];
            if (od.mode)
                os_octave4<true>(acc, gv, ext, od.ratio, od.amp, gtab + od.goff, od.ncx, plan[o].bx, plan[o].by, 0, gx, gy);
            else
                os_octave4<false>(acc, gv, ext, od.ratio, od.amp, nullptr, 0, 0.0, 0.0, seed_key + od.oct_key, gx, gy);
        }
        const int64_t ly = ty0 + r0 + r - args.oy;
        if (ly >= 0 && ly < args.height) {
            float* row = out_map + ly * args.ld;
            if (lx0 >= 0 && lx0 + 4 <= args.width && ((reinterpret_cast<uintptr_t>(row + lx0) & 15) == 0)) {
                *reinterpret_cast<float4*>(row + lx0) = make_float4(acc[0], acc[1], acc[2], acc[3]);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (lx0 + j >= 0 && lx0 + j < args.width) row[lx0 + j] = acc[j];
            }
        }
    }
}

}  // namespace

cudaError_t simplex2d_launch(const FbmArgs& a, float* out, cudaStream_t st) {
    // Plan: an octave gets a per-CTA gradient table when its tile touches
    // fewer vertices than the 4 x 8192 per-pixel lookups would hash.
    FbmArgs p = a;
    int bytes = 0;
    for (int o = 0; o < p.octaves; ++o) {
        OctDev& od = p.oct[o];
        od.mode = 0;
        const double fr = od.freq / p.R;
        od.ratio = fr;
        int nx, ny;
        table_dims(fr, &nx, &ny);
        const int64_t n = static_cast<int64_t>(nx) * ny;
        if (n < 4 * kTW * kTH && bytes + n <= kTableMaxBytes) {
            od.mode = 1;
            od.ncx = nx;
            od.ncy = ny;
            od.goff = bytes;
            bytes += static_cast<int>((n + 15) / 16 * 16);
        }
    }
    static PerDeviceOnce attr;
    cudaError_t e = attr.run([] {
        return cudaFuncSetAttribute(simplex2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTableMaxBytes);
    });
    if (e != cudaSuccess) return e;
    const int64_t tiles_x = (p.ox + p.width - p.tile_x0 + kTW - 1) / kTW;
    const int64_t tiles_y = (p.oy + p.height - p.tile_y0 + kTH - 1) / kTH;
    dim3 grid(static_cast<unsigned>(tiles_x), static_cast<unsigned>(tiles_y), static_cast<unsigned>(p.n_maps));
    simplex2d_kernel<<<grid, kThreads, bytes, st>>>(p, out);
    return cudaGetLastError();
}

}  // namespace tg
