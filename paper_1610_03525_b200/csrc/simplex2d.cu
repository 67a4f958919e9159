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
// Skew, floor and region decisions run in fp64 (as the oracle), the four
// contributions in fp32.  256 threads x 4 x 8 pixels, one fp32 store.
#include <cuda_runtime.h>

#include "fbm_params.h"
#include "lattice.cuh"

namespace tg {
namespace {

constexpr uint64_t kSimplexLane = 0x8EBC6AF09C88C6E3ULL;
constexpr double kStretch = -0.211324865405187117745425609749;  // (1/sqrt(3) - 1)/2
constexpr double kSquish = 0.366025403784438646763723170753;    // (sqrt(3) - 1)/2

// (2 - d^2)^4 * (g . d) for lattice vertex (xsv, ysv); gradient index = top
// 3 bits of the hash (the final fmix64 xorshift leaves the high word alone).
__device__ __forceinline__ float contrib(uint64_t base, int64_t xsv, int64_t ysv, float dx, float dy) {
    float attn = 2.0f - dx * dx - dy * dy;
    if (attn <= 0.0f) return 0.0f;
    uint32_t lo, hi;
    mix64_pre(pack_xy(base, xsv, ysv) ^ kSimplexLane, lo, hi);
    const uint32_t i = hi >> 29;
    const float gx = (i & 1u) ? 2.0f : 5.0f, gy = (i & 1u) ? 5.0f : 2.0f;
    const float sx = (i & 2u) ? -gx : gx, sy = (i & 4u) ? -gy : gy;
    attn *= attn;
    return attn * attn * fmaf(sx, dx, sy * dy);
}

__device__ __forceinline__ float opensimplex(uint64_t base, double x, double y) {
    const double so = (x + y) * kStretch;
    const double xs = x + so, ys = y + so;
    int64_t xsb = __double2ll_rd(xs), ysb = __double2ll_rd(ys);
    const double sq = static_cast<double>(xsb + ysb) * kSquish;
    const double xins = xs - static_cast<double>(xsb), yins = ys - static_cast<double>(ysb);
    const double in_sum = xins + yins;
    float dx0 = static_cast<float>(x - (static_cast<double>(xsb) + sq));
    float dy0 = static_cast<float>(y - (static_cast<double>(ysb) + sq));
    constexpr float S = static_cast<float>(kSquish);
    float v = contrib(base, xsb + 1, ysb, dx0 - 1.0f - S, dy0 - S);
    v += contrib(base, xsb, ysb + 1, dx0 - S, dy0 - 1.0f - S);
    int64_t xe, ye;
    float dxe, dye;
    if (in_sum <= 1.0) {
        const double zins = 1.0 - in_sum;
        if (zins > xins || zins > yins) {
            if (xins > yins) {
                xe = xsb + 1; ye = ysb - 1; dxe = dx0 - 1.0f; dye = dy0 + 1.0f;
            } else {
                xe = xsb - 1; ye = ysb + 1; dxe = dx0 + 1.0f; dye = dy0 - 1.0f;
            }
        } else {
            xe = xsb + 1; ye = ysb + 1; dxe = dx0 - 1.0f - 2.0f * S; dye = dy0 - 1.0f - 2.0f * S;
        }
    } else {
        const double zins = 2.0 - in_sum;
        if (zins < xins || zins < yins) {
            if (xins > yins) {
                xe = xsb + 2; ye = ysb; dxe = dx0 - 2.0f - 2.0f * S; dye = dy0 - 2.0f * S;
            } else {
                xe = xsb; ye = ysb + 2; dxe = dx0 - 2.0f * S; dye = dy0 - 2.0f - 2.0f * S;
            }
        } else {
            xe = xsb; ye = ysb; dxe = dx0; dye = dy0;
        }
        xsb += 1;
        ysb += 1;
        dx0 = dx0 - 1.0f - 2.0f * S;
        dy0 = dy0 - 1.0f - 2.0f * S;
    }
    v += contrib(base, xsb, ysb, dx0, dy0);
    v += contrib(base, xe, ye, dxe, dye);
    return v * (1.0f / 47.0f);
}

constexpr int kTW = 128, kTH = 64, kThreads = 256;

__global__ void __launch_bounds__(kThreads)
simplex2d_kernel(const __grid_constant__ FbmArgs args, float* __restrict__ out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t tx0 = args.tile_x0 + static_cast<int64_t>(blockIdx.x) * kTW;
    const int64_t ty0 = args.tile_y0 + static_cast<int64_t>(blockIdx.y) * kTH;
    const uint64_t seed_key = args.seed_key[blockIdx.z];
    const int c0 = lane * 4, r0 = warp * 8;
    const int64_t lx0 = tx0 + c0 - args.ox;
    const int64_t ly0 = ty0 + r0 - args.oy;
    float* out_map = out + static_cast<int64_t>(blockIdx.z) * args.map_stride;
    // one pixel at a time, octaves innermost (the evaluation has data-dependent
    // branches; a register array indexed by a rolled loop would spill)
#pragma unroll 1
    for (int p = 0; p < 32; ++p) {
        const int r = p >> 2, j = p & 3;
        const double gx = static_cast<double>(tx0 + c0 + j), gy = static_cast<double>(ty0 + r0 + r);
        float acc = 0.f;
        for (int o = 0; o < args.octaves; ++o) {
            const OctDev& od = args.oct[o];
            const double fr = __ddiv_rn(od.freq, args.R);  // uniform: hoisted by the compiler
            const double u = __dmul_rn(__dadd_rn(gx, 0.5), fr);
            const double v = __dmul_rn(__dadd_rn(gy, 0.5), fr);
            acc = fmaf(od.amp, opensimplex(seed_key + od.oct_key, u, v), acc);
        }
        const int64_t ly = ly0 + r, lx = lx0 + j;
        if (ly >= 0 && ly < args.height && lx >= 0 && lx < args.width) out_map[ly * args.ld + lx] = acc;
    }
}

}  // namespace

cudaError_t simplex2d_launch(const FbmArgs& a, float* out, cudaStream_t st) {
    const int64_t tiles_x = (a.ox + a.width - a.tile_x0 + kTW - 1) / kTW;
    const int64_t tiles_y = (a.oy + a.height - a.tile_y0 + kTH - 1) / kTH;
    dim3 grid(static_cast<unsigned>(tiles_x), static_cast<unsigned>(tiles_y), static_cast<unsigned>(a.n_maps));
    simplex2d_kernel<<<grid, kThreads, 0, st>>>(a, out);
    return cudaGetLastError();
}

}  // namespace tg
