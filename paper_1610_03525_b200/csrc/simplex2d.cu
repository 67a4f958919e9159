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

// Hashes on demand (fine octaves: more vertices than pixels in a tile).
struct HashGrad {
    uint64_t base;
    int64_t xb, yb;
    __device__ __forceinline__ HashGrad(uint64_t b, double xbd, double ybd) {
        base = b;
        xb = __double2ll_rd(xbd);
        yb = __double2ll_rd(ybd);
    }
    __device__ __forceinline__ uint32_t operator()(int a, int b) const { return grad_index(base, xb + a, yb + b); }
};

// Per-CTA table of the gradient indices of every vertex the tile can touch
// (coarse octaves: a few vertices shared by many pixels), filled once.
struct TableGrad {
    const uint8_t* row0;  // entry of vertex (xsb, ysb)
    int nx;
    __device__ __forceinline__ TableGrad(const uint8_t* t, int n, double bx, double by, double xbd, double ybd) {
        row0 = t + exact_int32(ybd - by) * n + exact_int32(xbd - bx);
        nx = n;
    }
    __device__ __forceinline__ uint32_t operator()(int a, int b) const { return row0[b * nx + a]; }
};

// (2 - d^2)^4 (g . d) for the vertex at offset (a, b) from (xsb, ysb):
// d = d0 - (a, b) - (a + b) * squish; the radial term clamps at zero, so the
// gradient is always read (branch-free).  g from the 8-entry vector table.
template <class G>
__device__ __forceinline__ float contrib(const G& grad, const float2* gv, int a, int b, float fa, float fb,
                                         float dx0, float dy0) {
    constexpr float S = static_cast<float>(kSquish);
    const float s = (fa + fb) * S;
    const float dx = dx0 - fa - s, dy = dy0 - fb - s;
    float attn = fmaxf(2.0f - dx * dx - dy * dy, 0.0f);
    const float2 g = gv[grad(a, b)];
    attn *= attn;
    return attn * attn * fmaf(g.x, dx, g.y * dy);
}

// Skew, floor and region decisions in fp64 (the oracle's order of
// operations); contributions in fp32, summed in the order v1, v2, v3, extra.
template <class G>
__device__ __forceinline__ float opensimplex(const G& grad, const float2* gv, double x, double y,
                                             double xb, double yb, double xs, double ys) {
    const double sq = (xb + yb) * kSquish;
    const double xins = xs - xb, yins = ys - yb;
    const double in_sum = xins + yins;
    const float dx0 = static_cast<float>(x - (xb + sq));
    const float dy0 = static_cast<float>(y - (yb + sq));
    const bool upper = in_sum > 1.0;
    // v3 = (c, c); extra vertex (ea, eb)
    int ea, eb;
    if (!upper) {
        const double zins = 1.0 - in_sum;
        const bool edge = zins > xins || zins > yins;
        ea = edge ? (xins > yins ? 1 : -1) : 1;
        eb = edge ? (xins > yins ? -1 : 1) : 1;
    } else {
        const double zins = 2.0 - in_sum;
        const bool edge = zins < xins || zins < yins;
        ea = edge ? (xins > yins ? 2 : 0) : 0;
        eb = edge ? (xins > yins ? 0 : 2) : 0;
    }
    const int c = upper ? 1 : 0;
    const float fc = upper ? 1.0f : 0.0f;
    float v = contrib(grad, gv, 1, 0, 1.0f, 0.0f, dx0, dy0);
    v += contrib(grad, gv, 0, 1, 0.0f, 1.0f, dx0, dy0);
    v += contrib(grad, gv, c, c, fc, fc, dx0, dy0);
    v += contrib(grad, gv, ea, eb, static_cast<float>(ea), static_cast<float>(eb), dx0, dy0);
    return v * (1.0f / 47.0f);
}

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
    __shared__ float2 gv[8];  // (+-5, +-2) / (+-2, +-5): bit 0 swaps, bits 1 / 2 negate x / y
    if (threadIdx.x < 8) {
        const int i = threadIdx.x;
        const float gx = (i & 1) ? 2.0f : 5.0f, gy = (i & 1) ? 5.0f : 2.0f;
        gv[i] = make_float2((i & 2) ? -gx : gx, (i & 4) ? -gy : gy);
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
            const double fr = od.ratio;  // freq / R, IEEE division on the host
            const double u = __dmul_rn(__dadd_rn(gx, 0.5), fr);
            const double v = __dmul_rn(__dadd_rn(gy, 0.5), fr);
            const double so = (u + v) * kStretch;
            const double xs = u + so, ys = v + so;
            const double xb = floor(xs), yb = floor(ys);
            float nv;
            if (od.mode)
                nv = opensimplex(TableGrad(gtab + od.goff, od.ncx, plan[o].bx, plan[o].by, xb, yb), gv, u, v, xb,
                                 yb, xs, ys);
            else
                nv = opensimplex(HashGrad(seed_key + od.oct_key, xb, yb), gv, u, v, xb, yb, xs, ys);
            acc = fmaf(od.amp, nv, acc);
        }
        const int64_t ly = ly0 + r, lx = lx0 + j;
        if (ly >= 0 && ly < args.height && lx >= 0 && lx < args.width) out_map[ly * args.ld + lx] = acc;
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
