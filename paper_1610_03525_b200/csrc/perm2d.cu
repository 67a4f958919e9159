// perm2d.cu — classic permutation-table Perlin gradient-noise fBm (BASELINE
// config 3's "permutation table of 256 from seed, 8 unit gradients").  The
// reference deliberately hashes gradient angles instead (
// its perlin3/perlin5 run in fbm2d.cu, pinned), so this method is new and
// parity unpinned: checked against the restatement in oracle/oracle.c
// (or_perm_gradient).  Definition: include/polyterrain_b200.h
// TG_METHOD_PERLIN_PERM.
//
// Per CTA (128 x 64 tile, 256 threads, 4 x 8 pixels per thread) the seed's
// table is built in shared memory: thread i hashes key_i, and a bitonic sort
// of the (key, index) pairs gives the permutation (no sequential shuffle), then P and the
// gradient of every table entry (the 8 unit vectors at k * 45 degrees) are
// laid out twice (512 entries) so that P[a + iy] needs no wrap.  Octaves run
// outermost: cell index and position per column / row (the fast path's
// x = (r + 0.5) / ppc, render_general's ((g + 0.5) / R) * freq in IEEE fp64
// for the rest, lattice-point octaves contribute exactly 0), then per pixel
// 4 gradient loads and the reference's Perlin cell (kernels2d.hpp:163-173).
#include <cuda_runtime.h>

#include "fbm_params.h"
#include "lattice.cuh"
#include "../../include/polyterrain_b200.h"

namespace tg {
namespace {

constexpr int kTW = 128, kTH = 64, kThreads = 256;

template <int ORDER>
__device__ __forceinline__ float fade(float t) {
    if constexpr (ORDER == 5) return t * t * t * fmaf(t, fmaf(6.f, t, -15.f), 10.f);  // kernels2d.hpp:26-38
    else return t * t * fmaf(-2.f, t, 3.f);
}

// Cell index and in-cell position of global coordinate g for octave od.
__device__ __forceinline__ void cell_coord(const OctDev& od, double R, int64_t g, int64_t* i, float* t) {
    if (od.cls == kClsFast) {
        int64_t q, r;
        if (od.shift >= 0) {
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
        *t = (static_cast<float>(r) + 0.5f) * od.inv_ppc;
    } else {
        const double u = __dmul_rn(__ddiv_rn(__dadd_rn(static_cast<double>(g), 0.5), R), od.freq);
        const int64_t q = __double2ll_rd(u);
        *i = q;
        *t = static_cast<float>(__dsub_rn(u, static_cast<double>(q)));
    }
}

// ppc = 1 << SH in {1, 2}: the thread's 4 x 8 pixels cover NCX x NCY cells;
// the corner rows are swept top to bottom keeping the previous row's
// gradients, so each corner gradient is read once ((NCX + 1) x (NCY + 1)
// reads instead of 4 per pixel), and each cell factorises as in the ppc >= 4
// path.
template <int SH, int ORDER>
__device__ __forceinline__ void perm_small(float (&acc)[8][4], const OctDev& od, const uint8_t* P2, const float2* GP,
                                           int64_t gx0, int64_t gy0, int ox, int oy, float amp) {
    constexpr int NCX = 4 >> SH, NCY = 8 >> SH, CPC = 1 << SH, RPC = 1 << SH;
    const int64_t ix0 = gx0 >> SH, iy0 = gy0 >> SH;
    int a[NCX + 1];
#pragma unroll
    for (int i = 0; i <= NCX; ++i) a[i] = P2[static_cast<int>((ix0 + i + ox) & 255)];
    float x[4], sx[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        x[j] = (static_cast<float>((gx0 + j) & (CPC - 1)) + 0.5f) * od.inv_ppc;
        sx[j] = fade<ORDER>(x[j]);
    }
    float2 top[NCX + 1];
    const int iyo0 = static_cast<int>((iy0 + oy) & 255);
#pragma unroll
    for (int i = 0; i <= NCX; ++i) top[i] = GP[a[i] + iyo0];
#pragma unroll
    for (int cy = 0; cy < NCY; ++cy) {
        const int iyo = static_cast<int>((iy0 + cy + 1 + oy) & 255);
        float2 bot[NCX + 1];
#pragma unroll
        for (int i = 0; i <= NCX; ++i) bot[i] = GP[a[i] + iyo];
#pragma unroll
        for (int cx = 0; cx < NCX; ++cx) {
            const float2 g00 = top[cx], g10 = top[cx + 1], g01 = bot[cx], g11 = bot[cx + 1];
#pragma unroll
            for (int jj = 0; jj < CPC; ++jj) {
                const int j = cx * CPC + jj;
                const float a0 = g00.x * x[j], a1 = g10.x * (x[j] - 1.f);
                const float b0 = g01.x * x[j], b1 = g11.x * (x[j] - 1.f);
                const float P0 = fmaf(sx[j], a1 - a0, a0), Q0 = fmaf(sx[j], g10.y - g00.y, g00.y);
                const float P1 = fmaf(sx[j], b1 - b0, b0), Q1 = fmaf(sx[j], g11.y - g01.y, g01.y);
#pragma unroll
                for (int rr = 0; rr < RPC; ++rr) {
                    const int r = cy * RPC + rr;
                    const float y = (static_cast<float>(rr) + 0.5f) * od.inv_ppc;
                    const float sy = fade<ORDER>(y), ym = y - 1.f;
                    const float h0 = fmaf(y, Q0, P0), h1 = fmaf(ym, Q1, P1);
                    acc[r][j] = fmaf(amp, fmaf(sy, h1 - h0, h0), acc[r][j]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i <= NCX; ++i) top[i] = bot[i];
    }
}

#ifndef TG_PERM_MINB
#define TG_PERM_MINB 2
#endif
template <int ORDER>
__global__ void __launch_bounds__(kThreads, TG_PERM_MINB) perm2d_kernel(const __grid_constant__ FbmArgs args, float* __restrict__ out) {
    __shared__ uint64_t key[256];
    __shared__ uint8_t P2[512];
    __shared__ float2 GP[512];
    __shared__ int off[kMaxOctaves][2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t s = args.seed_key[blockIdx.z] - kMapKeyBias;  // seed * K1
    key[tid] = mix64(s ^ (static_cast<uint64_t>(tid) * TG_PERM_KI) ^ TG_LANE_PERM);
    if (tid < args.octaves) {
        const uint64_t t = mix64((s + static_cast<uint64_t>(tid) * kOctMul) ^ TG_LANE_PERM);
        off[tid][0] = static_cast<int>(t & 255);
        off[tid][1] = static_cast<int>((t >> 8) & 255);
    }
    __syncthreads();
    {
        // the permutation = the indices sorted by (key, index): a bitonic sort
        // in shared memory (36 compare-exchange steps; ranking every key
        // against all 256 cost ~1.5 k instructions per thread and CTA)
        __shared__ uint8_t idx[256];
        idx[tid] = static_cast<uint8_t>(tid);
        __syncthreads();
        for (int k = 2; k <= 256; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                const int p = tid ^ j;
                if (p > tid) {
                    const uint64_t ka = key[tid], kb = key[p];
                    const uint8_t ia = idx[tid], ib = idx[p];
                    const bool gt = ka > kb || (ka == kb && ia > ib);
                    if (gt == ((tid & k) == 0)) {
                        key[tid] = kb, key[p] = ka;
                        idx[tid] = ib, idx[p] = ia;
                    }
                }
                __syncthreads();
            }
        }
        P2[tid] = P2[tid + 256] = idx[tid];
    }
    __syncthreads();
    {
        // the 8 unit gradients at k * 45 degrees, selected without a local array
        constexpr float R = 0.70710678118654752f;
        const int k = P2[tid] & 7;
        const float c = (k & 1) ? R : 1.f, z = (k & 1) ? R : 0.f;  // |component| on / off the axis
        const int q = k >> 1;                                         // quadrant
        const float gx = q == 0 ? c : q == 1 ? -z : q == 2 ? -c : z;
        const float gy = q == 0 ? z : q == 1 ? c : q == 2 ? -z : -c;
        GP[tid] = GP[tid + 256] = make_float2(gx, gy);
    }
    __syncthreads();

    const int64_t tx0 = args.tile_x0 + static_cast<int64_t>(blockIdx.x) * kTW;
    const int64_t ty0 = args.tile_y0 + static_cast<int64_t>(blockIdx.y) * kTH;
    const int c0 = lane * 4, r0 = warp * 8;
    float acc[8][4];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[r][j] = 0.f;
    for (int o = 0; o < args.octaves; ++o) {
        const OctDev& od = args.oct[o];
        if (od.cls == kClsSubInt || od.amp == 0.f) continue;  // lattice points: exactly 0
        const int ox = off[o][0], oy = off[o][1];
        const float amp = od.amp;
        if (od.cls == kClsFast && od.shift >= 2) {
            // ppc >= 4 (aligned): the thread's 4 columns share one cell and each
            // 4-row half of its rows one cell row, so the 4 corner gradients are
            // read once per cell row and the cell factorises into column terms
            // (kernels2d.hpp:163-173 regrouped): h0 = P0(x) + y Q0(x),
            // h1 = P1(x) + (y - 1) Q1(x), v = h0 + S(y) (h1 - h0).
            const int64_t ix = (tx0 + c0) >> od.shift;
            const int a = P2[static_cast<int>((ix + ox) & 255)], b = P2[static_cast<int>((ix + 1 + ox) & 255)];
            float x[4], sx[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t r = (tx0 + c0 + j) & (static_cast<int64_t>(od.ppc) - 1);
                x[j] = (static_cast<float>(r) + 0.5f) * od.inv_ppc;
                sx[j] = fade<ORDER>(x[j]);
            }
#pragma unroll
            for (int hr = 0; hr < 2; ++hr) {
                const int64_t iy = (ty0 + r0 + 4 * hr) >> od.shift;
                const int iyo = static_cast<int>((iy + oy) & 255);
                const float2 g00 = GP[a + iyo], g10 = GP[b + iyo], g01 = GP[a + iyo + 1], g11 = GP[b + iyo + 1];
                float P0[4], Q0[4], P1[4], Q1[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float a0 = g00.x * x[j], a1 = g10.x * (x[j] - 1.f);
                    const float b0 = g01.x * x[j], b1 = g11.x * (x[j] - 1.f);
                    P0[j] = fmaf(sx[j], a1 - a0, a0);
                    Q0[j] = fmaf(sx[j], g10.y - g00.y, g00.y);
                    P1[j] = fmaf(sx[j], b1 - b0, b0);
                    Q1[j] = fmaf(sx[j], g11.y - g01.y, g01.y);
                }
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    const int r = 4 * hr + rr;
                    const int64_t ry = (ty0 + r0 + r) & (static_cast<int64_t>(od.ppc) - 1);
                    const float y = (static_cast<float>(ry) + 0.5f) * od.inv_ppc;
                    const float sy = fade<ORDER>(y), ym = y - 1.f;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float h0 = fmaf(y, Q0[j], P0[j]), h1 = fmaf(ym, Q1[j], P1[j]);
                        acc[r][j] = fmaf(amp, fmaf(sy, h1 - h0, h0), acc[r][j]);
                    }
                }
            }
            continue;
        }
        if (od.cls == kClsFast && od.shift >= 0) {  // ppc 1 or 2
            if (od.shift == 1)
                perm_small<1, ORDER>(acc, od, P2, GP, tx0 + c0, ty0 + r0, ox, oy, amp);
            else
                perm_small<0, ORDER>(acc, od, P2, GP, tx0 + c0, ty0 + r0, ox, oy, amp);
            continue;
        }
        int a[4], b[4];
        float x[4], sx[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t ix;
            cell_coord(od, args.R, tx0 + c0 + j, &ix, &x[j]);
            sx[j] = fade<ORDER>(x[j]);
            a[j] = P2[static_cast<int>((ix + ox) & 255)];
            b[j] = P2[static_cast<int>((ix + 1 + ox) & 255)];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            int64_t iy;
            float y;
            cell_coord(od, args.R, ty0 + r0 + r, &iy, &y);
            const float sy = fade<ORDER>(y);
            const int iyo = static_cast<int>((iy + oy) & 255);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 g00 = GP[a[j] + iyo], g10 = GP[b[j] + iyo];
                const float2 g01 = GP[a[j] + iyo + 1], g11 = GP[b[j] + iyo + 1];
                const float xm = x[j] - 1.f, ym = y - 1.f;
                const float v00 = fmaf(g00.x, x[j], g00.y * y);
                const float v10 = fmaf(g10.x, xm, g10.y * y);
                const float v01 = fmaf(g01.x, x[j], g01.y * ym);
                const float v11 = fmaf(g11.x, xm, g11.y * ym);
                const float h0 = fmaf(sx[j], v10 - v00, v00);
                const float h1 = fmaf(sx[j], v11 - v01, v01);
                acc[r][j] = fmaf(amp, fmaf(sy, h1 - h0, h0), acc[r][j]);
            }
        }
    }
    const int64_t lx0 = tx0 + c0 - args.ox, ly0 = ty0 + r0 - args.oy;
    float* m = out + static_cast<int64_t>(blockIdx.z) * args.map_stride;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int64_t ly = ly0 + r;
        if (ly < 0 || ly >= args.height) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t lx = lx0 + j;
            if (lx >= 0 && lx < args.width) m[ly * args.ld + lx] = acc[r][j];
        }
    }
}

}  // namespace

cudaError_t perm2d_launch(int order, const FbmArgs& a, float* out, cudaStream_t st) {
    const int64_t tiles_x = (a.ox + a.width - a.tile_x0 + kTW - 1) / kTW;
    const int64_t tiles_y = (a.oy + a.height - a.tile_y0 + kTH - 1) / kTH;
    dim3 grid(static_cast<unsigned>(tiles_x), static_cast<unsigned>(tiles_y), static_cast<unsigned>(a.n_maps));
    if (order == 5)
        perm2d_kernel<5><<<grid, kThreads, 0, st>>>(a, out);
    else
        perm2d_kernel<3><<<grid, kThreads, 0, st>>>(a, out);
    return cudaGetLastError();
}

}  // namespace tg
