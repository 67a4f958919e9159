// fbm3d.cu — fused-octave 3D fBm volume (new, the
// reference has no 3D kernel: parity is property-pinned + restated oracle).
//
// Cell: separable zero-gradient trilinear blend with smoothstep weights,
//   v = lerp_z(lerp_y(lerp_x(h, Sx), Sy), Sz),
// which reduces on every face to kernels2d::zg_eval(..., separable) and has
// zero gradient at all 8 corners.  Lattice key: pack2 + iz * K5 (iz = 0 is the
// 2D lattice).  Per axis the sampling is the 2D rule (fast: x = (r+0.5)/ppc,
// else ((g+0.5)/R)*freq in fp64).
//
// Same structure as fbm2d.cu: a 128 x 8 x 8 voxel tile per CTA (thread = 4
// columns x 1 row x 8 slices), one prologue hashing every octave's unique
// corners into shared memory, one barrier, then per-octave evaluation with
// the cell factorised per (cell, y, z):  v(x) = B0 + Sx*(B1 - B0), the
// y-lerps hoisted per cell and B0 accumulated once per (y, z) when the
// thread's 4 columns share a cell.  Lattice-point octaves hash one corner per
// voxel; ppc = 1 is the mean of 8 corners.  Accumulators stay in registers;
// one fp32 store per voxel.
#include <cuda_runtime.h>

#include <cmath>

#include "devattr.h"
#include "fbm_params.h"
#include "lattice.cuh"

namespace tg {

namespace {

#ifndef TG_3D_LEAN_MIN_BLOCKS
#define TG_3D_LEAN_MIN_BLOCKS 4
#endif

constexpr int kThreads3 = 256;
constexpr int kTX = 128, kTY = 8, kTZ = 8;
constexpr int kCap3 = 13312;  // corner floats per CTA

template <int ORDER>
__device__ __forceinline__ float smooth3(float t) {
    if constexpr (ORDER == 5) return t * t * t * fmaf(t, fmaf(6.f, t, -15.f), 10.f);
    else return t * t * fmaf(-2.f, t, 3.f);
}

__device__ __forceinline__ void coord3(const OctDev& od, double R, int64_t g, int64_t* i, float* t) {
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

__device__ __forceinline__ uint64_t pack3(uint64_t base, int64_t ix, int64_t iy, int64_t iz) {
    return base + static_cast<uint64_t>(ix) * kIxMul + static_cast<uint64_t>(iy) * kIyMul +
           static_cast<uint64_t>(iz) * kIzMul;
}

__device__ __forceinline__ float lerp(float a, float b, float s) { return fmaf(s, b - a, a); }

// Column pairs (0, 1), (2, 3) of a row accumulated in packed fp32x2 (FFMA2 /
// FADD2: one issue slot per pair, each lane rounded as the scalar op).
#ifndef TG_F32X2_3D
#define TG_F32X2_3D 1
#endif
__device__ __forceinline__ void fma4(float (&a)[4], const float (&x)[4], float y) {
#if TG_F32X2_3D
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const float2 r = __ffma2_rn(make_float2(x[2 * p], x[2 * p + 1]), make_float2(y, y),
                                    make_float2(a[2 * p], a[2 * p + 1]));
        a[2 * p] = r.x;
        a[2 * p + 1] = r.y;
    }
#else
#pragma unroll
    for (int j = 0; j < 4; ++j) a[j] = fmaf(x[j], y, a[j]);
#endif
}
__device__ __forceinline__ void fma4s(float (&a)[4], float x, const float (&y)[4]) {
#if TG_F32X2_3D
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const float2 r = __ffma2_rn(make_float2(x, x), make_float2(y[2 * p], y[2 * p + 1]),
                                    make_float2(a[2 * p], a[2 * p + 1]));
        a[2 * p] = r.x;
        a[2 * p + 1] = r.y;
    }
#else
#pragma unroll
    for (int j = 0; j < 4; ++j) a[j] = fmaf(x, y[j], a[j]);
#endif
}

// One plan entry per octave is computed by the host (capi.cu plan3):
// mode in OctDev.mode, grid shape ncx, ncy, pad(=ncz), pitch (x stride), goff.
enum Mode3 : int32_t { kM3Sub = 0, kM3P1 = 1, kM3Blk = 2, kM3Gen = 3, kM3Direct = 4 };

struct Tab3 {
    float xt[kTX], xs[kTX];
    int32_t xi[kTX];
    float yt[kTY], ys[kTY];
    int32_t yi[kTY];
    float zt[kTZ], zs[kTZ];
    int32_t zi[kTZ];
};

constexpr int kTabs3 = 2;

struct Smem3 {
    Tab3 tab[kTabs3];
    float grid[kCap3];
};

// Lean kernels (no general octaves) use only the corner grid: 53 KB, so 4
// CTAs fit an SM.
template <bool LEAN>
constexpr size_t smem3() {
    return LEAN ? sizeof(float) * kCap3 : sizeof(Smem3);
}

// LEAN: no general octaves in the plan (host-decided): the per-voxel general
// path is compiled out, which lowers the register pressure of the rest
// enough for 4 CTAs per SM (64 registers, no spills; with the 53 KB
// corner-only shared memory: 0.96 -> 0.87 (3 CTAs) -> 0.81 ms at config 4).
template <int ORDER, bool LEAN>
__global__ void __launch_bounds__(kThreads3, LEAN ? TG_3D_LEAN_MIN_BLOCKS : 2)
fbm3d_kernel(const __grid_constant__ Fbm3Args a, float* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char raw3[];
    Smem3& S = *reinterpret_cast<Smem3*>(raw3);
    // lean kernels have no sampling tables: the corner grid starts at 0
    float* const grid3 = LEAN ? reinterpret_cast<float*>(raw3) : S.grid;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tx0 = a.tile_x0 + static_cast<int64_t>(blockIdx.x) * kTX;
    const int64_t ty0 = a.tile_y0 + static_cast<int64_t>(blockIdx.y) * kTY;
    const int64_t tz0 = a.tile_z0 + static_cast<int64_t>(blockIdx.z) * kTZ;
    const int c0 = lane * 4;

    // Packed key of every aligned octave's first tile corner, one octave per
    // lane (64-bit index products once per warp instead of once per thread),
    // read back by shuffle in the prologue.
    uint64_t lane_p0 = 0;
    if (lane < a.octaves) {
        const OctDev& od = a.oct[lane];
        if (od.lut_off >= 0)
            lane_p0 = pack3(a.seed_key + od.oct_key, tx0 >> od.shift, ty0 >> od.shift, tz0 >> od.shift);
    }

    // ---- prologue: all octaves' tile corners (raw map_height values) ------
    for (int o = 0; o < a.octaves; ++o) {
        const OctDev& od = a.oct[o];
        const int mode = od.mode;
        if (mode == kM3Sub || mode == kM3Direct) continue;
        const uint64_t base = a.seed_key + od.oct_key;
        int64_t ix0, iy0, iz0;
        int ncx = od.ncx, ncy = od.ncy, ncz = od.pad;
        if (LEAN || od.lut_off >= 0) {  // lean plans hold aligned grids only (launch3)
            ix0 = tx0 >> od.shift;
            iy0 = ty0 >> od.shift;
            iz0 = tz0 >> od.shift;
        } else {
            int64_t e;
            float t;
            coord3(od, a.R, tx0, &ix0, &t);
            coord3(od, a.R, tx0 + kTX - 1, &e, &t);
            ncx = static_cast<int>(e - ix0 + 2);
            coord3(od, a.R, ty0, &iy0, &t);
            coord3(od, a.R, ty0 + kTY - 1, &e, &t);
            ncy = static_cast<int>(e - iy0 + 2);
            coord3(od, a.R, tz0, &iz0, &t);
            coord3(od, a.R, tz0 + kTZ - 1, &e, &t);
            ncz = static_cast<int>(e - iz0 + 2);
            if constexpr (LEAN) __trap();  // the host never sends general octaves to a lean kernel
            Tab3& tb = S.tab[od.tslot];
            if (tid < kTX) {
                int64_t i;
                float x;
                coord3(od, a.R, tx0 + tid, &i, &x);
                tb.xi[tid] = static_cast<int32_t>(i - ix0);
                tb.xt[tid] = x;
                tb.xs[tid] = smooth3<ORDER>(x);
            } else if (tid < kTX + kTY) {
                const int r = tid - kTX;
                int64_t i;
                float y;
                coord3(od, a.R, ty0 + r, &i, &y);
                tb.yi[r] = static_cast<int32_t>(i - iy0);
                tb.yt[r] = y;
                tb.ys[r] = smooth3<ORDER>(y);
            } else if (tid < kTX + kTY + kTZ) {
                const int r = tid - kTX - kTY;
                int64_t i;
                float z;
                coord3(od, a.R, tz0 + r, &i, &z);
                tb.zi[r] = static_cast<int32_t>(i - iz0);
                tb.zt[r] = z;
                tb.zs[r] = smooth3<ORDER>(z);
            }
        }
        const uint64_t p0 =
            (LEAN || od.lut_off >= 0) ? __shfl_sync(0xffffffffu, lane_p0, o) : pack3(base, ix0, iy0, iz0);
        const int pitch = od.pitch, plane = pitch * od.ncy;  // strides use the planned bounds
        float* g = grid3 + od.goff;
        const int nrows = ncy * ncz;
        if ((LEAN || od.lut_off >= 0) && od.shift <= 5) {
            // aligned power-of-two grid, Wm = 128 >> s >= 4 corner columns
            // before the last: 4 consecutive x per lane (four hash chains, one
            // 16-byte store), 2^s corner rows (cy, cz) per warp pass; the last
            // column through a flat loop.  rw / ncy by a multiplier (rw < 2^7).
            // starting warp / thread rotated per octave (the row counts do
            // not divide evenly over the 8 warps)
            const int wv = (warp - o) & 7, tv = (tid - 32 * o) & (kThreads3 - 1);
            const int sh = od.shift, lsh = 5 - sh, Wm = kTX >> sh;
            const int cg = lane & ((1 << lsh) - 1), rsub = lane >> lsh, rpw = 1 << sh;
            const int cdiv = od.cdiv;
            const uint64_t px = p0 + static_cast<uint64_t>(4 * cg) * kIxMul;
            for (int rw = wv * rpw + rsub; rw < nrows; rw += (kThreads3 / 32) * rpw) {
                const int cz = (rw * cdiv) >> 16, cy = rw - cz * ncy;
                const uint64_t p = px + static_cast<uint64_t>(static_cast<uint32_t>(cy)) * kIyMul +
                                   static_cast<uint64_t>(static_cast<uint32_t>(cz)) * kIzMul;
                float h[4];
                map_height4(p, add64(p, kIxMul), add64(p, 2 * kIxMul), add64(p, 3 * kIxMul), h);
                *reinterpret_cast<float4*>(g + cz * plane + cy * pitch + 4 * cg) = make_float4(h[0], h[1], h[2], h[3]);
            }
            for (int rw = tv; rw < nrows; rw += kThreads3) {
                const int cz = (rw * cdiv) >> 16, cy = rw - cz * ncy;
                g[cz * plane + cy * pitch + Wm] =
                    map_height(p0 + static_cast<uint64_t>(static_cast<uint32_t>(Wm)) * kIxMul +
                               static_cast<uint64_t>(static_cast<uint32_t>(cy)) * kIyMul +
                               static_cast<uint64_t>(static_cast<uint32_t>(cz)) * kIzMul);
            }
        } else {
            const int n = ncx * nrows;
            const float rx = 1.0f / static_cast<float>(ncx), ry = 1.0f / static_cast<float>(ncy);
            for (int i0 = tid; i0 < n; i0 += 4 * kThreads3) {
                float d[4];
                int dst[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int i = min(i0 + u * kThreads3, n - 1);
                    const int rw = static_cast<int>((static_cast<float>(i) + 0.5f) * rx);
                    const int cx = i - rw * ncx;
                    const int cz = static_cast<int>((static_cast<float>(rw) + 0.5f) * ry);
                    const int cy = rw - cz * ncy;
                    dst[u] = cz * plane + cy * pitch + cx;
                    d[u] = map_height(pack3(p0, cx, cy, cz));
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i0 + u * kThreads3 < n) g[dst[u]] = d[u];
            }
        }
    }
    __syncthreads();

    float acc[kTZ][4], racc[kTZ];
#pragma unroll
    for (int z = 0; z < kTZ; ++z) {
        racc[z] = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[z][j] = kMapOffset ? kMapOffsetUnits * a.hoff : 0.f;  // map_height offsets
    }

    for (int o = 0; o < a.octaves; ++o) {
        const OctDev& od = a.oct[o];
        const int mode = od.mode;
        const float amp = od.amp * kMapScale;
        const uint64_t base = a.seed_key + od.oct_key;
        const int pitch = od.pitch, plane = od.pitch * od.ncy;

        if (mode == kM3Sub) {  // lattice points: v = h(ix, iy, iz)
            // host key constants (fbm3d_plan); two slices per step = 8
            // independent hash chains
            const uint64_t kx = od.kx, kz = od.kz;
            uint64_t K = a.seed_key + od.key0 + static_cast<uint64_t>(blockIdx.x * kTX + c0) * kx +
                         static_cast<uint64_t>(blockIdx.y * kTY + warp) * od.ky +
                         static_cast<uint64_t>(blockIdx.z * kTZ) * kz;
#pragma unroll
            for (int z = 0; z < kTZ; z += 2) {
                uint64_t p[8];
                p[0] = K;
                p[4] = add64(K, kz);
#pragma unroll
                for (int j = 1; j < 4; ++j) {
                    p[j] = add64(p[j - 1], kx);
                    p[4 + j] = add64(p[3 + j], kx);
                }
                float h[8];
                map_heightN<8>(p, h);
                const float h0[4] = {h[0], h[1], h[2], h[3]}, h1[4] = {h[4], h[5], h[6], h[7]};
                fma4s(acc[z], amp, h0);
                fma4s(acc[z + 1], amp, h1);
                if (z + 2 < kTZ) K = add64(p[4], kz);
            }
            continue;
        }

        if (mode == kM3P1) {  // x = y = z = 1/2: the mean of the 8 corners
            const float* g = grid3 + od.goff + warp * pitch + c0;
            const float q = 0.125f * amp;
            auto face = [&](int z, float (&F)[4]) {
                const float* r0p = g + z * plane;
                const float* r1p = r0p + pitch;
                const float4 u = *reinterpret_cast<const float4*>(r0p);
                const float4 w = *reinterpret_cast<const float4*>(r1p);
                const float u4 = r0p[4], w4 = r1p[4];
                const float s0 = u.x + w.x, s1 = u.y + w.y, s2 = u.z + w.z, s3 = u.w + w.w, s4 = u4 + w4;
                F[0] = s0 + s1;
                F[1] = s1 + s2;
                F[2] = s2 + s3;
                F[3] = s3 + s4;
            };
            float Fa[4];
            face(0, Fa);
#pragma unroll
            for (int z = 0; z < kTZ; ++z) {
                float Fb[4];
                face(z + 1, Fb);
                float Fs[4];
#pragma unroll
                for (int p = 0; p < 2; ++p) {
                    const float2 t = __fadd2_rn(make_float2(Fa[2 * p], Fa[2 * p + 1]), make_float2(Fb[2 * p], Fb[2 * p + 1]));
                    Fs[2 * p] = t.x;
                    Fs[2 * p + 1] = t.y;
                }
                fma4s(acc[z], q, Fs);
#pragma unroll
                for (int j = 0; j < 4; ++j) Fa[j] = Fb[j];
            }
            continue;
        }

        if (mode == kM3Blk) {  // power-of-two ppc >= 2 on the aligned tile grid
            const int sh = od.shift, mask = od.ppc - 1;
            const float4* L = a.lut + od.lut_off;
            // planar S(x) copy of the row LUT: S at float [ppc + r] (kernels.cu row_lut)
            const float* LS = reinterpret_cast<const float*>(a.lut + kLutN4) + od.ppc;
            const int xo = static_cast<int>(tx0 & mask) + c0;
            const int yo = static_cast<int>(ty0 & mask) + warp;
            const int zo = static_cast<int>(tz0 & mask);
            const float sy = L[yo & mask].y;
            float sx[4];
            if (sh >= 2) {  // xo % 4 == 0 and ppc >= 4: 4 consecutive entries
                const float4 v = __ldg(reinterpret_cast<const float4*>(LS + (xo & mask)));
                sx[0] = v.x;
                sx[1] = v.y;
                sx[2] = v.z;
                sx[3] = v.w;
            } else {  // ppc = 2: x = 1/4, 3/4 alternate
                sx[0] = sx[2] = LS[0];
                sx[1] = sx[3] = LS[1];
            }
            const float* gy = grid3 + od.goff + (yo >> sh) * pitch;
            if (sh >= 2) {
                // the thread's 4 columns share one x-cell; B0 -> per-slice accumulator.
                // ppc >= 8: the 8 slices lie in one z-cell (zo % 8 == 0), S(z)
                // at 8 consecutive entries; ppc = 4: two z-cells, S(z & 3).
                const float* g = gy + (xo >> sh);
                float szv[kTZ];
                if (sh >= 3) {
                    const float4 s0 = __ldg(reinterpret_cast<const float4*>(LS + zo));
                    const float4 s1 = __ldg(reinterpret_cast<const float4*>(LS + zo + 4));
                    szv[0] = s0.x; szv[1] = s0.y; szv[2] = s0.z; szv[3] = s0.w;
                    szv[4] = s1.x; szv[5] = s1.y; szv[6] = s1.z; szv[7] = s1.w;
                } else {
                    const float4 s0 = __ldg(reinterpret_cast<const float4*>(LS));
                    szv[0] = szv[4] = s0.x; szv[1] = szv[5] = s0.y; szv[2] = szv[6] = s0.z; szv[3] = szv[7] = s0.w;
                }
#pragma unroll
                for (int zc = 0; zc < 2; ++zc) {
                    if (zc == 1 && sh >= 3) break;  // one z-cell
                    const float* q = g + ((zo >> sh) + zc) * plane;
                    // y-lerps of the x=0 / x=1 edges at z = cz, cz+1
                    const float e0 = amp * lerp(q[0], q[pitch], sy);
                    const float e1 = amp * lerp(q[plane], q[plane + pitch], sy);
                    const float e2 = amp * lerp(q[1], q[pitch + 1], sy);
                    const float e3 = amp * lerp(q[plane + 1], q[plane + pitch + 1], sy);
                    const int z0 = sh >= 3 ? 0 : 4 * zc, z1 = sh >= 3 ? kTZ : 4 * zc + 4;
#pragma unroll
                    for (int z = 0; z < kTZ; ++z) {
                        if (z < z0 || z >= z1) continue;
                        const float sz = szv[z];
                        const float b0 = lerp(e0, e1, sz), d = lerp(e2, e3, sz) - b0;
                        racc[z] += b0;
                        fma4(acc[z], sx, d);
                    }
                }
            } else {
                // ppc = 2: columns (0,1) and (2,3) are two x-cells
                const float* g = gy + (xo >> 1);
                const float sz0 = LS[0], sz1 = LS[1];
#pragma unroll
                for (int zc = 0; zc < kTZ / 2; ++zc) {
                    const float* q = g + ((zo >> 1) + zc) * plane;
                    float e[3][2];  // y-lerped corner columns x = 0..2 at z = cz, cz+1
#pragma unroll
                    for (int u = 0; u < 3; ++u) {
                        e[u][0] = amp * lerp(q[u], q[pitch + u], sy);
                        e[u][1] = amp * lerp(q[plane + u], q[plane + pitch + u], sy);
                    }
#pragma unroll
                    for (int zz = 0; zz < 2; ++zz) {
                        const int z = 2 * zc + zz;
                        const float sz = zz ? sz1 : sz0;
                        const float b0 = lerp(e[0][0], e[0][1], sz);
                        const float b1 = lerp(e[1][0], e[1][1], sz);
                        const float b2 = lerp(e[2][0], e[2][1], sz);
#if TG_F32X2_3D
                        // columns (0, 1) lerp b0 -> b1, (2, 3) b1 -> b2 (x = 1/4, 3/4)
                        const float2 sxp = make_float2(sx[0], sx[1]);
                        const float d01 = b1 - b0, d12 = b2 - b1;
                        const float2 l0 = __ffma2_rn(sxp, make_float2(d01, d01), make_float2(b0, b0));
                        const float2 l1 = __ffma2_rn(sxp, make_float2(d12, d12), make_float2(b1, b1));
                        const float2 s0 = __fadd2_rn(make_float2(acc[z][0], acc[z][1]), l0);
                        const float2 s1 = __fadd2_rn(make_float2(acc[z][2], acc[z][3]), l1);
                        acc[z][0] = s0.x;
                        acc[z][1] = s0.y;
                        acc[z][2] = s1.x;
                        acc[z][3] = s1.y;
#else
                        acc[z][0] += lerp(b0, b1, sx[0]);
                        acc[z][1] += lerp(b0, b1, sx[1]);
                        acc[z][2] += lerp(b1, b2, sx[2]);
                        acc[z][3] += lerp(b1, b2, sx[3]);
#endif
                    }
                }
            }
            continue;
        }

        // general octaves: per-voxel cell lookup (grid or hashed corners)
        if constexpr (LEAN) continue;
        const bool direct = mode == kM3Direct;
        float sx[4];
        int64_t ixj[4];
        float sy;
        int64_t iy;
        if (!direct) {
            const Tab3& tb = S.tab[od.tslot];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                sx[j] = tb.xs[c0 + j];
                ixj[j] = tb.xi[c0 + j];
            }
            sy = tb.ys[warp];
            iy = tb.yi[warp];
        } else {
            float t;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                coord3(od, a.R, tx0 + c0 + j, &ixj[j], &t);
                sx[j] = smooth3<ORDER>(t);
            }
            coord3(od, a.R, ty0 + warp, &iy, &t);
            sy = smooth3<ORDER>(t);
        }
#pragma unroll
        for (int z = 0; z < kTZ; ++z) {
            float sz;
            int64_t iz;
            if (!direct) {
                sz = S.tab[od.tslot].zs[z];
                iz = S.tab[od.tslot].zi[z];
            } else {
                float t;
                coord3(od, a.R, tz0 + z, &iz, &t);
                sz = smooth3<ORDER>(t);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float h[8];
                if (!direct) {
                    const int b = static_cast<int>(iz) * plane + static_cast<int>(iy) * pitch + static_cast<int>(ixj[j]);
                    const float* q = grid3 + od.goff + b;
                    h[0] = q[0];
                    h[1] = q[1];
                    h[2] = q[pitch];
                    h[3] = q[pitch + 1];
                    h[4] = q[plane];
                    h[5] = q[plane + 1];
                    h[6] = q[plane + pitch];
                    h[7] = q[plane + pitch + 1];
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        h[k] = map_height(pack3(base, ixj[j] + (k & 1), iy + ((k >> 1) & 1), iz + ((k >> 2) & 1)));
                }
                const float b0 = lerp(lerp(h[0], h[2], sy), lerp(h[4], h[6], sy), sz);
                const float b1 = lerp(lerp(h[1], h[3], sy), lerp(h[5], h[7], sy), sz);
                acc[z][j] = fmaf(amp, lerp(b0, b1, sx[j]), acc[z][j]);
            }
        }
    }
    // store (x fastest): one 16-byte store per slice when the thread's 4
    // voxels are inside the window and aligned, else per voxel
    const int64_t ly = ty0 + warp - a.oy;
    if (ly < 0 || ly >= a.ny) return;
    const int64_t lx0 = tx0 + c0 - a.ox;
    const bool vec = lx0 >= 0 && lx0 + 4 <= a.nx && ((lx0 | a.nx) & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    float* row = out + ((tz0 - a.oz) * a.ny + ly) * a.nx;
    const int64_t zstride = a.ny * a.nx;
#pragma unroll
    for (int z = 0; z < kTZ; ++z, row += zstride) {
        const int64_t lz = tz0 + z - a.oz;
        if (lz < 0 || lz >= a.nz) continue;
        if (vec) {
            *reinterpret_cast<float4*>(row + lx0) =
                make_float4(acc[z][0] + racc[z], acc[z][1] + racc[z], acc[z][2] + racc[z], acc[z][3] + racc[z]);
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t lx = lx0 + j;
                if (lx >= 0 && lx < a.nx) row[lx] = acc[z][j] + racc[z];
            }
        }
    }
}

template <int ORDER, bool LEAN>
cudaError_t launch3v(const Fbm3Args& a, float* out, cudaStream_t st) {
    static PerDeviceOnce configured;
    cudaError_t e = configured.run([] {
        return cudaFuncSetAttribute(fbm3d_kernel<ORDER, LEAN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem3<LEAN>()));
    });
    if (e != cudaSuccess) return e;
    dim3 grid(static_cast<unsigned>((a.ox + a.nx - a.tile_x0 + kTX - 1) / kTX),
              static_cast<unsigned>((a.oy + a.ny - a.tile_y0 + kTY - 1) / kTY),
              static_cast<unsigned>((a.oz + a.nz - a.tile_z0 + kTZ - 1) / kTZ));
    fbm3d_kernel<ORDER, LEAN><<<grid, kThreads3, smem3<LEAN>(), st>>>(a, out);
    return cudaGetLastError();
}

template <int ORDER>
cudaError_t launch3(const Fbm3Args& a, float* out, cudaStream_t st) {
    bool lean = true;
    for (int o = 0; o < a.octaves; ++o) lean = lean && a.oct[o].mode != kM3Gen && a.oct[o].mode != kM3Direct;
    return lean ? launch3v<ORDER, true>(a, out, st) : launch3v<ORDER, false>(a, out, st);
}

}  // namespace

void fbm3d_tile(int* tx, int* ty, int* tz) {
    *tx = kTX;
    *ty = kTY;
    *tz = kTZ;
}

// Host plan for the 3D kernel: modes, corner-grid shapes and offsets.
void fbm3d_plan(Fbm3Args* a, int zg_sep_only) {
    (void)zg_sep_only;
    int goff = 0, slot = 0;
    for (int o = 0; o < a->octaves; ++o) {
        OctDev& d = a->oct[o];
        d.tslot = -1;
        d.lut_off = -1;
        if (d.cls == kClsSubInt) {
            // key(x, y, z) = seed*K1 + key0 + (bx*128 + c)*kx + (by*8 + w)*ky + (bz*8 + z)*kz
            // with u = g*k + k/2 on every axis (lattice.hpp:46-50 + the 3D term)
            d.mode = kM3Sub;
            const uint64_t k = static_cast<uint64_t>(d.k), h = k >> 1;
            d.kx = k * kIxMul;
            d.ky = k * kIyMul;
            d.kz = k * kIzMul;
            d.key0 = d.oct_key + (static_cast<uint64_t>(a->tile_x0) * k + h) * kIxMul +
                     (static_cast<uint64_t>(a->tile_y0) * k + h) * kIyMul +
                     (static_cast<uint64_t>(a->tile_z0) * k + h) * kIzMul;
            continue;
        }
        int64_t nx, ny, nz;
        int mode;
        if (d.cls == kClsFast && d.shift >= 0 && d.shift <= kLutLog2Max) {
            d.lut_off = (1 << d.shift) - 1;
            nx = (d.ppc >= kTX ? 1 : kTX / d.ppc) + 1;
            ny = (d.ppc >= kTY ? 1 : kTY / d.ppc) + 1;
            nz = (d.ppc >= kTZ ? 1 : kTZ / d.ppc) + 1;
            mode = d.ppc == 1 ? kM3P1 : kM3Blk;
        } else {
            double fx, fy, fz;
            if (d.cls == kClsFast) {
                fx = (kTX - 1) / d.ppc + 3;
                fy = (kTY - 1) / d.ppc + 3;
                fz = (kTZ - 1) / d.ppc + 3;
            } else {
                const double span = d.freq / a->R;
                fx = std::ceil((kTX - 1) * span) + 3.0;
                fy = std::ceil((kTY - 1) * span) + 3.0;
                fz = std::ceil((kTZ - 1) * span) + 3.0;
            }
            nx = fx > 1e6 ? 1000000 : static_cast<int64_t>(fx);
            ny = fy > 1e6 ? 1000000 : static_cast<int64_t>(fy);
            nz = fz > 1e6 ? 1000000 : static_cast<int64_t>(fz);
            mode = kM3Gen;
        }
        const int64_t pitch = (nx + 3) & ~int64_t(3);
        const int64_t size = pitch * ny * nz;
        if (nx * ny * nz > kCap3 || goff + size > kCap3 || (mode == kM3Gen && slot >= kTabs3)) {
            d.mode = kM3Direct;
            d.lut_off = -1;
            continue;
        }
        d.mode = mode;
        d.ncx = static_cast<int32_t>(nx);
        d.ncy = static_cast<int32_t>(ny);
        d.pad = static_cast<int32_t>(nz);
        d.pitch = static_cast<int32_t>(pitch);
        d.goff = goff;
        d.cdiv = static_cast<int32_t>((65536 + ny - 1) / ny);  // row / ncy for rows < 2^7 (prologue)
        goff += static_cast<int>(size);
        if (mode == kM3Gen) d.tslot = slot++;
    }
}

cudaError_t fbm3d_launch(int order, const Fbm3Args& a, float* out, cudaStream_t st) {
    return order == 5 ? launch3<5>(a, out, st) : launch3<3>(a, out, st);
}

}  // namespace tg
