// fbm3d.cu — fused-octave 3D fBm volume (new, the
// reference has no 3D kernel).
//
// Cell: separable zero-gradient trilinear blend with smoothstep weights,
//   v = lerp_z(lerp_y(lerp_x(h, Sx), Sy), Sz),
// which reduces on every face to kernels2d::zg_eval(..., separable) and has
// zero gradient at all 8 corners.  Lattice key: pack2 + iz * K5 (iz = 0 is
// the 2D lattice).  Per axis the sampling is the 2D rule (fast: x = (r+0.5)/ppc,
// else ((g+0.5)/R)*freq in fp64).  Same tile/shared-corner structure as
// fbm2d.cu: a 128 x 8 x 8 voxel tile, accumulators in registers over all
// octaves, one fp32 store per voxel.
#include <cuda_runtime.h>

#include "fbm_params.h"
#include "lattice.cuh"

namespace tg {

namespace {

constexpr int kThreads3 = 256;
constexpr int kTX = 128, kTY = 8, kTZ = 8;
constexpr int kCap3 = (kTX + 2) * (kTY + 2) * (kTZ + 2);

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

__device__ __forceinline__ float h3(uint64_t base, int64_t ix, int64_t iy, int64_t iz, float amp,
                                    int zero) {
    if (zero) return 0.f;
    const uint64_t p = base + static_cast<uint64_t>(ix) * kIxMul + static_cast<uint64_t>(iy) * kIyMul +
                       static_cast<uint64_t>(iz) * kIzMul;
    return amp * height_from_hash(mix64(p));
}

struct Smem3 {
    float xs[kTX], xv[kTX];
    int64_t xi[kTX];
    float ys[kTY], zs[kTZ];
    int64_t yi[kTY], zi[kTZ];
    float grid[kCap3];
};

__device__ __forceinline__ float lerp(float a, float b, float s) { return fmaf(s, b - a, a); }

template <int ORDER>
__global__ void __launch_bounds__(kThreads3)
fbm3d_kernel(const __grid_constant__ Fbm3Args a, float* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char raw3[];
    Smem3& S = *reinterpret_cast<Smem3*>(raw3);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t tx0 = a.tile_x0 + static_cast<int64_t>(blockIdx.x) * kTX;
    const int64_t ty0 = a.tile_y0 + static_cast<int64_t>(blockIdx.y) * kTY;
    const int64_t tz0 = a.tile_z0 + static_cast<int64_t>(blockIdx.z) * kTZ;
    const int c0 = lane * 4;
    float acc[kTZ][4];
#pragma unroll
    for (int z = 0; z < kTZ; ++z)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[z][j] = 0.f;

    for (int o = 0; o < a.octaves; ++o) {
        const OctDev& od = a.oct[o];
        const uint64_t base = a.seed_key + od.oct_key;
        if (od.cls == kClsSubInt) {  // samples on lattice points: v = h(ix, iy, iz)
            if (a.zero) continue;
            const int64_t k = od.k, half = od.k >> 1;
            const int64_t iy = (ty0 + warp) * k + half;
#pragma unroll
            for (int z = 0; z < kTZ; ++z) {
                const int64_t iz = (tz0 + z) * k + half;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t ix = (tx0 + c0 + j) * k + half;
                    acc[z][j] += h3(base, ix, iy, iz, od.amp, 0);
                }
            }
            continue;
        }
        __syncthreads();
        if (tid < kTX) {
            int64_t i;
            float t;
            coord3(od, a.R, tx0 + tid, &i, &t);
            S.xi[tid] = i;
            S.xv[tid] = t;
            S.xs[tid] = smooth3<ORDER>(t);
        } else if (tid < kTX + kTY) {
            const int r = tid - kTX;
            int64_t i;
            float t;
            coord3(od, a.R, ty0 + r, &i, &t);
            S.yi[r] = i;
            S.ys[r] = smooth3<ORDER>(t);
        } else if (tid < kTX + kTY + kTZ) {
            const int r = tid - kTX - kTY;
            int64_t i;
            float t;
            coord3(od, a.R, tz0 + r, &i, &t);
            S.zi[r] = i;
            S.zs[r] = smooth3<ORDER>(t);
        }
        int64_t ix0, ixe, iy0, iye, iz0, ize;
        float d;
        coord3(od, a.R, tx0, &ix0, &d);
        coord3(od, a.R, tx0 + kTX - 1, &ixe, &d);
        coord3(od, a.R, ty0, &iy0, &d);
        coord3(od, a.R, ty0 + kTY - 1, &iye, &d);
        coord3(od, a.R, tz0, &iz0, &d);
        coord3(od, a.R, tz0 + kTZ - 1, &ize, &d);
        const int64_t nx = ixe - ix0 + 2, ny = iye - iy0 + 2, nz = ize - iz0 + 2;
        const bool direct = nx * ny * nz > kCap3;
        const int ncx = static_cast<int>(nx), ncy = static_cast<int>(ny), ncz = static_cast<int>(nz);
        if (!direct) {
            const int planes = ncy * ncz;
            for (int pl = warp; pl < planes; pl += kThreads3 / 32) {
                const int cz = pl / ncy, cy = pl - cz * ncy;
                for (int cx = lane; cx < ncx; cx += 32)
                    S.grid[(cz * ncy + cy) * ncx + cx] = h3(base, ix0 + cx, iy0 + cy, iz0 + cz, od.amp, a.zero);
            }
        }
        __syncthreads();
        const float sy = S.ys[warp];
        const int64_t iy = S.yi[warp];
        float sx[4];
        int64_t ixj[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            sx[j] = S.xs[c0 + j];
            ixj[j] = S.xi[c0 + j];
        }
#pragma unroll
        for (int z = 0; z < kTZ; ++z) {
            const float sz = S.zs[z];
            const int64_t iz = S.zi[z];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float h[8];
                if (!direct) {
                    const int b = (static_cast<int>(iz - iz0) * ncy + static_cast<int>(iy - iy0)) * ncx +
                                  static_cast<int>(ixj[j] - ix0);
                    h[0] = S.grid[b];
                    h[1] = S.grid[b + 1];
                    h[2] = S.grid[b + ncx];
                    h[3] = S.grid[b + ncx + 1];
                    h[4] = S.grid[b + ncx * ncy];
                    h[5] = S.grid[b + ncx * ncy + 1];
                    h[6] = S.grid[b + ncx * ncy + ncx];
                    h[7] = S.grid[b + ncx * ncy + ncx + 1];
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        h[q] = h3(base, ixj[j] + (q & 1), iy + ((q >> 1) & 1), iz + ((q >> 2) & 1), od.amp,
                                  a.zero);
                }
                // x-lerped edges, then y, then z (multilinear in Sx, Sy, Sz)
                const float b0 = lerp(lerp(h[0], h[2], sy), lerp(h[4], h[6], sy), sz);
                const float b1 = lerp(lerp(h[1], h[3], sy), lerp(h[5], h[7], sy), sz);
                acc[z][j] += lerp(b0, b1, sx[j]);
            }
        }
    }
    // store (x fastest)
    const int64_t ly = ty0 + warp - a.oy;
    if (ly < 0 || ly >= a.ny) return;
#pragma unroll
    for (int z = 0; z < kTZ; ++z) {
        const int64_t lz = tz0 + z - a.oz;
        if (lz < 0 || lz >= a.nz) continue;
        float* row = out + (lz * a.ny + ly) * a.nx;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t lx = tx0 + c0 + j - a.ox;
            if (lx >= 0 && lx < a.nx) row[lx] = acc[z][j];
        }
    }
}

template <int ORDER>
cudaError_t launch3(const Fbm3Args& a, float* out, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(fbm3d_kernel<ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sizeof(Smem3)));
        if (e != cudaSuccess) return e;
        configured = true;
    }
    dim3 grid(static_cast<unsigned>((a.ox + a.nx - a.tile_x0 + kTX - 1) / kTX),
              static_cast<unsigned>((a.oy + a.ny - a.tile_y0 + kTY - 1) / kTY),
              static_cast<unsigned>((a.oz + a.nz - a.tile_z0 + kTZ - 1) / kTZ));
    fbm3d_kernel<ORDER><<<grid, kThreads3, sizeof(Smem3), st>>>(a, out);
    return cudaGetLastError();
}

}  // namespace

void fbm3d_tile(int* tx, int* ty, int* tz) {
    *tx = kTX;
    *ty = kTY;
    *tz = kTZ;
}

cudaError_t fbm3d_launch(int order, const Fbm3Args& a, float* out, cudaStream_t st) {
    return order == 5 ? launch3<5>(a, out, st) : launch3<3>(a, out, st);
}

}  // namespace tg
