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
// Lattice selection needs no fp64: the four vertices the 2014 region logic
// picks include every vertex with 2 - |d|^2 > 0 (tests/test_opensimplex_geometry.py),
// so a pixel that an fp32 decision puts across a cell / region boundary only
// swaps a vertex whose attenuation is O(eps) there.  Each thread's group of
// kPX pixels of a row is located once in fp64 (u = (g + 0.5) fr, skew, floors);
// the other pixels step from it in fp32 and floor by a round-down add.  The
// four contributions of a pixel pair run in packed fp32x2 (FFMA2 / FMUL2 /
// FADD2, one issue slot for two pixels), the clamp is the saturate of a
// scalar FFMA.  Coarse octaves read 4-byte gradient entries (bf16 pairs) from
// a per-CTA vertex table (hashed once per CTA); fine octaves hash per lookup.
// 256 threads x 16 x 2 pixels, octaves innermost, one fp32 store per pixel.
#include <cuda_runtime.h>

#include "devattr.h"
#include "fbm_params.h"
#include "lattice.cuh"

namespace tg {
namespace {

constexpr uint64_t kSimplexLane = 0x8EBC6AF09C88C6E3ULL;
constexpr double kStretch = -0.211324865405187117745425609749;  // (1/sqrt(3) - 1)/2
constexpr double kSquish = 0.366025403784438646763723170753;    // (sqrt(3) - 1)/2

// Gradient index of the vertex with packed key `key` = top 3 bits of its
// hash (the final fmix64 xorshift leaves the high word alone).
__device__ __forceinline__ uint32_t grad_index_key(uint64_t key) {
    uint32_t lo, hi;
    mix64_pre(key ^ kMapLane(kSimplexLane), lo, hi);
    return hi >> 29;
}

// integral v, |v| < 2^31: the integer sits in the low mantissa word of v + 1.5*2^52
__device__ __forceinline__ int exact_int32(double v) {
    return __double2loint(v + 6755399441055744.0);
}

// floor of |x| < 2^22 by one round-down add: t = x + 1.5*2^23 holds floor(x)
// in its low mantissa bits (as an integer: bits(t) - kMagicBits) and t - 1.5*2^23
// is floor(x) as a float.
constexpr float kMagic = 12582912.0f;
constexpr uint32_t kMagicBits = 0x4B400000u;

// 4-byte vertex-table entry: the gradient's components as bf16 halves
// (+-5, +-2 are exact): x = bits & 0xffff0000, y = bits << 16.
__device__ __forceinline__ uint32_t grad_entry(float2 g) {
    return (__float_as_uint(g.x) & 0xFFFF0000u) | (__float_as_uint(g.y) >> 16);
}
// decode on the ALU pipe (LOP3, PRMT): the FMA pipes carry the fp32x2 math
__device__ __forceinline__ float entry_gx(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ float entry_gy(uint32_t w) { return __uint_as_float(__byte_perm(w, 0u, 0x1044)); }

// Contributions of one vertex slot to a pixel pair, (2 - |d|^2)^4 (g . d)
// with d = (dx, dy), in packed fp32x2 (FFMA2 / FMUL2 / FADD2: one issue slot
// for both pixels).
#ifndef TG_OS_SAT
#define TG_OS_SAT 1
#endif
// TG_OS_SAT: displacements carry a factor kDS = 1/sqrt(2), so a = 1 - |d'|^2 =
// attn / 2 and the clamp at zero is the saturate of the last scalar FFMA
// (FMA pipe) instead of two FMNMX (ALU pipe); attn^4 (g . d) = 16 sqrt(2) a^4
// (g . d') folds into the octave scale.
constexpr float kDS = TG_OS_SAT ? 0.70710678118654752f : 1.0f;
constexpr float kContribScale = TG_OS_SAT ? 22.627416997969522f : 1.0f;  // 16 sqrt(2)

__device__ __forceinline__ float2 contrib2(float2 dx, float2 dy, float2 gx, float2 gy, float2 v) {
#if TG_OS_SAT
    const float2 t = __ffma2_rn(dx, dx, make_float2(-1.0f, -1.0f));  // dx^2 - 1
    float2 m;
    m.x = __saturatef(fmaf(-dy.x, dy.x, -t.x));  // 1 - dx^2 - dy^2, clamped to [0, 1]
    m.y = __saturatef(fmaf(-dy.y, dy.y, -t.y));
#else
    const float2 m2 = make_float2(-2.0f, -2.0f);
    float2 m = __ffma2_rn(dx, dx, m2);
    m = __ffma2_rn(dy, dy, m);
    m.x = fminf(m.x, 0.0f);
    m.y = fminf(m.y, 0.0f);
#endif
    m = __fmul2_rn(m, m);
    m = __fmul2_rn(m, m);
    float2 dot = __fmul2_rn(gy, dy);
    dot = __ffma2_rn(gx, dx, dot);
    return __ffma2_rn(m, dot, v);
}

// The six region cases of the 2014 OpenSimplex (upper edge (2,0) / (0,2),
// upper interior (0,0), lower edge (1,-1) / (-1,1), lower interior (1,1)):
// the extra vertex's negated displacement and its lattice offset — as the
// index delta b*nx + a in a table octave's vertex table (one set per table
// octave), as the packed-key delta a*K3 + b*K4 for the hashed octaves.
struct CaseT {
    float nox, noy;
    int dext;  // b * nx + a for the octave's vertex table
    int pad;
};
struct CaseH {
    float nox, noy;
    uint32_t dlo, dhi;
};

constexpr int kTW = 128, kTH = 64, kThreads = 256;
#ifndef TG_OS_PX
#define TG_OS_PX 16
#endif
// a thread's pixel group: kPX consecutive pixels of a row (located once in
// fp64), kRows rows
constexpr int kPX = TG_OS_PX, kNP = kPX / 2, kCols = kTW / kPX, kRows = kTH * kCols / kThreads;
static_assert(kTW % kPX == 0 && kRows * kThreads == kTH * kCols, "tile");
constexpr int kTableMargin = 6;            // vertices beyond the tile's stretched range
#ifndef TG_OS_TABLE_KB
#define TG_OS_TABLE_KB 100
#endif
constexpr int kTableMaxBytes = TG_OS_TABLE_KB * 1024;  // per CTA, all table octaves together (4 B per vertex)

// Stretched-coordinate range of a tile: xs = u + (u + v) * kStretch with
// kStretch < 0, so xs is largest at (u1, v0) and smallest at (u0, v1); ys
// symmetric.  Table size bound: spans + margin (host and device agree).
__host__ __device__ inline void table_dims(double fr, int* nx, int* ny) {
    const double a = 1.0 + kStretch, b = -kStretch;  // 0.7887, 0.2113
    *nx = static_cast<int>(ceil((kTW * a + kTH * b) * fr)) + 2 * kTableMargin;
    *ny = static_cast<int>(ceil((kTH * a + kTW * b) * fr)) + 2 * kTableMargin;
}

// OctDev::mode bits of this kernel: a per-CTA vertex table; group stepping
constexpr int kOsTable = 1, kOsStep = 2;

struct TabPlan {
    double bx, by;  // table origin (integral)
};

// Region of one pixel from its in-cell coordinates: the case index (see
// CaseT) and whether it lies in the upper triangle.  Only the vertex SET
// matters: the 2014 geometry sums every vertex with 2 - |d|^2 > 0 (the four
// it picks include all of them), so near a region boundary the vertex that
// changes has attn ~ 0 there and an fp32 decision that lands in the
// neighbouring region changes the sum by O(eps^4) — no fp64 selection.
__device__ __forceinline__ int region_case(float xi, float yi, float s, bool& up) {
    up = s > 1.0f;
    const bool xgt = xi > yi;
    // lower: edge <=> s + min(xi, yi) < 1; upper: edge <=> s + max(xi, yi) > 2
    const float q = (up != xgt) ? yi : xi;
    const bool edge = (s + q > (up ? 2.0f : 1.0f)) == up;
    // case index (CaseT order): up ? (edge ? !xgt : 2) : 3 + (edge ? !xgt : 2)
    const int ce = edge ? (xgt ? 0 : 1) : 2;
    return up ? ce : ce + 3;
}

// A pixel located in fp64 (u = (g + 0.5) fr, the skew, both floors): its
// in-cell offset (fx, fy) in fp32 and its cell as the vertex-table index
// minus the magic bits (table octaves) or the packed key minus the magic
// offsets (hashed octaves), so that a later round-down-add floor of
// fx + dx gives the neighbouring cells by plain adds.
template <bool kTable>
__device__ __forceinline__ void os_locate(double gx, double gy, double fr, int nx, double bx, double by, uint64_t base,
                                          float& fx, float& fy, uint32_t& ib, uint64_t& kb) {
    const double u = __dmul_rn(gx, fr), v = __dmul_rn(gy, fr);
    const double so = __dmul_rn(__dadd_rn(u, v), kStretch);
    const double xs = __dadd_rn(u, so), ys = __dadd_rn(v, so);
    const double xb = floor(xs), yb = floor(ys);
    fx = __double2float_rn(__dsub_rn(xs, xb));
    fy = __double2float_rn(__dsub_rn(ys, yb));
    if (kTable)
        ib = static_cast<uint32_t>(exact_int32(yb - by) * nx + exact_int32(xb - bx)) - kMagicBits * (nx + 1u);
    else
        kb = pack_xy(base, __double2ll_rd(xb), __double2ll_rd(yb)) - static_cast<uint64_t>(kMagicBits) * (kIxMul + kIyMul);
}

// The four vertices of a pixel pair at stretched offsets (xs2, ys2) from
// their located cells (ib / kb per pixel): floor by a round-down add, region,
// the vertex gradients (table or hash), the contributions in fp32x2.
template <bool kTable>
__device__ __forceinline__ float2 os_pair(float2 xs2, float2 ys2, uint32_t ib0, uint32_t ib1, uint64_t kb0, uint64_t kb1,
                                          const uint32_t* ge, const CaseT* cst, const CaseH* csh, const uint32_t* tab,
                                          int nx) {
    constexpr float S = static_cast<float>(kSquish);
    constexpr float C1 = 1.0f + 2.0f * S;
    const float2 mg2 = make_float2(kMagic, kMagic), nmg2 = make_float2(-kMagic, -kMagic);
    const float2 tx = __fadd2_rd(xs2, mg2), ty = __fadd2_rd(ys2, mg2);
    const float2 m1 = make_float2(-1.0f, -1.0f);  // xs - floor(xs) = fma(floor, -1, xs)
    const float2 xi = __ffma2_rn(__fadd2_rn(tx, nmg2), m1, xs2);
    const float2 yi = __ffma2_rn(__fadd2_rn(ty, nmg2), m1, ys2);
    const float2 sum = __fadd2_rn(xi, yi);
    bool up0, up1;
    const int c0 = region_case(xi.x, yi.x, sum.x, up0);
    const int c1 = region_case(xi.y, yi.y, sum.y, up1);
    // displacement from the cell origin: (xi + s S, yi + s S)
    const float2 s2 = make_float2(S, S);
    const float2 sk2 = make_float2(S * kDS, S * kDS), k2 = make_float2(kDS, kDS);
    const float2 dx0 = __ffma2_rn(sum, sk2, TG_OS_SAT ? __fmul2_rn(xi, k2) : xi);
    const float2 dy0 = __ffma2_rn(sum, sk2, TG_OS_SAT ? __fmul2_rn(yi, k2) : yi);
    float2 gxa[4], gya[4];
    float2 nox3, noy3;  // negated displacement of the extra vertex
    if (kTable) {
        const CaseT e0 = cst[c0], e1 = cst[c1];
        nox3 = make_float2(e0.nox, e1.nox);
        noy3 = make_float2(e0.noy, e1.noy);
        const uint32_t i0 = ib0 + __float_as_uint(ty.x) * nx + __float_as_uint(tx.x);
        const uint32_t i1 = ib1 + __float_as_uint(ty.y) * nx + __float_as_uint(tx.y);
        const uint32_t w0[4] = {tab[i0 + 1], tab[i0 + nx], tab[i0 + (up0 ? nx + 1 : 0)], tab[i0 + e0.dext]};
        const uint32_t w1[4] = {tab[i1 + 1], tab[i1 + nx], tab[i1 + (up1 ? nx + 1 : 0)], tab[i1 + e1.dext]};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            gxa[k] = make_float2(entry_gx(w0[k]), entry_gx(w1[k]));
            gya[k] = make_float2(entry_gy(w0[k]), entry_gy(w1[k]));
        }
    } else {
        const CaseH e0 = csh[c0], e1 = csh[c1];
        nox3 = make_float2(e0.nox, e1.nox);
        noy3 = make_float2(e0.noy, e1.noy);
        const uint64_t k0 = kb0 + static_cast<uint64_t>(__float_as_uint(tx.x)) * kIxMul +
                            static_cast<uint64_t>(__float_as_uint(ty.x)) * kIyMul;
        const uint64_t k1 = kb1 + static_cast<uint64_t>(__float_as_uint(tx.y)) * kIxMul +
                            static_cast<uint64_t>(__float_as_uint(ty.y)) * kIyMul;
        const uint64_t d0 = (static_cast<uint64_t>(e0.dhi) << 32) | e0.dlo;
        const uint64_t d1 = (static_cast<uint64_t>(e1.dhi) << 32) | e1.dlo;
        const uint32_t g0[4] = {grad_index_key(add64(k0, kIxMul)), grad_index_key(add64(k0, kIyMul)),
                                grad_index_key(up0 ? add64(k0, kIxMul + kIyMul) : k0), grad_index_key(add64(k0, d0))};
        const uint32_t g1[4] = {grad_index_key(add64(k1, kIxMul)), grad_index_key(add64(k1, kIyMul)),
                                grad_index_key(up1 ? add64(k1, kIxMul + kIyMul) : k1), grad_index_key(add64(k1, d1))};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t a = ge[g0[k]], b = ge[g1[k]];
            gxa[k] = make_float2(entry_gx(a), entry_gx(b));
            gya[k] = make_float2(entry_gy(a), entry_gy(b));
        }
    }
    // vertices (1, 0), (0, 1), the triangle's own corner (c, c), the extra one
    constexpr float A1 = -(1.0f + S) * kDS, B1 = -S * kDS;
    const float2 nfc = make_float2(up0 ? -C1 * kDS : 0.0f, up1 ? -C1 * kDS : 0.0f);
    float2 nv = make_float2(0.0f, 0.0f);
    nv = contrib2(__fadd2_rn(dx0, make_float2(A1, A1)), __fadd2_rn(dy0, make_float2(B1, B1)), gxa[0], gya[0], nv);
    nv = contrib2(__fadd2_rn(dx0, make_float2(B1, B1)), __fadd2_rn(dy0, make_float2(A1, A1)), gxa[1], gya[1], nv);
    nv = contrib2(__fadd2_rn(dx0, nfc), __fadd2_rn(dy0, nfc), gxa[2], gya[2], nv);
    nv = contrib2(__fadd2_rn(dx0, nox3), __fadd2_rn(dy0, noy3), gxa[3], gya[3], nv);
    return nv;
}

// One octave for the thread's kPX consecutive pixels of a row (rows and
// octaves are rolled loops around it).  kStep: the group's first pixel is
// located in fp64 and the others step from it in fp32 (xs_j = fx + j fr(1 + St),
// ys_j = fy + j fr St; the host allows it where the step's rounding, ~ulp of
// j fr, stays far inside the tolerance); otherwise every pixel is located in
// fp64.  Lattice selection itself needs no fp64 (region_case).
template <bool kTable, bool kStep>
__device__ __forceinline__ void os_octave(float2 (&acc)[kNP], const uint32_t* ge, const CaseT* cst, const CaseH* csh,
                                          double fr, float amp, const uint32_t* tab, int nx, double bx, double by,
                                          uint64_t base, double gx0, double gy) {
    const float sc = amp * (kContribScale / 47.0f);
    if (kStep) {
        float fx, fy;
        uint32_t ib = 0;
        uint64_t kb = 0;
        os_locate<kTable>(gx0, gy, fr, nx, bx, by, base, fx, fy, ib, kb);
        const float ax = static_cast<float>(fr * (1.0 + kStretch)), ay = static_cast<float>(fr * kStretch);
        const float2 fx2 = make_float2(fx, fx), fy2 = make_float2(fy, fy);
        const float2 ax2 = make_float2(ax, ax), ay2 = make_float2(ay, ay);
#pragma unroll
        for (int p = 0; p < kNP; ++p) {
            const float2 jj = make_float2(2.0f * p, 2.0f * p + 1.0f);
            const float2 nv = os_pair<kTable>(__ffma2_rn(jj, ax2, fx2), __ffma2_rn(jj, ay2, fy2), ib, ib, kb, kb, ge,
                                              cst, csh, tab, nx);
            acc[p] = __ffma2_rn(make_float2(sc, sc), nv, acc[p]);
        }
    } else {
#pragma unroll 1
        for (int p = 0; p < kNP; ++p) {
            float fx0, fy0, fx1, fy1;
            uint32_t ib0 = 0, ib1 = 0;
            uint64_t kb0 = 0, kb1 = 0;
            os_locate<kTable>(gx0 + 2 * p, gy, fr, nx, bx, by, base, fx0, fy0, ib0, kb0);
            os_locate<kTable>(gx0 + 2 * p + 1, gy, fr, nx, bx, by, base, fx1, fy1, ib1, kb1);
            const float2 nv = os_pair<kTable>(make_float2(fx0, fx1), make_float2(fy0, fy1), ib0, ib1, kb0, kb1, ge, cst,
                                              csh, tab, nx);
            // rolled loop: the pair's accumulator by selects (no local memory)
#pragma unroll
            for (int q = 0; q < kNP; ++q)
                if (q == p) acc[q] = __ffma2_rn(make_float2(sc, sc), nv, acc[q]);
        }
    }
}

__global__ void __launch_bounds__(kThreads)
simplex2d_kernel(const __grid_constant__ FbmArgs args, float* __restrict__ out) {
    extern __shared__ uint32_t gtab[];
    __shared__ TabPlan plan[kMaxOctaves];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t tx0 = args.tile_x0 + static_cast<int64_t>(blockIdx.x) * kTW;
    const int64_t ty0 = args.tile_y0 + static_cast<int64_t>(blockIdx.y) * kTH;
    const uint64_t seed_key = args.seed_key[blockIdx.z];
    // table octaves (host plan: oct[o].mode != 0, goff = entry offset, ncx/ncy)
    if (threadIdx.x < args.octaves && (args.oct[threadIdx.x].mode & kOsTable)) {
        const OctDev& od = args.oct[threadIdx.x];
        const double fr = od.ratio;
        const double u0 = __dmul_rn(__dadd_rn(static_cast<double>(tx0), 0.5), fr);
        const double v0 = __dmul_rn(__dadd_rn(static_cast<double>(ty0), 0.5), fr);
        const double xs_min = u0 + (u0 + (v0 + kTH * fr)) * kStretch;
        const double ys_min = v0 + ((u0 + kTW * fr) + v0) * kStretch;
        plan[threadIdx.x] = {floor(xs_min) - kTableMargin, floor(ys_min) - kTableMargin};
    }
    // region cases: per table octave (index deltas in its table), and the
    // octave-independent packed-key deltas
    __shared__ CaseT cst[kMaxOctaves][6];
    __shared__ CaseH csh[6];
    constexpr int ea[6] = {2, 0, 0, 1, -1, 1}, eb[6] = {0, 2, 0, -1, 1, 1};
    for (int q = threadIdx.x; q < 6 * args.octaves; q += kThreads) {
        const int i = q % 6, o = q / 6;
        const float s = static_cast<float>(ea[i] + eb[i]) * static_cast<float>(kSquish);
        const float nox = -(static_cast<float>(ea[i]) + s) * kDS, noy = -(static_cast<float>(eb[i]) + s) * kDS;
        cst[o][i] = {nox, noy, eb[i] * args.oct[o].ncx + ea[i], 0};
        if (o == 0) {
            const uint64_t d = static_cast<uint64_t>(static_cast<int64_t>(ea[i])) * kIxMul +
                               static_cast<uint64_t>(static_cast<int64_t>(eb[i])) * kIyMul;
            csh[i] = {nox, noy, static_cast<uint32_t>(d), static_cast<uint32_t>(d >> 32)};
        }
    }
    // the 8 gradients (+-5, +-2) / (+-2, +-5) (bit 0 swaps, bits 1 / 2 negate x / y)
    // as packed bf16 entries
    __shared__ uint32_t ge[8];
    if (threadIdx.x < 8) {
        const int i = threadIdx.x;
        const float gxv = (i & 1) ? 2.0f : 5.0f, gyv = (i & 1) ? 5.0f : 2.0f;
        ge[i] = grad_entry(make_float2((i & 2) ? -gxv : gxv, (i & 4) ? -gyv : gyv));
    }
    __syncthreads();
    for (int o = 0; o < args.octaves; ++o) {
        const OctDev& od = args.oct[o];
        if (!(od.mode & kOsTable)) continue;
        const uint64_t base = seed_key + od.oct_key;
        uint32_t* t = gtab + od.goff;
        const int64_t bx = __double2ll_rd(plan[o].bx), by = __double2ll_rd(plan[o].by);
        for (int j = warp; j < od.ncy; j += kThreads / 32)  // one warp per table row
            for (int i = lane; i < od.ncx; i += 32)
                t[j * od.ncx + i] = ge[grad_index_key(pack_xy(base, bx + i, by + j))];
    }
    __syncthreads();
    const int c0 = (threadIdx.x % kCols) * kPX, r0 = (threadIdx.x / kCols) * kRows;
    const double gx0 = static_cast<double>(tx0 + c0) + 0.5;  // first pixel centre g + 0.5 (exact)
    const int64_t lx0 = tx0 + c0 - args.ox;
    float* out_map = out + static_cast<int64_t>(blockIdx.z) * args.map_stride;
#pragma unroll 1
    for (int r = 0; r < kRows; ++r) {
        const double gy = static_cast<double>(ty0 + r0 + r) + 0.5;
        float2 acc[kNP];
#pragma unroll
        for (int p = 0; p < kNP; ++p) acc[p] = make_float2(0.f, 0.f);
#pragma unroll 1
        for (int o = 0; o < args.octaves; ++o) {
            const OctDev& od = args.oct[o];
            const uint32_t* tab = gtab + od.goff;
            const uint64_t base = seed_key + od.oct_key;
            switch (od.mode) {
                case kOsTable | kOsStep:
                    os_octave<true, true>(acc, ge, cst[o], csh, od.ratio, od.amp, tab, od.ncx, plan[o].bx, plan[o].by, 0, gx0,
                                          gy);
                    break;
                case kOsStep:
                    os_octave<false, true>(acc, ge, cst[0], csh, od.ratio, od.amp, nullptr, 0, 0.0, 0.0, base, gx0, gy);
                    break;
                case kOsTable:
                    os_octave<true, false>(acc, ge, cst[o], csh, od.ratio, od.amp, tab, od.ncx, plan[o].bx, plan[o].by, 0,
                                           gx0, gy);
                    break;
                default:
                    os_octave<false, false>(acc, ge, cst[0], csh, od.ratio, od.amp, nullptr, 0, 0.0, 0.0, base, gx0, gy);
            }
        }
        const int64_t ly = ty0 + r0 + r - args.oy;
        if (ly >= 0 && ly < args.height) {
            float* row = out_map + ly * args.ld;
#pragma unroll
            for (int q = 0; q < kPX / 4; ++q) {
                const int64_t lx = lx0 + 4 * q;
                const float v[4] = {acc[2 * q].x, acc[2 * q].y, acc[2 * q + 1].x, acc[2 * q + 1].y};
                if (lx >= 0 && lx + 4 <= args.width && ((reinterpret_cast<uintptr_t>(row + lx) & 15) == 0)) {
                    *reinterpret_cast<float4*>(row + lx) = make_float4(v[0], v[1], v[2], v[3]);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (lx + j >= 0 && lx + j < args.width) row[lx + j] = v[j];
                }
            }
        }
    }
}

}  // namespace

cudaError_t simplex2d_launch(const FbmArgs& a, float* out, cudaStream_t st) {
    // Plan: an octave gets a per-CTA gradient table when its tile touches
    // fewer vertices than the 4 x 8192 per-pixel lookups would hash.
    FbmArgs p = a;
    // Stepping error (module comment): ~6e-7 * kPX * fr lattice units x the
    // noise slope (< 5) x amp; allowed where it stays under 1e-8 of the
    // amplitude sum (every octave together < 3.2e-7 of it, against the
    // 1e-5 * A parity bound).
    double amp_sum = 0.0;
    for (int o = 0; o < p.octaves; ++o) amp_sum += fabs(static_cast<double>(p.oct[o].amp));
    int bytes = 0;
    for (int o = 0; o < p.octaves; ++o) {
        OctDev& od = p.oct[o];
        od.mode = 0;
        const double fr = od.freq / p.R;
        od.ratio = fr;
        if (kPX * fr * fabs(static_cast<double>(od.amp)) <= amp_sum / 60.0) od.mode = kOsStep;
        int nx, ny;
        table_dims(fr, &nx, &ny);
        const int64_t n = static_cast<int64_t>(nx) * ny;
        if (n < 4 * kTW * kTH && bytes + 4 * n <= kTableMaxBytes) {
            od.mode |= kOsTable;
            od.ncx = nx;
            od.ncy = ny;
            od.goff = bytes / 4;  // entries
            bytes += static_cast<int>((4 * n + 15) / 16 * 16);
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
