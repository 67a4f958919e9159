// vgring.cu — the variogram by register-ring walks (config 5's lag set).
//
// The variogram is new (the reference has no variogram; BASELINE.json config 5
// asks for lags 1..4096 in powers of two, summed in fp64 over both axes).  Its
// cost is the fp64 pipe: every pair is DADD + DFMA on fp32 samples widened
// exactly to fp64.  The generic kernels in analysis.cu fetch one partner
// operand per pair from shared memory / L2 (8 B per pair as fp64), which caps
// them at half the fp64 rate.  Here every lag h = s * m with a stride class
// s in {1, 32, 1024} and m a power of two up to the ring size is summed by a
// WALK: a thread visits the positions q0, q0 + s, q0 + 2s, ... of one axis,
// widens each sample once, and keeps the last R samples in registers (an
// unrolled ring), so the pairs (k - m, k) of every m <= R come from registers:
// per sample 1 load + 1 conversion + (DADD + DFMA) per lag of the class.
//
//   class 0: s = 1,    m in {1, 2, 4, 8, 16}  (ring of 16)   lags 1 .. 16
//   class 1: s = 32,   m in {1, 2, 4, 8, 16}  (ring of 16)   lags 32 .. 512
//   class 2: s = 1024, m in {1, 2, 4}         (ring of 4)    lags 1024 .. 4096
//
// Six walk kinds (3 classes x 2 axes), each its own kernel of warp-level
// work items reading global memory through a per-warp cp.async staging ring
// (no barriers; one walk's loop per SM at a time keeps the instruction cache
// warm — the six kinds mixed in one grid stalled 25 % on instruction fetch):
//   X0  lane = row (32 rows), 512 consecutive columns, 16-byte copies
//   X1  lane = residue (one row), columns rho + 32 k, 128-byte warp copies
//   X2  lane = residue, 2 residues per lane (rho + 512 i), columns rho + 1024 k
//   Y0  lane = column (32 columns), 512 consecutive rows
//   Y1  lane = column, rows rho + 32 k;   Y2  lane = column, rows rho + 1024 k
// Each kind reads the map once (config 5: 6 x 4.3 GB); classes 0/1 run at
// ~55-60 % of the fp64 pipe, class 2 is HBM-bound.  Tried and measured slower
// (profiles/r02_variogram.md): one mixed grid (I-cache), per-row CTAs running
// the three x walks side by side (L2 reuse did not materialise: 2.5 reads),
// shared-memory row segments filled by bulk copies (3 warps per SMSP, barrier
// imbalance between the classes).
// A pair is owned by its SECOND point (the partner), so a walk needs only the
// R samples before its first step (pre-fill), never an apron after it.
// Lag sets the ring path cannot express fall back to the generic kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "devattr.h"

namespace tg {
int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);

namespace {

constexpr int kStride1 = 32, kStride2 = 1024;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kL = 512;
#ifndef TG_VGR_NS2
#define TG_VGR_NS2 2
#endif
constexpr int kNS2 = TG_VGR_NS2;  // class-2 sequences per lane (residues 1024 / kNS2 apart)
constexpr int kYG = 16;           // Y2 residue groups per item  // steps per X0 / X1 / Y0 / Y1 item
#ifndef TG_VGR_MINB
#define TG_VGR_MINB 2
#endif

struct RingPlan {
    uint32_t mask[3];  // bit j: lag stride_c << j requested
    int slot[3][5];    // index of that lag in the caller's list (first occurrence), -1 if absent
};

// Item counts.  x: X0 nx0 column segments per 32-row band, X1 nx1 segments
// per row, X2 one item per row (nx2 != 0: class present).  y, per 32-column
// strip: Y0 ny0 row segments, Y1 32 residues x ny1 segments, Y2 ny2 residue
// groups.  hw[c]: partner-row bound of class c on the y axis.
struct WalkPlan {
    int64_t nx0, nx1, nx2;
    int64_t ny0, ny1, ny2;
    int64_t hw[3];
};

__device__ __forceinline__ int clamp_step(int64_t v) {
    return static_cast<int>(v < -(int64_t(1) << 30) ? -(int64_t(1) << 30) : v > (int64_t(1) << 30) ? (int64_t(1) << 30) : v);
}

// ceil(a / b) for b > 0, any sign of a
__device__ __forceinline__ int64_t cdiv(int64_t a, int64_t b) { return a >= 0 ? (a + b - 1) / b : -((-a) / b); }

// Per-warp staging of the walks' samples: cp.async (LDGSTS) copies of the
// next two chunks are in flight while one is summed, without holding
// registers.  Layout per stage: [seq][step][lane] floats (each lane reads back
// only what it copied: no warp synchronisation), or for the contiguous X0 walk
// [lane][R + 4] (16-byte copies, conflict-free 16-byte reads).
#ifndef TG_VGR_STAGES
#define TG_VGR_STAGES 4
#endif
constexpr int kStages = TG_VGR_STAGES;  // chunks staged per warp (kStages - 1 in flight)
constexpr int kStageFloats = 32 * 20;  // >= NS * R * 32 and 32 * (16 + 4)
__device__ __forceinline__ void cp_async4z(uint32_t dst, const float* src, bool ok) {  // zero-filled if !ok
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const float* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// NS sequences walked in lockstep over the steps [ka, kb) (chunks of R aligned
// to ka, ka a multiple of R).  Sequence i's step k is b[i][k * sstride] for k
// in [0, nk[i]) (other steps stage as 0 and never pair), axis position
// rho[i] + s k with 0 <= rho < s.  Pair (k - m, k) counts when
// k < min(kb, nk[i]), k >= m (first point >= 0) and k - m < kp[i] (the first
// point's row < P on the y axis; kp = 2^30 on the x axis).  acc[j] sums lag
// s << j.  Two rings of R samples per sequence alternate roles chunk by chunk
// (the previous chunk and the one being filled), so no sample is ever moved
// between registers.  VEC4: steps contiguous and 16-byte aligned (X0);
// SSTRIDE > 0: sstride known at compile time (x axis: immediate offsets).
template <int R, int NS, int NM, bool ALL, bool VEC4, int SSTRIDE>
__device__ __forceinline__ void walk(float* stage, const float* const (&b)[NS], const int64_t (&nk)[NS],
                                     const int (&kp)[NS], int64_t sstride, int ka, int kb, uint32_t mask,
                                     double (&acc)[NM]) {
    static_assert(NS * R * 32 <= kStageFloats && (!VEC4 || NS == 1), "stage size");
    const int lane = threadIdx.x & 31;
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(stage));
    auto soff = [&](int i, int u) { return VEC4 ? lane * (R + 4) + u : (i * R + u) * 32 + lane; };
    // stage chunk q (steps ka + q R ..) into stage slot (q + 1) % kStages
    auto issue = [&](int q) {
        const int k0 = ka + q * R;
        const uint32_t dst = sbase + static_cast<uint32_t>(((q + 1 + kStages) % kStages) * kStageFloats) * 4u;
        if (k0 < kb) {
#pragma unroll
            for (int i = 0; i < NS; ++i) {
                if (VEC4) {
#pragma unroll
                    for (int u = 0; u < R; u += 4) {
                        const int k = k0 + u;
                        if (k >= 0 && k + 4 <= nk[i]) {
                            cp_async16(dst + 4u * soff(i, u), b[i] + k, true);
                        } else {  // ragged end (or before the start): element copies, zero-filled
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const bool in = k + e >= 0 && k + e < nk[i];
                                cp_async4z(dst + 4u * (soff(i, u) + e), b[i] + (in ? k + e : 0), in);
                            }
                        }
                    }
                } else if (k0 >= 0 && k0 + R <= nk[i]) {  // whole chunk present: no per-element tests
                    const float* p = b[i] + k0 * sstride;
                    const uint32_t d = dst + 4u * soff(i, 0);
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        if (SSTRIDE > 0)
                            cp_async4(d + 128u * u, p + u * SSTRIDE);
                        else
                            cp_async4(d + 128u * u, p), p += sstride;
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        const int k = k0 + u;
                        const bool ok = k >= 0 && k < nk[i];
                        cp_async4z(dst + 4u * soff(i, u), b[i] + (ok ? k : 0) * sstride, ok);
                    }
                }
            }
        }
        cp_commit();  // (possibly empty) group per chunk keeps the wait counts uniform
    };
    int lim = kb;  // chunks ending at or before lim have every pair valid (but k >= m)
#pragma unroll
    for (int i = 0; i < NS; ++i) lim = min(lim, min(static_cast<int>(nk[i] < kb ? nk[i] : kb), kp[i] + 1));
    auto slot = [&](int q) { return stage + ((q + 1 + kStages) % kStages) * kStageFloats; };
    // chunk q: prev = ring of steps k0 - R .., cur <- this chunk's samples
    auto chunk = [&](int q, const double (&prev)[NS][R], double (&cur)[NS][R]) {
        const int k0 = ka + q * R;
        const float* sp = slot(q);
        if (VEC4) {
#pragma unroll
            for (int u = 0; u < R; u += 4) {
                const float4 t = *reinterpret_cast<const float4*>(sp + soff(0, u));
                cur[0][u] = t.x, cur[0][u + 1] = t.y, cur[0][u + 2] = t.z, cur[0][u + 3] = t.w;
            }
        } else {
#pragma unroll
            for (int i = 0; i < NS; ++i)
#pragma unroll
                for (int u = 0; u < R; ++u) cur[i][u] = static_cast<double>(sp[soff(i, u)]);
        }
        // every pair counts (FIRST: the sequence start, pairs with k < m skipped at
        // compile time; unrolled for the short class-2 rings only, whose first
        // chunk is 1 in 8 at config 5 — the 16-rings take the compact path there)
        auto body = [&](auto first_c) {
            constexpr bool FIRST = decltype(first_c)::value;
#pragma unroll
            for (int u = 0; u < R; ++u)
#pragma unroll
                for (int i = 0; i < NS; ++i)
#pragma unroll
                    for (int j = 0; j < NM; ++j) {
                        const int m = 1 << j;
                        if (!(ALL || ((mask >> j) & 1u))) continue;
                        if (FIRST && u < m) continue;
                        const double d = cur[i][u] - (u - m >= 0 ? cur[i][u - m] : prev[i][u - m + R]);
                        acc[j] = fma(d, d, acc[j]);
                    }
        };
        if (k0 + R <= lim && k0 != 0) {
            body(std::false_type{});
        } else if (R <= 4 && k0 + R <= lim) {
            body(std::true_type{});
        } else {
            // sequence start or edge chunk (rare): compact loop over the staged
            // fp32 samples of this chunk and the previous one, every pair tested
            const float* pp = slot(q - 1);
#pragma unroll 1
            for (int u = 0; u < R; ++u) {
                const int k = k0 + u;
#pragma unroll
                for (int i = 0; i < NS; ++i) {
                    const double v = static_cast<double>(sp[soff(i, u)]);
                    const bool in = k < kb && k < nk[i];
#pragma unroll
                    for (int j = 0; j < NM; ++j) {
                        const int m = 1 << j;
                        if (((mask >> j) & 1u) && in && k >= m && k - m < kp[i]) {
                            const double d = v - static_cast<double>(u >= m ? sp[soff(i, u - m)] : pp[soff(i, u - m + R)]);
                            acc[j] = fma(d, d, acc[j]);
                        }
                    }
                }
            }
        }
    };
    auto step = [&](int q, const double (&prev)[NS][R], double (&cur)[NS][R]) {
        cp_wait<kStages - 2>();  // chunk q has landed (q + 1 .. may still be in flight)
        chunk(q, prev, cur);
        issue(q + kStages - 1);  // into the slot of chunk q - 1 (read by chunk q's edge path)
    };
    double ra[NS][R], rb[NS][R];
#pragma unroll
    for (int q = -1; q < kStages - 1; ++q) issue(q);
    cp_wait<kStages - 1>();
#pragma unroll
    for (int i = 0; i < NS; ++i)
#pragma unroll
        for (int u = 0; u < R; ++u) ra[i][u] = static_cast<double>(slot(-1)[soff(i, u)]);
    for (int q = 0; ka + q * R < kb; q += 2) {
        step(q, ra, rb);
        if (ka + (q + 1) * R >= kb) break;
        step(q + 1, rb, ra);
    }
    cp_wait<0>();  // the stage is reused by the warp's next walk
}

// Walk entry points of the six item kinds.
struct Acc5 {
    double a[5];
};
struct Acc3 {
    double a[3];
};

// kp: first-point limit in steps (y axis: ceil((P - rho) / s); x axis: 2^30).
template <bool ALL, bool VEC4, int SSTRIDE>
__device__ __forceinline__ Acc5 walk16(float* stage, const float* b0, int64_t nk0, int kp0, int64_t sstride, int ka,
                                    int kb, uint32_t mask) {
    double acc[5] = {0, 0, 0, 0, 0};
    const float* const b[1] = {b0};
    const int64_t nk[1] = {nk0};
    const int kp[1] = {kp0};
    walk<16, 1, 5, ALL, VEC4, SSTRIDE>(stage, b, nk, kp, sstride, ka, kb, mask, acc);
    return Acc5{{acc[0], acc[1], acc[2], acc[3], acc[4]}};
}

// Class 2 (s = 1024): ng groups of kNS2 sequences; group t walks residues
// rho0 + t * gstep + (1024 / kNS2) i (bases b0 + t * gstep * estep +
// i * (1024 / kNS2) * estep), positions rho + 1024 k < lim, all their steps;
// y axis (ycheck): first points < P.  estep: elements per axis position.
template <bool ALL, int SSTRIDE>
__device__ __forceinline__ Acc3 walk4xN(float* stage, const float* b0, int64_t estep, int rho0, int gstep, int ng,
                                     int64_t lim, bool ycheck, int64_t P, uint32_t mask) {
    double acc[3] = {0, 0, 0};
    for (int t = 0; t < ng; ++t) {
        const float* b[kNS2];
        int64_t nk[kNS2];
        int kp[kNS2];
        int64_t kmax = 0;
#pragma unroll
        for (int i = 0; i < kNS2; ++i) {
            const int rho = rho0 + t * gstep + kStride2 / kNS2 * i;
            b[i] = b0 + static_cast<int64_t>(rho - rho0) * estep;
            nk[i] = std::max<int64_t>(0, cdiv(lim - rho, kStride2));
            kp[i] = ycheck ? clamp_step(cdiv(P - rho, kStride2)) : (1 << 30);
            kmax = std::max(kmax, nk[i]);
        }
        if (kmax > 0)
            walk<4, kNS2, 3, ALL, false, SSTRIDE>(stage, b, nk, kp, kStride2 * estep, 0,
                                         static_cast<int>((kmax + 3) & ~int64_t(3)), mask, acc);
    }
    return Acc3{{acc[0], acc[1], acc[2]}};
}

// One kernel per item kind (each SM then runs one walk's loop at a time: the
// six kinds mixed in one grid thrashed the instruction cache).
enum Kind { kX0, kX1, kX2, kY0, kY1, kY2 };
template <int KIND, bool ALL>
__global__ void __launch_bounds__(kThreads, TG_VGR_MINB)
vg_walk(const float* __restrict__ z, int64_t W, int64_t ld, int64_t P, bool vec, const __grid_constant__ RingPlan plan,
        const __grid_constant__ WalkPlan wp, double* __restrict__ sums) {
    constexpr int AX = KIND >= kY0 ? 1 : 0, C = KIND % 3, NM = C == 2 ? 3 : 5;
    __shared__ double part_s[kWarps][8];
    extern __shared__ __align__(16) float stage_s[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* const stage = stage_s + warp * kStages * kStageFloats;
    const uint32_t mask = plan.mask[C];
    double tot[NM];
#pragma unroll
    for (int j = 0; j < NM; ++j) tot[j] = 0.0;
    const int64_t items = KIND == kX0 ? ((P + 31) / 32) * wp.nx0
                          : KIND == kX1 ? P * wp.nx1
                          : KIND == kX2 ? P
                          : KIND == kY0 ? ((W + 31) / 32) * wp.ny0
                          : KIND == kY1 ? ((W + 31) / 32) * 32 * wp.ny1
                                        : ((W + 31) / 32) * wp.ny2;
    const int64_t wid = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * kThreads) >> 5;
    for (int64_t it = wid; it < items; it += nw) {
        double a[NM];
#pragma unroll
        for (int j = 0; j < NM; ++j) a[j] = 0.0;
        if constexpr (KIND == kX0) {  // lane = row, columns [512 r, 512 r + 512)
            const int64_t band = it / wp.nx0, r = it - band * wp.nx0;
            const int64_t row = 32 * band + lane;
            if (row < P) {
                const int ka = static_cast<int>(r * kL);
                const int kb = static_cast<int>(std::min<int64_t>(ka + kL, W));
                const Acc5 t = vec ? walk16<ALL, true, 0>(stage, z + row * ld, W, 1 << 30, 1, ka, kb, mask)
                                   : walk16<ALL, false, 0>(stage, z + row * ld, W, 1 << 30, 1, ka, kb, mask);
#pragma unroll
                for (int j = 0; j < NM; ++j) a[j] = t.a[j];
            }
        } else if constexpr (KIND == kX1) {  // one row, lane = residue, columns lane + 32 k
            const int64_t row = it / wp.nx1, r = it - row * wp.nx1;
            const int ka = static_cast<int>(r * kL);
            const int64_t n = std::max<int64_t>(0, cdiv(W - lane, kStride1));
            const int kb = static_cast<int>(std::max<int64_t>(ka, std::min<int64_t>(ka + kL, n)));
            const Acc5 t = walk16<ALL, false, 0>(stage, z + row * ld + lane, n, 1 << 30, kStride1, ka, kb, mask);
#pragma unroll
            for (int j = 0; j < NM; ++j) a[j] = t.a[j];
        } else if constexpr (KIND == kX2) {  // one row, residues 32 t + lane + (1024 / kNS2) i, columns rho + 1024 k
            const Acc3 t = walk4xN<ALL, 0>(stage, z + it * ld + lane, 1, lane, 32, kStride2 / 32 / kNS2, W, false, P, mask);
#pragma unroll
            for (int j = 0; j < NM; ++j) a[j] = t.a[j];
        } else {
            const int64_t per = KIND == kY0 ? wp.ny0 : KIND == kY1 ? 32 * wp.ny1 : wp.ny2;
            const int64_t g = it / per, r = it - g * per;
            const int64_t col = 32 * g + lane;
            if (col < W) {
                const float* base = z + col;
                if constexpr (KIND == kY0) {  // rows [512 r, 512 r + 512) of the partner range
                    const int64_t hw = wp.hw[0];
                    const int ka = static_cast<int>(r * kL);
                    const int kb = static_cast<int>(std::min<int64_t>(ka + kL, hw));
                    const Acc5 t = walk16<ALL, false, 0>(stage, base, hw, clamp_step(P), ld, ka, kb, mask);
#pragma unroll
                    for (int j = 0; j < NM; ++j) a[j] = t.a[j];
                } else if constexpr (KIND == kY1) {  // rows rho + 32 k
                    const int rh = static_cast<int>(r / wp.ny1);
                    const int ka = static_cast<int>((r % wp.ny1) * kL);
                    const int64_t n = std::max<int64_t>(0, cdiv(wp.hw[1] - rh, kStride1));
                    if (ka < n) {
                        const int kb = static_cast<int>(std::min<int64_t>(ka + kL, n));
                        const Acc5 t = walk16<ALL, false, 0>(stage, base + rh * ld, n, clamp_step(cdiv(P - rh, kStride1)),
                                                             kStride1 * ld, ka, kb, mask);
#pragma unroll
                        for (int j = 0; j < NM; ++j) a[j] = t.a[j];
                    }
                } else {  // Y2: rows rho + 1024 k, rho = kYG r + t + (1024 / kNS2) i, t < kYG
                    const Acc3 t = walk4xN<ALL, 0>(stage, base + kYG * r * ld, ld, static_cast<int>(kYG * r), 1, kYG,
                                                   wp.hw[2], true, P, mask);
#pragma unroll
                    for (int j = 0; j < NM; ++j) a[j] = t.a[j];
                }
            }
        }
#pragma unroll
        for (int j = 0; j < NM; ++j) tot[j] += a[j];
    }
    // CTA sum of the lane totals, one fp64 atomic per lag
#pragma unroll
    for (int j = 0; j < NM; ++j) {
        double v = tot[j];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) part_s[warp][j] = v;
    }
    __syncthreads();
    if (threadIdx.x < NM) {
        const int j = threadIdx.x, slot = plan.slot[C][j];
        if (slot >= 0) {
            double t = 0.0;
            for (int w = 0; w < kWarps; ++w) t += part_s[w][j];
            atomicAdd(&sums[2 * slot + AX], t);
        }
    }
}

}  // namespace

// Host entry from tg_variogram_band_f32: returns 1 when the lag set is not
// expressible by the ring walks (caller uses the generic kernels), 0 when the
// kernel was enqueued on s, or a negative TG status.
int vg_ring_enqueue(const float* z, int64_t W, int64_t H, int64_t ld, int64_t P, const int32_t* lags, int n_lags,
                    double* sums, int sm, cudaStream_t s, cudaStream_t sy) {
    if (getenv("TG_VG_GENERIC")) return 1;  // timing / cross-check switch
    RingPlan plan{};
    for (auto& c : plan.slot)
        for (int& v : c) v = -1;
    for (int i = 0; i < n_lags; ++i) {
        const int64_t h = lags[i];
        if (h < 1 || h > 4096 || (h & (h - 1))) return 1;
        const int c = h <= 16 ? 0 : h <= 512 ? 1 : 2;
        const int64_t st = c == 0 ? 1 : c == 1 ? kStride1 : kStride2;
        const int j = __builtin_ctzll(static_cast<uint64_t>(h / st));
        if (plan.slot[c][j] < 0) plan.slot[c][j] = i;  // a repeated lag is summed once; the caller copies it
        plan.mask[c] |= 1u << j;
    }
    static const int axes = getenv("TG_VG_AXES") ? atoi(getenv("TG_VG_AXES")) : 3;  // timing experiments
    if (P <= 0) return 0;
    WalkPlan wp{};
    if (axes & 1) {
        wp.nx0 = plan.mask[0] ? (W + kL - 1) / kL : 0;
        wp.nx1 = plan.mask[1] ? ((W + kStride1 - 1) / kStride1 + kL - 1) / kL : 0;  // segments per row
        wp.nx2 = plan.mask[2] ? 32 : 0;
    }
    if (axes & 2) {
        const int64_t st[3] = {1, kStride1, kStride2};
        for (int c = 0; c < 3; ++c) {
            const int64_t mm = plan.mask[c] ? (int64_t(1) << (31 - __builtin_clz(plan.mask[c]))) : 0;
            wp.hw[c] = std::min<int64_t>(H, P + st[c] * mm);
        }
        wp.ny0 = plan.mask[0] ? (wp.hw[0] + kL - 1) / kL : 0;
        wp.ny1 = plan.mask[1] ? ((wp.hw[1] + kStride1 - 1) / kStride1 + kL - 1) / kL : 0;  // per residue
        wp.ny2 = plan.mask[2] ? kStride2 / kNS2 / kYG : 0;
    }
    const bool all = plan.mask[0] == 31u && plan.mask[1] == 31u && plan.mask[2] == 7u;
    const bool vec = (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(z) & 15) == 0;
    static const int per_sm = getenv("TG_VGR_GRID") ? atoi(getenv("TG_VGR_GRID")) : TG_VGR_MINB;
    const size_t smem = static_cast<size_t>(kWarps) * kStages * kStageFloats * sizeof(float);
    using K = void (*)(const float*, int64_t, int64_t, int64_t, bool, RingPlan, WalkPlan, double*);
    static const K kt[2][6] = {
        {vg_walk<kX0, false>, vg_walk<kX1, false>, vg_walk<kX2, false>, vg_walk<kY0, false>, vg_walk<kY1, false>,
         vg_walk<kY2, false>},
        {vg_walk<kX0, true>, vg_walk<kX1, true>, vg_walk<kX2, true>, vg_walk<kY0, true>, vg_walk<kY1, true>,
         vg_walk<kY2, true>}};
    static PerDeviceOnce attr;
    cudaError_t e = attr.run([&] {
        cudaError_t r = cudaSuccess;
        for (auto& row : kt)
            for (K f : row)
                if (r == cudaSuccess) r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        return r;
    });
    if (e != cudaSuccess) return set_cuda_error(e, "variogram walks smem opt-in");
    const int64_t strips = (W + 31) / 32;
    const int64_t items[6] = {((P + 31) / 32) * wp.nx0, P * wp.nx1, wp.nx2 ? P : 0,
                              strips * wp.ny0, strips * 32 * wp.ny1, strips * wp.ny2};
    for (int kd = 0; kd < 6; ++kd) {
        if (items[kd] == 0) continue;
        const int64_t grid =
            std::max<int64_t>(1, std::min<int64_t>((items[kd] + kWarps - 1) / kWarps, per_sm * static_cast<int64_t>(sm)));
        // the HBM-bound class-2 walks (kinds 2, 5) on the side stream beside the
        // fp64-bound classes 0 / 1 when the caller forked one (TG_VG_CONCURRENT)
        kt[all ? 1 : 0][kd]<<<static_cast<unsigned>(grid), kThreads, smem, (kd == 2 || kd == 5) ? sy : s>>>(
            z, W, ld, P, vec, plan, wp, sums);
        if ((e = cudaGetLastError()) != cudaSuccess) return set_cuda_error(e, "variogram walks");
    }
    return 0;
}

}  // namespace tg
