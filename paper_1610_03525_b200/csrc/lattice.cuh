// lattice.cuh — seeded corner data on the device (terrain/lattice.hpp:16-83).
//
// Bit-exact with the reference: the packed key (lattice.hpp:46-50) and the
// murmur3 fmix64 finalizer (lattice.hpp:35-42) run on 32-bit integer
// hardware as 64-bit wrap-around arithmetic.  Heights are produced as
// float(corner_height) rounded to nearest: the reference's double
// to_unit(z)*2-1 equals t * 2^-52 with t = (int64)(z ^ 2^63) >> 11 exactly,
// so one s64->f32 conversion rounds the exact value once.
#pragma once

#include <cstdint>

#ifndef TG_MAP_HEIGHT_HI
#define TG_MAP_HEIGHT_HI 1
#endif
// TG_MAP_SIGNED=1 (default): signed top word (sign flip in the last IMAD.HI
// addend, I2FP.S32), height = f * 2^-31 with no per-octave offset, so the
// fp32 partial sums stay at the magnitude of the map itself and the absolute
// error scales with the window's own amplitude (north-star 1e-5 * A in every
// 64 x 64 window, tests/test_gpu_fullshape.py).  0: unsigned word + the
// -sum(amp) offset (FbmArgs::hoff) — the partial sums then run near 2 sum(amp)
// and a low-amplitude window exceeds 1e-5 * A.
#ifndef TG_MAP_SIGNED
#define TG_MAP_SIGNED 1
#endif

namespace tg {

constexpr uint64_t kSeedMul = 0x9E3779B97F4A7C15ULL;  // lattice.hpp:47
constexpr uint64_t kOctMul = 0xBF58476D1CE4E5B9ULL;   // lattice.hpp:47
constexpr uint64_t kIxMul = 0x94D049BB133111EBULL;    // lattice.hpp:48
constexpr uint64_t kIyMul = 0xD6E8FEB86659FD93ULL;    // lattice.hpp:49
constexpr uint64_t kIzMul = 0xA24BAED4963EE407ULL;    // 3D extension (TG_PACK_K5, new)
constexpr uint64_t kAngleLane = 0xA0761D6478BD642FULL;      // lattice.hpp:53
constexpr uint64_t kMagnitudeLane = 0xE7037ED1A0B428DBULL;  // lattice.hpp:54

// z *= M (mod 2^64) on 32-bit halves in exactly three IMADs: the wide
// product of the low words, then both cross terms accumulated into its high
// word.  Inline PTX keeps ptxas from re-associating into four instructions.
#define TG_MUL64(lo, hi, ML, MH)                                                     \
    do {                                                                             \
        uint32_t plo_, phi_;                                                         \
        asm("{\n\t.reg .b64 p;\n\tmul.wide.u32 p, %2, " #ML ";\n\t"                 \
            "mov.b64 {%0, %1}, p;\n\tmad.lo.u32 %1, %3, " #ML ", %1;\n\t"           \
            "mad.lo.u32 %1, %2, " #MH ", %1;\n\t}"                                  \
            : "=r"(plo_), "=r"(phi_)                                                 \
            : "r"(lo), "r"(hi));                                                     \
        lo = plo_;                                                                   \
        hi = phi_;                                                                   \
    } while (0)

// lattice.hpp:35-42 (murmur3 fmix64) up to, but excluding, the final
// xorshift: z ^= z >> 33 only touches the low word (lo ^= hi >> 1).
__device__ __forceinline__ void mix64_pre(uint64_t z, uint32_t& lo, uint32_t& hi) {
    lo = static_cast<uint32_t>(z);
    hi = static_cast<uint32_t>(z >> 32);
    lo ^= hi >> 1;
    TG_MUL64(lo, hi, 0xED558CCD, 0xFF51AFD7);
    lo ^= hi >> 1;
    TG_MUL64(lo, hi, 0x1A85EC53, 0xC4CEB9FE);
}

// lattice.hpp:35-42 — the full 64-bit finalizer.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    uint32_t lo, hi;
    mix64_pre(z, lo, hi);
    lo ^= hi >> 1;
    return (static_cast<uint64_t>(hi) << 32) | lo;
}

// 64-bit add kept as IADD3 + IADD3.X (stops ptxas from re-deriving per-pixel
// keys with extra wide multiplies).
__device__ __forceinline__ uint64_t add64(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.u64 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

// lattice.hpp:46-50 split as pack = base + ix*K3 + iy*K4 with
// base = seed*K1 + octave*K2 hoisted per octave.  ix/iy are signed 64-bit and
// wrap two's-complement exactly like the reference's static_cast<uint64_t>.
__device__ __forceinline__ uint64_t pack_xy(uint64_t base, int64_t ix, int64_t iy) {
    return base + static_cast<uint64_t>(ix) * kIxMul + static_cast<uint64_t>(iy) * kIyMul;
}

// corner_height scaled by 2^63 as an exact-rounding float:
//   corner_height = (z >> 11)*2^-52 - 1 = t*2^-52,  t = (int64)(z ^ 2^63) >> 11,
// and RN(t * 2^11) = RN(t) * 2^11, so converting (z ^ 2^63) with its low 11
// bits cleared rounds the exact reference value once.  The caller multiplies
// by amp * 2^-63 (a power-of-two rescale, exact).  The clear folds into the
// final xorshift: one LOP3 computes (lo ^ (hi >> 1)) & ~0x7ff.
__device__ __forceinline__ float height_scaled_from_pre(uint32_t lo, uint32_t hi) {
    const uint32_t l = (lo ^ (hi >> 1)) & 0xFFFFF800u;
    float f;
    // one LOP3 for the sign flip of the high word, then s64 -> f32 (RN)
    asm("{\n\t.reg .b32 h;\n\t.reg .b64 v;\n\txor.b32 h, %2, 0x80000000;\n\t"
        "mov.b64 v, {%1, h};\n\tcvt.rn.f32.s64 %0, v;\n\t}"
        : "=f"(f)
        : "r"(l), "r"(hi));
    return f;
}

// Four independent keys in lock step: the same 12-instruction chain per key,
// interleaved in program order so each warp has 4-way instruction-level
// parallelism through the 4-5 cycle IMAD/ALU latencies (a single fmix64
// chain is fully serial).
__device__ __forceinline__ void height_scaled4(uint64_t p0, uint64_t p1, uint64_t p2, uint64_t p3,
                                              float (&out)[4]) {
    uint32_t l[4] = {static_cast<uint32_t>(p0), static_cast<uint32_t>(p1), static_cast<uint32_t>(p2),
                     static_cast<uint32_t>(p3)};
    uint32_t h[4] = {static_cast<uint32_t>(p0 >> 32), static_cast<uint32_t>(p1 >> 32),
                     static_cast<uint32_t>(p2 >> 32), static_cast<uint32_t>(p3 >> 32)};
#pragma unroll
    for (int i = 0; i < 4; ++i) l[i] ^= h[i] >> 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) TG_MUL64(l[i], h[i], 0xED558CCD, 0xFF51AFD7);
#pragma unroll
    for (int i = 0; i < 4; ++i) l[i] ^= h[i] >> 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) TG_MUL64(l[i], h[i], 0x1A85EC53, 0xC4CEB9FE);
#pragma unroll
    for (int i = 0; i < 4; ++i) out[i] = height_scaled_from_pre(l[i], h[i]);
}

__device__ __forceinline__ float height_scaled(uint64_t packed) {
    uint32_t lo, hi;
    mix64_pre(packed, lo, hi);
    return height_scaled_from_pre(lo, hi);
}

// Map-path corner height from the top word of fmix64 only.  The final
// xorshift (z ^= z >> 33) touches only the low word, and the second multiply
// needs only its high word (mul.hi of the low words plus both cross terms).
//
// Signed form (TG_MAP_SIGNED=1, default).  Map-path keys carry a +2^63 bias
// (kMapKeyBias, added to seed*K1 by the host planner, so every key the
// kernels derive from it carries it): with hi' = hi ^ 2^31,
//   * the xorshifts read lo ^= (hi' >> 1) ^ 2^30 — the same value, the 2^30
//     riding free in the 3-input LOP3;
//   * the first multiply's high word comes out as hi1 + 2^31 (the cross term
//     hi' * C1lo = hi * C1lo + 2^31, C1lo odd), i.e. the flipped hi1' again;
//   * the last multiply's top word likewise comes out as t + 2^31 = t ^ 2^31.
// Read as int32, t ^ 2^31 = floor(corner_height * 2^31): the map height is
// float(int32) * 2^-31 with no per-octave offset and no extra instruction, so
// fp32 partial sums stay at the magnitude of the map itself and the absolute
// error scales with each window's own amplitude (tests/test_gpu_fullshape.py
// checks 1e-5 * A in every 64 x 64 window).  Lanes xor'ed into map-path keys
// (Perlin / generic gradients, OpenSimplex) carry the same bias (kMapLane).
//
// Unsigned form (TG_MAP_SIGNED=0): u = the top word, corner_height =
// (u + frac) * 2^-31 - 1; the -1 of every octave folds into one per-pixel
// offset (FbmArgs::hoff), so partial sums run near 2 sum(amp) and a
// low-amplitude window exceeds 1e-5 * A (round 1).
#if TG_MAP_HEIGHT_HI && TG_MAP_SIGNED
constexpr uint64_t kMapKeyBias = 0x8000000000000000ULL;
constexpr uint32_t kXsBias = 0x40000000u;  // (2^31 >> 1) carried by the xorshift
#else
constexpr uint64_t kMapKeyBias = 0;
constexpr uint32_t kXsBias = 0;
#endif
constexpr uint64_t kMapLane(uint64_t lane) { return lane ^ kMapKeyBias; }

#define TG_TOP_WORD(out, l, h)                                                         \
    asm("{\n\t.reg .b32 q;\n\tmul.hi.u32 q, %1, 0x1A85EC53;\n\t"                     \
        "mad.lo.u32 q, %2, 0x1A85EC53, q;\n\tmad.lo.u32 %0, %1, 0xC4CEB9FE, q;\n\t}"  \
        : "=r"(out)                                                                   \
        : "r"(l), "r"(h))

__device__ __forceinline__ uint32_t hash_top_word(uint64_t p) {
    uint32_t lo = static_cast<uint32_t>(p), hi = static_cast<uint32_t>(p >> 32);
    lo ^= (hi >> 1) ^ kXsBias;
    TG_MUL64(lo, hi, 0xED558CCD, 0xFF51AFD7);
    lo ^= (hi >> 1) ^ kXsBias;
    uint32_t t;
    TG_TOP_WORD(t, lo, hi);
    return t;
}

// N independent keys in lock step (N-way instruction-level parallelism).
template <int N>
__device__ __forceinline__ void hash_top_wordN(const uint64_t (&p)[N], uint32_t (&out)[N]) {
    uint32_t l[N], h[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
        l[i] = static_cast<uint32_t>(p[i]);
        h[i] = static_cast<uint32_t>(p[i] >> 32);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) l[i] ^= (h[i] >> 1) ^ kXsBias;
#pragma unroll
    for (int i = 0; i < N; ++i) TG_MUL64(l[i], h[i], 0xED558CCD, 0xFF51AFD7);
#pragma unroll
    for (int i = 0; i < N; ++i) l[i] ^= (h[i] >> 1) ^ kXsBias;
#pragma unroll
    for (int i = 0; i < N; ++i) TG_TOP_WORD(out[i], l[i], h[i]);
}

// Four independent keys in lock step (see height_scaled4).
__device__ __forceinline__ void hash_top_word4(uint64_t p0, uint64_t p1, uint64_t p2, uint64_t p3,
                                               uint32_t (&out)[4]) {
    const uint64_t p[4] = {p0, p1, p2, p3};
    hash_top_wordN<4>(p, out);
}

// The height representation of the map kernels: the corner height is
// map_height(p) * kMapScale - kMapOffsetUnits (the second term, unsigned form
// only, folded into FbmArgs::hoff = -sum(amp)).
//   TG_MAP_HEIGHT_HI=1 (default): one I2FP of the top word, |error| <= 2^-24,
//     10 instructions per key (signed: float(int32) * 2^-31).
//   TG_MAP_HEIGHT_HI=0: the exactly rounded height_scaled path, 14 per key.

#if TG_MAP_HEIGHT_HI
constexpr float kMapScale = 0x1p-31f;
#if TG_MAP_SIGNED
constexpr float kMapOffsetUnits = 0.0f;
__device__ __forceinline__ float top_word_height(uint32_t t) { return static_cast<float>(static_cast<int32_t>(t)); }
constexpr bool kMapOffset = false;
#else
constexpr float kMapOffsetUnits = 1.0f;
__device__ __forceinline__ float top_word_height(uint32_t t) { return static_cast<float>(t); }
constexpr bool kMapOffset = true;
#endif
__device__ __forceinline__ float map_height(uint64_t p) { return top_word_height(hash_top_word(p)); }
template <int N>
__device__ __forceinline__ void map_heightN(const uint64_t (&p)[N], float (&o)[N]) {
    uint32_t t[N];
    hash_top_wordN<N>(p, t);
#pragma unroll
    for (int i = 0; i < N; ++i) o[i] = top_word_height(t[i]);
}
__device__ __forceinline__ void map_height4(uint64_t p0, uint64_t p1, uint64_t p2, uint64_t p3, float (&o)[4]) {
    uint32_t t[4];
    hash_top_word4(p0, p1, p2, p3, t);
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = top_word_height(t[i]);
}
#else
constexpr float kMapScale = 0x1p-63f;
constexpr bool kMapOffset = false;
constexpr float kMapOffsetUnits = 0.0f;
__device__ __forceinline__ float map_height(uint64_t p) { return height_scaled(p); }
template <int N>
__device__ __forceinline__ void map_heightN(const uint64_t (&p)[N], float (&o)[N]) {
#pragma unroll
    for (int i = 0; i < N; ++i) o[i] = height_scaled(p[i]);
}
__device__ __forceinline__ void map_height4(uint64_t p0, uint64_t p1, uint64_t p2, uint64_t p3, float (&o)[4]) {
    height_scaled4(p0, p1, p2, p3, o);
}
#endif

// float(corner_height) with one round-to-nearest (lattice.hpp:56-64).
__device__ __forceinline__ float height_from_hash(uint64_t z) {
    const int64_t t = static_cast<int64_t>(z ^ 0x8000000000000000ULL) >> 11;
    return __ll2float_rn(t) * 0x1p-52f;
}

// to_unit(z) = (z >> 11) * 2^-53 as float from the top 32 bits (|error| <=
// 2^-25; used for angles and gradient magnitudes whose components are checked
// within tolerance, not bit-exact — cos/sin are libm-dependent).
__device__ __forceinline__ float unit_from_hash(uint64_t z) {
    return static_cast<float>(static_cast<uint32_t>(z >> 32)) * 0x1p-32f;
}

// (sin, cos)(2*pi*u) for u in [0, 1] turns with the hardware approximations
// on the centred angle 2*pi*(u - [u >= 1/2]) in [-pi, pi), where their
// absolute error is ~2^-21.4 (components checked within tolerance).
__device__ __forceinline__ void fast_sincos_turns(float u, float* s, float* c) {
    const float v = u >= 0.5f ? u - 1.0f : u;
    __sincosf(6.28318530717958647692f * v, s, c);
}

__device__ __forceinline__ float corner_height(uint64_t base, int64_t ix, int64_t iy) {
    return height_scaled(pack_xy(base, ix, iy)) * 0x1p-63f;
}

// corner_unit_gradient (lattice.hpp:80-83): angle = unit * 2*pi, so
// (cos, sin)(angle) = sincospi(2 * unit).
__device__ __forceinline__ void corner_unit_gradient(uint64_t base, int64_t ix, int64_t iy,
                                                     float* c, float* s) {
    const uint64_t z = mix64(pack_xy(base, ix, iy) ^ kAngleLane);
    fast_sincos_turns(unit_from_hash(z), s, c);
}

// corner_gradient (lattice.hpp:72-77): magnitude uniform in [0, w].
__device__ __forceinline__ void corner_gradient(uint64_t base, int64_t ix, int64_t iy, float w,
                                                float* gx, float* gy) {
    const uint64_t p = pack_xy(base, ix, iy);
    float c, s;
    fast_sincos_turns(unit_from_hash(mix64(p ^ kAngleLane)), &s, &c);
    const float m = unit_from_hash(mix64(p ^ kMagnitudeLane)) * w;
    *gx = m * c;
    *gy = m * s;
}

}  // namespace tg
