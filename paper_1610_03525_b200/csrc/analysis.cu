// analysis.cu — the fractal-analysis pass after generation.
//
//   upper median      analysis.hpp:244-250 (nth_element at n/2) -> 3-pass radix select
//   coastline_mask    analysis.hpp:213-240 -> warp-ballot bit mask (1 bit/pixel)
//   box_count         analysis.hpp:269-299 -> per-box OR over the bit mask, popcount
//   variogram         new (BASELINE.json config 5): fp64-accumulated block reduction
// All integer results (median element, mask bits, land/coast/box counts) are
// exact, so they equal the reference run on the same fp32 map.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/polyterrain_b200.h"
#include "devattr.h"
#include "select.h"

namespace tg {
int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
int check_device();

namespace {

__device__ __forceinline__ uint32_t fkey(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// ---- radix select -------------------------------------------------------------
struct SelectState {
    uint32_t prefix;  // selected high bits so far
    uint32_t mask;    // which bits of the key are fixed
    uint64_t k;       // rank still to find within the matching elements
};

constexpr int kBins = 2048;

constexpr int kHistBlocks = 148 * 4;  // 4 x 512 threads per SM

// Keys outside the current prefix take no part.  Plain shared atomics: the
// first digit (sign, exponent, 2 mantissa bits) spreads heights over a few
// dozen bins, so same-address replays within a warp stay cheap (a match.any
// merge measured 3x slower per element).
__device__ __forceinline__ void hist_add(unsigned int* sh, uint32_t key, uint32_t prefix, uint32_t mask,
                                         int shift, uint32_t dmask) {
    if ((key & mask) == prefix) atomicAdd(&sh[(key >> shift) & dmask], 1u);
}

// Shared-memory histogram flushed into the global one (non-zero bins only).
__device__ __forceinline__ void hist_flush(const unsigned int* sh, unsigned long long* hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < kBins; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], static_cast<unsigned long long>(sh[i]));
}

// Neighbouring heights share digits, so a warp's keys pile onto a few bins and
// plain shared atomics serialise on equal addresses.  Each thread merges its
// batch into runs of equal bins; the last run of every lane goes in as ONE
// atomic when the whole warp's last runs share a bin (the common case on a
// smooth map), else one atomic per lane.  All 32 lanes must call it.
template <int N>
__device__ __forceinline__ void hist_runs(unsigned int* sh, const uint32_t (&bin)[N], const bool (&ok)[N]) {
    uint32_t cur = 0xffffffffu, cnt = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) {  // branch-free bookkeeping; the flush is one predicated atomic
        const bool flush = ok[i] && bin[i] != cur && cnt != 0;
        if (flush) atomicAdd(&sh[cur], cnt);
        cnt = ok[i] ? (bin[i] == cur ? cnt + 1 : 1) : cnt;
        cur = ok[i] ? bin[i] : cur;
    }
    const uint32_t b0 = __shfl_sync(0xffffffffu, cur, 0);
    if (__all_sync(0xffffffffu, cnt == 0 || cur == b0)) {
        const uint32_t tot = __reduce_add_sync(0xffffffffu, cnt);
        if ((threadIdx.x & 31) == 0 && tot) atomicAdd(&sh[b0], tot);
    } else if (cnt) {
        atomicAdd(&sh[cur], cnt);
    }
}

__global__ void radix_hist(const float* __restrict__ x, uint64_t n, const SelectState* st,
                           int shift, int bits, unsigned long long* __restrict__ hist) {
    __shared__ unsigned int sh[kBins];
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint32_t prefix = st->prefix, mask = st->mask;
    const uint32_t dmask = (1u << bits) - 1u;
    const uint64_t n4 = (reinterpret_cast<uintptr_t>(x) & 15) == 0 ? n / 4 : 0;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    for (; i + stride < n4; i += 2 * stride) {  // two independent 16-byte loads in flight
        const float4 v = x4[i], u = x4[i + stride];
        hist_add(sh, fkey(v.x), prefix, mask, shift, dmask);
        hist_add(sh, fkey(v.y), prefix, mask, shift, dmask);
        hist_add(sh, fkey(v.z), prefix, mask, shift, dmask);
        hist_add(sh, fkey(v.w), prefix, mask, shift, dmask);
        hist_add(sh, fkey(u.x), prefix, mask, shift, dmask);
        hist_add(sh, fkey(u.y), prefix, mask, shift, dmask);
        hist_add(sh, fkey(u.z), prefix, mask, shift, dmask);
        hist_add(sh, fkey(u.w), prefix, mask, shift, dmask);
    }
    for (; i < n4; i += stride) {
        const float4 v = x4[i];
        hist_add(sh, fkey(v.x), prefix, mask, shift, dmask);
        hist_add(sh, fkey(v.y), prefix, mask, shift, dmask);
        hist_add(sh, fkey(v.z), prefix, mask, shift, dmask);
        hist_add(sh, fkey(v.w), prefix, mask, shift, dmask);
    }
    for (uint64_t i = n4 * 4 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
        hist_add(sh, fkey(x[i]), prefix, mask, shift, dmask);
    hist_flush(sh, hist);
}

// Strided-window form (row bands with halos): blocks stride over rows.
__global__ void radix_hist2d(const float* __restrict__ x, int64_t width, int64_t rows, int64_t ld,
                             const SelectState* st, int shift, int bits,
                             unsigned long long* __restrict__ hist) {
    __shared__ unsigned int sh[kBins];
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint32_t prefix = st->prefix, mask = st->mask;
    const uint32_t dmask = (1u << bits) - 1u;
    for (int64_t y = blockIdx.x; y < rows; y += gridDim.x)
        for (int64_t i = threadIdx.x; i < width; i += blockDim.x)
            hist_add(sh, fkey(x[y * ld + i]), prefix, mask, shift, dmask);
    hist_flush(sh, hist);
}

// ---- radix select with a sampled candidate window -----------------------------
// Three full histogram passes cost three reads of the map.  Instead the first
// pass also compacts every key whose first digit lies in a window of digits
// predicted from a strided sample (the sample's ranks rank_frac +- delta), and
// the second and third passes histogram only those keys when the selected
// first digit falls inside the window (otherwise they read the map again:
// the result is exact either way).  1 read + ~1 % writes instead of 3 reads.
__device__ __forceinline__ uint32_t d1(uint32_t key) { return key >> 21; }  // first digit (11 bits)

// Top-digit histogram of n_s samples, one at a hashed position in each stride
// of `step` linear positions (row-major, width w, pitch ld).
__global__ void sample_hist(const float* __restrict__ x, int64_t width, int64_t ld, uint64_t step, int n_s,
                            unsigned long long* __restrict__ hist) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n_s; j += gridDim.x * blockDim.x) {
        // j-th stride with a hashed offset inside it (a plain stride samples a
        // few columns only when it divides the width)
        const uint64_t p = j * step + (static_cast<uint32_t>(j) * 2654435761u) % step;
        const int64_t y = static_cast<int64_t>(p / width), c = static_cast<int64_t>(p - y * width);
        atomicAdd(&hist[d1(fkey(x[y * ld + c]))], 1ull);
    }
}

// Pass 1: first-digit histogram of every key; keys with d1 in [wlo, whi] are
// appended to this block's own segment of keys (seg entries; a warp-aggregated
// shared-memory counter; writes stop at seg, the count goes on) — one global
// store of the count per block, no global atomics on a shared counter.
__device__ __forceinline__ void keep_key(unsigned int* scnt, uint32_t key, uint32_t wlo, uint32_t whi,
                                         uint32_t* __restrict__ out, uint64_t seg, bool active) {
    const uint32_t d = d1(key);
    const bool in = active && d - wlo <= whi - wlo;
    const uint32_t b = __ballot_sync(0xffffffffu, in);
    if (b) {
        const int lane = threadIdx.x & 31;
        unsigned int base = 0;
        if (lane == __ffs(b) - 1) base = atomicAdd(scnt, static_cast<unsigned int>(__popc(b)));
        base = __shfl_sync(0xffffffffu, base, __ffs(b) - 1);
        const uint64_t at = base + __popc(b & ((1u << lane) - 1u));
        if (in && at < seg) out[at] = key;
    }
}

__global__ void __launch_bounds__(512) radix_hist_keep(const float* __restrict__ x, int64_t width, int64_t rows,
                                                       int64_t ld, bool vec, uint32_t wlo, uint32_t whi,
                                                       uint32_t* __restrict__ keys, uint64_t seg,
                                                       unsigned long long* __restrict__ bcnt,
                                                       unsigned long long* __restrict__ hist) {
    __shared__ unsigned int sh[kBins];
    __shared__ unsigned int scnt;
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) sh[i] = 0;
    if (threadIdx.x == 0) scnt = 0;
    __syncthreads();
    uint32_t* out = keys + blockIdx.x * seg;
    if (vec) {  // 16-byte loads (ld and width multiples of 4, aligned base)
        const int64_t w4 = width / 4, n4 = w4 * rows;
        const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
        // every lane of a warp iterates the same number of times (ballots need the whole warp)
        const int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + (threadIdx.x & ~31);
        constexpr int kV = 2;  // 16-byte loads in flight per thread
        const int lane = threadIdx.x & 31;
        for (int64_t ib = i0; ib < n4; ib += kV * stride) {
            uint32_t k[4 * kV];
            bool ok[4 * kV];
#pragma unroll
            for (int q = 0; q < kV; ++q) {
                const int64_t i = ib + q * stride + lane;
                const bool act = i < n4;
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (act) {
                    if (ld == width) {  // contiguous rows: linear index (no 64-bit division per load)
                        v = __ldg(reinterpret_cast<const float4*>(x) + i);
                    } else {
                        const int64_t y = i / w4, c = i - y * w4;
                        v = __ldg(reinterpret_cast<const float4*>(x + y * ld) + c);
                    }
                }
                k[4 * q] = fkey(v.x), k[4 * q + 1] = fkey(v.y), k[4 * q + 2] = fkey(v.z), k[4 * q + 3] = fkey(v.w);
#pragma unroll
                for (int e = 0; e < 4; ++e) ok[4 * q + e] = act;
            }
            int mine = 0;
#pragma unroll
            for (int e = 0; e < 4 * kV; ++e) {
                if (ok[e]) atomicAdd(&sh[d1(k[e])], 1u);
                mine += (ok[e] && d1(k[e]) - wlo <= whi - wlo) ? 1 : 0;
            }
            // one shared atomic per warp for its kept keys, lane offsets by a warp scan
            int incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const int tot = __shfl_sync(0xffffffffu, incl, 31);
            if (tot) {
                unsigned int base = 0;
                if (lane == 31) base = atomicAdd(&scnt, static_cast<unsigned int>(tot));
                base = __shfl_sync(0xffffffffu, base, 31);
                uint64_t at = base + static_cast<unsigned int>(incl - mine);
#pragma unroll
                for (int e = 0; e < 4 * kV; ++e)
                    if (ok[e] && d1(k[e]) - wlo <= whi - wlo) {
                        if (at < seg) out[at] = k[e];
                        ++at;
                    }
            }
        }
    } else {
        for (int64_t y = blockIdx.x; y < rows; y += gridDim.x)
            for (int64_t i0 = threadIdx.x & ~int64_t(31); i0 < width; i0 += blockDim.x) {
                const int64_t i = i0 + (threadIdx.x & 31);
                const bool act = i < width;
                const uint32_t k[1] = {act ? fkey(x[y * ld + i]) : 0u};
                const uint32_t b[1] = {d1(k[0])};
                const bool ok[1] = {act};
                hist_runs(sh, b, ok);
                keep_key(&scnt, k[0], wlo, whi, out, seg, act);
            }
    }
    hist_flush(sh, hist);
    if (threadIdx.x == 0) bcnt[blockIdx.x] = scnt;
}

// Contiguous form of radix_hist_keep (ld == width, 16-byte aligned, n % 4 ==
// 0): the radix_hist loop (two 16-byte loads in flight, no per-key range
// tests in full iterations) plus the candidate compaction.
template <bool kTail>
__device__ __forceinline__ void keep8(unsigned int* sh, unsigned int* scnt, const float4 v, const float4 u, bool a0,
                                      bool a1, uint32_t wlo, uint32_t whi, uint32_t* __restrict__ out, uint64_t seg) {
    const uint32_t k[8] = {fkey(v.x), fkey(v.y), fkey(v.z), fkey(v.w), fkey(u.x), fkey(u.y), fkey(u.z), fkey(u.w)};
    int mine = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const bool ok = !kTail || (e < 4 ? a0 : a1);
        if (ok) atomicAdd(&sh[d1(k[e])], 1u);
        mine += (ok && d1(k[e]) - wlo <= whi - wlo) ? 1 : 0;
    }
    if (__any_sync(0xffffffffu, mine != 0)) {  // rare: a warp with candidates
        const int lane = threadIdx.x & 31;
        int incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        unsigned int base = 0;
        if (lane == 31) base = atomicAdd(scnt, static_cast<unsigned int>(incl));
        base = __shfl_sync(0xffffffffu, base, 31);
        uint64_t at = base + static_cast<unsigned int>(incl - mine);
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if ((!kTail || (e < 4 ? a0 : a1)) && d1(k[e]) - wlo <= whi - wlo) {
                if (at < seg) out[at] = k[e];
                ++at;
            }
    }
}

__global__ void __launch_bounds__(512) radix_hist_keep_lin(const float4* __restrict__ x4, uint64_t n4, uint32_t wlo,
                                                           uint32_t whi, uint32_t* __restrict__ keys, uint64_t seg,
                                                           unsigned long long* __restrict__ bcnt,
                                                           unsigned long long* __restrict__ hist) {
    __shared__ unsigned int sh[kBins];
    __shared__ unsigned int scnt;
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) sh[i] = 0;
    if (threadIdx.x == 0) scnt = 0;
    __syncthreads();
    uint32_t* out = keys + blockIdx.x * seg;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t lane = threadIdx.x & 31;
    uint64_t ib = blockIdx.x * static_cast<uint64_t>(blockDim.x) + (threadIdx.x & ~31u);
    for (; ib + stride + 32 <= n4; ib += 2 * stride)  // whole warps, both loads in range
        keep8<false>(sh, &scnt, __ldg(x4 + ib + lane), __ldg(x4 + ib + stride + lane), true, true, wlo, whi, out, seg);
    for (; ib < n4; ib += 2 * stride) {  // warp-uniform tail
        const uint64_t i = ib + lane, j = i + stride;
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        keep8<true>(sh, &scnt, i < n4 ? __ldg(x4 + i) : z, j < n4 ? __ldg(x4 + j) : z, i < n4, j < n4, wlo, whi, out,
                    seg);
    }
    hist_flush(sh, hist);
    if (threadIdx.x == 0) bcnt[blockIdx.x] = scnt;
}

// Passes 2 and 3 over the kept keys (block b reads segment b).
__global__ void radix_hist_keys(const uint32_t* __restrict__ keys, uint64_t seg, const unsigned long long* bcnt,
                                uint32_t prefix, uint32_t mask, int shift, int bits,
                                unsigned long long* __restrict__ hist) {
    __shared__ unsigned int sh[kBins];
    for (int i = threadIdx.x; i < kBins; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint64_t n = bcnt[blockIdx.x];
    const uint32_t* in = keys + blockIdx.x * seg;
    const uint32_t dmask = (1u << bits) - 1u;
    for (uint64_t i0 = 0; i0 < n; i0 += 8 * blockDim.x) {  // 8 consecutive kept keys per thread
        const uint64_t i = i0 + 8 * threadIdx.x;
        uint32_t b[8];
        bool ok[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint32_t k = i + e < n ? in[i + e] : 0u;
            b[e] = (k >> shift) & dmask;
            ok[e] = i + e < n && (k & mask) == prefix;
        }
        hist_runs(sh, b, ok);
    }
    hist_flush(sh, hist);
}

// ---- coastline bit mask -------------------------------------------------------
// coast = land & !(all four neighbours land); neighbours outside the map
// count as land (the reference only tests in-bounds neighbours,
// analysis.hpp:228-229).  A warp owns a 1024-pixel column segment (lane i
// holds word w0 + i as a ballot of 32 land tests) and walks a strip of
// kCoastRows rows down the map carrying the land words of the row above and
// the current row, so every sample is read once (plus one halo row per strip)
// instead of three times.
// Band form: `rows` rows of width R (row pitch ld) starting at h; the rows
// just above/below exist (h - ld, h + rows*ld) when has_top / has_bot — halos
// regenerated by the caller for row-band shards.
constexpr int kCoastRows = 32;

// Land word of lane's w = w0 + lane in `row` (x >= R: not land), split into
// the 32 loads (issued one row ahead) and the 32 ballots.
__device__ __forceinline__ void land_load(const float* __restrict__ row, int64_t w0, int64_t R, int lane,
                                          float (&v)[32]) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const int64_t x = (w0 + i) * 32 + lane;
        v[i] = x < R ? __ldg(row + x) : -INFINITY;
    }
}
__device__ __forceinline__ uint32_t land_bits(const float (&v)[32], float sea, int lane) {
    uint32_t L = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const uint32_t b = __ballot_sync(0xffffffffu, v[i] >= sea);
        if (lane == i) L = b;
    }
    return L;
}

// The 32 loads of the next row are in flight while the current row's coast
// bits are formed (the latency of one row per warp was the bound: 80 %
// long-scoreboard stalls with the loads issued row by row).
#ifndef TG_COAST_MINB
#define TG_COAST_MINB 3
#endif
__global__ void __launch_bounds__(256, TG_COAST_MINB)
coast_bits_kernel(const float* __restrict__ h, int64_t R, int64_t rows, int64_t ld,
                                  int has_top, int has_bot, float sea, int srows,
                                  uint32_t* __restrict__ bits, uint8_t* __restrict__ mask8,
                                  unsigned long long* __restrict__ counts /* land, coast */) {
    const int64_t words = (R + 31) / 32;
    const int64_t segs = (words + 31) / 32;
    const int64_t strips = (rows + srows - 1) / srows;
    const int lane = threadIdx.x & 31;
    const int64_t warp_global = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    unsigned long long land = 0, coast = 0;
    float v[32];
    for (int64_t t = warp_global; t < strips * segs; t += nwarps) {
        const int64_t st = t / segs;
        const int64_t w0 = (t - st * segs) * 32;
        const int64_t y0 = st * srows, y1 = min(rows, y0 + srows);
        const int64_t w = w0 + lane;
        const int64_t valid = R - w * 32;  // bits beyond R count as land for the horizontal test
        const uint32_t beyond = valid >= 32 ? 0u : ~((1u << (valid > 0 ? valid : 0)) - 1u);
        uint32_t Lu = 0xffffffffu;
        if (y0 > 0 || has_top) {
            land_load(h + (y0 - 1) * ld, w0, R, lane, v);
            Lu = land_bits(v, sea, lane);
        }
        land_load(h + y0 * ld, w0, R, lane, v);
        uint32_t Lc = land_bits(v, sea, lane);
        const bool more0 = y0 + 1 < rows || has_bot;
        if (more0) land_load(h + (y0 + 1) * ld, w0, R, lane, v);
        for (int64_t y = y0; y < y1; ++y) {
            const float* row = h + y * ld;
            const bool more = y + 1 < rows || has_bot;
            const uint32_t Ld = more ? land_bits(v, sea, lane) : 0xffffffffu;
            if (y + 1 < y1 && (y + 2 < rows || has_bot)) land_load(row + 2 * ld, w0, R, lane, v);  // next row in flight
            // horizontal neighbours: bit b-1 / b+1 incl. the adjacent words' edge bits
            const uint32_t prev = __shfl_up_sync(0xffffffffu, Lc, 1);
            const uint32_t next = __shfl_down_sync(0xffffffffu, Lc, 1);
            if (w < words) {
                uint32_t prev_hi, next_lo;
                if (lane == 0)
                    prev_hi = w == 0 ? 1u : (row[w * 32 - 1] >= sea ? 1u : 0u);
                else
                    prev_hi = prev >> 31;
                if (lane == 31 || w + 1 >= words)
                    next_lo = (w + 1) * 32 >= R ? 1u : (row[(w + 1) * 32] >= sea ? 1u : 0u);
                else
                    next_lo = next & 1u;
                const uint32_t Lr = (Lc >> 1) | (next_lo << 31) | (beyond >> 1);  // land at x+1
                const uint32_t Ll = (Lc << 1) | prev_hi;                         // land at x-1
                const uint32_t coast_bits = Lc & ~(Ll & Lr & Lu & Ld);
                if (bits) bits[y * words + w] = coast_bits;
                land += __popc(Lc);
                coast += __popc(coast_bits);
                if (mask8) {
                    const int64_t nbit = valid >= 32 ? 32 : valid;
                    for (int b = 0; b < nbit; ++b) mask8[y * R + w * 32 + b] = (coast_bits >> b) & 1u;
                }
            }
            Lu = Lc;
            Lc = Ld;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        land += __shfl_xor_sync(0xffffffffu, land, o);
        coast += __shfl_xor_sync(0xffffffffu, coast, o);
    }
    if (lane == 0) {
        atomicAdd(&counts[0], land);
        atomicAdd(&counts[1], coast);
    }
}

__global__ void pack_mask_kernel(const uint8_t* __restrict__ m, int64_t R, uint32_t* __restrict__ bits,
                                 unsigned long long* __restrict__ counts) {
    const int64_t words = (R + 31) / 32;
    unsigned long long pix = 0;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < R * words;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t y = t / words, w = t - y * words;
        uint32_t v = 0;
        for (int b = 0; b < 32; ++b) {
            const int64_t x = w * 32 + b;
            if (x < R && m[y * R + x]) v |= 1u << b;
        }
        bits[t] = v;
        pix += __popc(v);
    }
    atomicAdd(&counts[1], pix);
}

__device__ __forceinline__ bool is_pow2_dev(int v) { return v > 0 && (v & (v - 1)) == 0; }

// Power-of-two box sides on the packed coast bits: eps <= 32 is one thread per
// (box row, 32-bit word) — OR of eps rows, then an OR-fold within each group
// of eps bits and a popcount of the group leaders; eps > 32 is one thread per
// box over eps rows x eps/32 words.  Bits past the row end are zero, so
// partial far-edge boxes count as in analysis.hpp:284.
__global__ void boxcount_pow2_kernel(const uint32_t* __restrict__ bits, int64_t R, int64_t rows,
                                     const int32_t* sizes, int n_sizes, unsigned long long* __restrict__ out) {
    const int s = blockIdx.y;
    if (s >= n_sizes) return;
    const int eps = sizes[s];
    if (!is_pow2_dev(eps) || eps <= 32) return;  // eps <= 32: boxcount_pow2_fused_kernel
    const int64_t words = (R + 31) / 32;
    const int64_t bpy = (rows + eps - 1) / eps;
    unsigned long long occ = 0;
    if (eps <= 32) {
        const uint32_t lead = eps == 32 ? 1u : eps == 16 ? 0x00010001u : eps == 8 ? 0x01010101u
                            : eps == 4 ? 0x11111111u : eps == 2 ? 0x55555555u : 0xFFFFFFFFu;
        for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < bpy * words;
             t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int64_t by = t / words, w = t - by * words;
            const int64_t y0 = by * eps, y1 = min(rows, y0 + eps);
            uint32_t m = 0;
            for (int64_t y = y0; y < y1; ++y) m |= __ldg(bits + y * words + w);
            for (int sh = 1; sh < eps; sh <<= 1) m |= m >> sh;
            occ += __popc(m & lead);
        }
    } else {
        const int64_t wpb = eps / 32;
        const int64_t bpx = (words + wpb - 1) / wpb;
        for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < bpy * bpx;
             t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int64_t by = t / bpx, bx = t - by * bpx;
            const int64_t y0 = by * eps, y1 = min(rows, y0 + eps);
            const int64_t wa = bx * wpb, wb = min(words, wa + wpb);
            uint32_t m = 0;
            for (int64_t y = y0; y < y1 && !m; ++y)
                for (int64_t w = wa; w < wb; ++w) m |= __ldg(bits + y * words + w);
            occ += m ? 1 : 0;
        }
    }
    for (int o = 16; o > 0; o >>= 1) occ += __shfl_xor_sync(0xffffffffu, occ, o);
    if ((threadIdx.x & 31) == 0 && occ) atomicAdd(&out[s], occ);
}

// All power-of-two sides 1..32 in one pass over the bits: a thread owns one
// word column of a 32-row block, ORs its rows pairwise up the levels
// (2, 4, 8, 16, 32 rows; the groups are anchored at multiples of eps since the
// block starts at a multiple of 32), folds each level's OR within the word by
// eps bits and counts the group leaders.  idx[j] = bit mask of the indices
// of the size 2^j in the caller's list (n_sizes <= 64).
struct Pow2Slots {
    unsigned long long idx[6];
};
__global__ void boxcount_pow2_fused_kernel(const uint32_t* __restrict__ bits, int64_t R, int64_t rows,
                                           const __grid_constant__ Pow2Slots ps, unsigned long long* __restrict__ out) {
    const int64_t words = (R + 31) / 32;
    const int64_t blocks_y = (rows + 31) / 32;
    unsigned long long occ[6] = {0, 0, 0, 0, 0, 0};
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < blocks_y * words;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t by = t / words, w = t - by * words;
        const int64_t y0 = by * 32;
        const int nr = static_cast<int>(rows - y0 < 32 ? rows - y0 : 32);
        uint32_t a[32];
#pragma unroll
        for (int r = 0; r < 32; ++r) a[r] = r < nr ? __ldg(bits + (y0 + r) * words + w) : 0u;
        constexpr uint32_t lead[6] = {0xFFFFFFFFu, 0x55555555u, 0x11111111u, 0x01010101u, 0x00010001u, 1u};
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            const int ng = 32 >> j;  // groups of 2^j rows in the block
#pragma unroll
            for (int g = 0; g < 32; ++g) {
                if (g < ng) {
                    uint32_t m = a[g];
#pragma unroll
                    for (int sh = 1; sh < (1 << j); sh <<= 1) m |= m >> sh;
                    occ[j] += __popc(m & lead[j]);
                }
            }
            if (j < 5) {
#pragma unroll
                for (int g = 0; g < 16; ++g)
                    if (g < (ng >> 1)) a[g] = a[2 * g] | a[2 * g + 1];
            }
        }
    }
#pragma unroll
    for (int j = 0; j < 6; ++j) {
        unsigned long long v = occ[j];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v)
            for (unsigned long long m = ps.idx[j]; m; m &= m - 1) atomicAdd(&out[__ffsll(m) - 1], v);
    }
}

// Occupied boxes of side eps (partial far-edge boxes count, analysis.hpp:284);
// any side that is not a power of two.
__global__ void boxcount_kernel(const uint32_t* __restrict__ bits, int64_t R, int64_t rows,
                                const int32_t* sizes, int n_sizes, unsigned long long* __restrict__ out) {
    const int s = blockIdx.y;
    if (s >= n_sizes || is_pow2_dev(sizes[s])) return;
    const int64_t eps = sizes[s];
    const int64_t words = (R + 31) / 32;
    const int64_t bpx = (R + eps - 1) / eps, bpy = (rows + eps - 1) / eps;
    unsigned long long occ = 0;
    for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < bpx * bpy;
         b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t by = b / bpx, bx = b - by * bpx;
        const int64_t x0 = bx * eps, x1 = min(R, x0 + eps);
        const int64_t y0 = by * eps, y1 = min(rows, y0 + eps);
        const int64_t wa = x0 >> 5, wb = (x1 - 1) >> 5;
        bool hit = false;
        for (int64_t y = y0; y < y1 && !hit; ++y) {
            const uint32_t* row = bits + y * words;
            for (int64_t w = wa; w <= wb; ++w) {
                uint32_t m = 0xffffffffu;
                if (w == wa) m &= 0xffffffffu << (x0 & 31);
                if (w == wb) {
                    const int hi = static_cast<int>((x1 - 1) & 31);
                    m &= hi == 31 ? 0xffffffffu : ((1u << (hi + 1)) - 1u);
                }
                if (row[w] & m) {
                    hit = true;
                    break;
                }
            }
        }
        occ += hit ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) occ += __shfl_xor_sync(0xffffffffu, occ, o);
    if ((threadIdx.x & 31) == 0 && occ) atomicAdd(&out[s], occ);
}

// ---- variogram ----------------------------------------------------------------
constexpr int kMaxLags = 32;
constexpr int kFusedLags = 16;  // lags per pass (accumulators in registers)

struct LagSet {
    int n;
    int hmax;           // largest real lag of the set
    int h[kFusedLags];  // padded with 0 (the sample itself, d = 0) on both axes
};

#ifndef TG_VG_SEGC
#define TG_VG_SEGC 8192
#endif
constexpr int kSegC = TG_VG_SEGC;  // columns per x work item
constexpr int kApron = 4096;   // x-lag partners beyond the segment kept in smem
constexpr int kVgThreads = 256;
constexpr int kYC = 4 * kVgThreads;  // columns per y column strip (4 per thread)

// x-axis pairs of up to 16 lags in ONE pass over the map.  A work item is
// (row y, column segment [x0, x0 + C)); the segment plus an apron of up to
// 4096 columns is widened to fp64 once into shared memory, so every x-lag
// pair is two shared loads + DADD + DFMA with no conversion.  The difference
// of two fp32 values is exact in fp64; sums are fp64.  Pairs whose first
// point lies in rows [0, P) of a W x H window (P = H for a whole map; P < H
// when the rows below a band were regenerated as lookahead).  sums[2*l].
// An item whose every pair lies inside the row (all but the last segment of
// a row) runs without per-pair bounds checks.
// kLongX: some lag exceeds the apron (its partners are read from global memory).
#ifndef TG_VGX_MIN_BLOCKS
#define TG_VGX_MIN_BLOCKS 2
#endif
#ifndef TG_VGX_GRID
#define TG_VGX_GRID 2  // x CTAs per SM
#endif
#ifndef TG_VGY_GRID
#define TG_VGY_GRID 3  // y CTAs per SM
#endif
#ifndef TG_VG_CONCURRENT
#define TG_VG_CONCURRENT 0
#endif
template <int NL, bool kLongX>
__global__ void __launch_bounds__(kVgThreads, TG_VGX_MIN_BLOCKS)
variogram_x_kernel(const float* __restrict__ z, int64_t W, int64_t ld, int64_t P,
                   const __grid_constant__ LagSet L, int64_t nseg, int seg_cap, double* __restrict__ sums) {
    extern __shared__ double seg[];
    double ax[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) ax[l] = 0.0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t items = P * nseg;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        const int64_t y = it / nseg;
        const int64_t x0 = (it - y * nseg) * kSegC;
        const int wl = static_cast<int>(W - x0 < (int64_t(1) << 30) ? W - x0 : (int64_t(1) << 30));  // columns from x0
        const int cw = wl < kSegC ? wl : kSegC;
        const int sw = wl < seg_cap ? wl : seg_cap;  // segment + apron
        const float* row = z + y * ld + x0;
        __syncthreads();  // previous item's readers are done with seg
        for (int i = threadIdx.x; i < sw; i += kVgThreads) seg[i] = static_cast<double>(__ldg(row + i));
        __syncthreads();
        if (!kLongX && cw + L.hmax <= wl) {
            // interior item: every partner x + h < cw + hmax <= min(wl, seg_cap)
            for (int x = threadIdx.x; x < cw; x += kVgThreads) {
                const double v = seg[x];
#pragma unroll
                for (int l = 0; l < NL; ++l) {
                    const double d = seg[x + L.h[l]] - v;
                    ax[l] = fma(d, d, ax[l]);
                }
            }
        } else {
            for (int x = threadIdx.x; x < cw; x += kVgThreads) {
                const double v = seg[x];
#pragma unroll
                for (int l = 0; l < NL; ++l) {
                    const int h = L.h[l];
                    if (x + h < wl) {
                        // without kLongX every h <= kApron, so x + h < sw: in smem
                        const double p =
                            (kLongX && x + h >= sw) ? static_cast<double>(__ldg(row + x + h)) : seg[x + h];
                        const double d = p - v;
                        ax[l] = fma(d, d, ax[l]);
                    }
                }
            }
        }
    }
    __syncthreads();
    double* part = seg;  // [8 warps][16]
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        double a = ax[l];
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) part[warp * kFusedLags + l] = a;
    }
    __syncthreads();
    if (threadIdx.x < L.n) {
        double t = 0.0;
        for (int w = 0; w < kVgThreads / 32; ++w) t += part[w * kFusedLags + threadIdx.x];
        atomicAdd(&sums[2 * threadIdx.x], t);
    }
}

// y-axis pairs of up to 16 lags.  A work item is (column strip of 1024) x
// (kYRows rows); the CTA walks its strip down the rows, each thread 4
// consecutive columns as one 16-byte load per row, so the partner rows of the
// short lags are still in L1 from the previous rows, and items are handed out
// grid-stride (one index division per item, no wave tail at any map shape).
// The partner rows y + h of all lags are loaded back to back (64-bit row
// offsets, any ld); a lag without a partner row reads its own row (d = 0,
// adds nothing).  sums[2*l + 1].
#ifndef TG_VGY_MIN_BLOCKS
#define TG_VGY_MIN_BLOCKS 3
#endif
#ifndef TG_VGY_NEAR
#define TG_VGY_NEAR (1 << 30)
#endif
constexpr int kNearRows = TG_VGY_NEAR;
#ifndef TG_VGY_ROWS
#define TG_VGY_ROWS 32
#endif
constexpr int kYRows = TG_VGY_ROWS;  // rows per y work item (one column strip)
template <int NL, bool kFull>
__device__ __forceinline__ void variogram_y_rows(const float* __restrict__ row, int64_t y, int64_t y1, int64_t H,
                                                 int64_t ld, int nv, const LagSet& L, double (&ay)[NL]) {
    // Partner rows of lags beyond kNearRows bypass L1 (L1::no_allocate) so the
    // near rows stay resident there until the walk reaches them.
    auto load_far = [&](const float* q, float (&o)[4]) {
        if (kFull) {
            asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3])
                         : "l"(q));
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) o[k] = k < nv ? __ldg(q + k) : 0.f;
        }
    };
    auto load = [&](const float* q, float (&o)[4]) {
        if (kFull) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(q));
            o[0] = t.x;
            o[1] = t.y;
            o[2] = t.z;
            o[3] = t.w;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) o[k] = k < nv ? __ldg(q + k) : 0.f;
        }
    };
    for (; y < y1; ++y, row += ld) {
        float a[4];
        load(row, a);
        double v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = static_cast<double>(a[k]);
#pragma unroll
        for (int g = 0; g < NL; g += 4) {  // up to 4 partner rows in flight per group
            constexpr int kG = 4;
            float b[kG][4];
#pragma unroll
            for (int l = 0; l < kG; ++l) {
                if (g + l < NL) {
                    const int64_t h = L.h[g + l];
                    const float* q = y + h < H ? row + h * ld : row;
                    if (h > kNearRows)
                        load_far(q, b[l]);
                    else
                        load(q, b[l]);
                }
            }
#pragma unroll
            for (int l = 0; l < kG; ++l) {
                if (g + l < NL) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const double d = static_cast<double>(b[l][k]) - v[k];
                        ay[g + l] = fma(d, d, ay[g + l]);
                    }
                }
            }
        }
    }
}

template <int NL, bool kVec>
__global__ void __launch_bounds__(kVgThreads, TG_VGY_MIN_BLOCKS)
variogram_y_kernel(const float* __restrict__ z, int64_t W, int64_t H, int64_t ld, int64_t P,
                   const __grid_constant__ LagSet L, double* __restrict__ sums) {
    double ay[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) ay[l] = 0.0;
    const int64_t nchunk = (W + kYC - 1) / kYC;
    const int64_t nrb = (P + kYRows - 1) / kYRows;
    for (int64_t it = blockIdx.x; it < nchunk * nrb; it += gridDim.x) {
        const int64_t rb = it / nchunk;
        const int64_t y0 = rb * kYRows;
        const int64_t y1 = y0 + kYRows < P ? y0 + kYRows : P;
        const int64_t x = (it - rb * nchunk) * kYC + 4 * threadIdx.x;
        if (x >= W) continue;
        const int nv = W - x < 4 ? static_cast<int>(W - x) : 4;
        const float* row = z + y0 * ld + x;
        if (kVec && nv == 4)
            variogram_y_rows<NL, true>(row, y0, y1, H, ld, nv, L, ay);
        else
            variogram_y_rows<NL, false>(row, y0, y1, H, ld, nv, L, ay);
    }
    __shared__ double part[kVgThreads / 32][kFusedLags];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        double a = ay[l];
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        if (lane == 0) part[warp][l] = a;
    }
    __syncthreads();
    if (threadIdx.x < L.n) {
        double t = 0.0;
        for (int w = 0; w < kVgThreads / 32; ++w) t += part[w][threadIdx.x];
        atomicAdd(&sums[2 * threadIdx.x + 1], t);
    }
}

}  // namespace
int vg_ring_enqueue(const float* z, int64_t W, int64_t H, int64_t ld, int64_t P, const int32_t* lags, int n_lags,
                    double* sums, int sm, cudaStream_t s, cudaStream_t sy);
namespace {

struct Scratch {
    void* p = nullptr;
    cudaStream_t s;
    explicit Scratch(cudaStream_t st) : s(st) {}
    cudaError_t alloc(size_t n) { return cudaMallocAsync(&p, n, s); }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
};

}  // namespace

// One pass of the (possibly distributed) upper-median radix select over a
// window (width x rows, pitch ld): the digit histogram (shift, bits) of the
// keys matching prefix/mask, to the host.  With a cache, the first pass
// (mask == 0) also keeps a candidate window of keys (see radix_hist_keep) and
// later passes read only those when the chosen first digit lies inside it.
int select_hist(const float* map, int64_t width, int64_t rows, int64_t ld, uint32_t prefix, uint32_t mask, int shift,
                int bits, uint64_t* out_hist, SelectCache* cache, cudaStream_t s) {
    const uint64_t n = static_cast<uint64_t>(width) * static_cast<uint64_t>(rows);
    const size_t hb = kBins * sizeof(unsigned long long);
    if (cache && cache->dev_hist == nullptr) {
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&cache->dev_hist), hb + 64, s);
        if (e != cudaSuccess) return set_cuda_error(e, "select alloc");
    }
    Scratch scr(s);
    unsigned long long* hist = nullptr;
    unsigned long long* cnt = nullptr;
    if (cache) {
        hist = cache->dev_hist;
        cnt = hist + kBins;
    } else {
        cudaError_t e = scr.alloc(hb + 64);
        if (e != cudaSuccess) return set_cuda_error(e, "select alloc");
        hist = static_cast<unsigned long long*>(scr.p);
        cnt = hist + kBins;
    }
    cudaError_t e = cudaMemsetAsync(hist, 0, hb + 8, s);
    const bool vec = (ld & 3) == 0 && (width & 3) == 0 && (reinterpret_cast<uintptr_t>(map) & 15) == 0;
    const int hblocks = static_cast<int>(std::min<int64_t>(std::max<int64_t>(rows, 1), kHistBlocks));
    if (cache && mask == 0 && shift == 21 && bits == 11 && n >= (uint64_t(1) << 22)) {
        // window of first digits from a strided sample of 2^18 keys
        constexpr int kS = 1 << 18;
        std::vector<unsigned long long> sh(kBins);
        if (e == cudaSuccess) sample_hist<<<128, 512, 0, s>>>(map, width, ld, n / kS, kS, hist);
        if (e == cudaSuccess) e = cudaMemcpyAsync(sh.data(), hist, hb, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return set_cuda_error(e, "select sample");
        const double lo = (cache->rank_frac - cache->delta) * kS, hi = (cache->rank_frac + cache->delta) * kS;
        uint64_t c = 0;
        int wlo = -1, whi = -1;
        for (int d = 0; d < kBins; ++d) {
            const uint64_t c1 = c + sh[d];
            if (wlo < 0 && static_cast<double>(c1) > lo) wlo = d;
            if (whi < 0 && static_cast<double>(c1) > hi) whi = d;
            c = c1;
        }
        if (wlo < 0) wlo = kBins - 1;
        if (whi < 0) whi = kBins - 1;
        uint64_t in = 0;
        for (int d = wlo; d <= whi; ++d) in += sh[d];
        // twice the expected window count (blocks see near-equal shares of it)
        const uint64_t cap = static_cast<uint64_t>(2.0 * static_cast<double>(in + 64) / kS * static_cast<double>(n)) +
                             (uint64_t(1) << 20);
        cache->valid = false;
        if (static_cast<double>(in) / kS <= 0.3) {
            if (cache->cap < cap) {
                if (cache->keys) cudaFreeAsync(cache->keys, s);
                cache->keys = nullptr;
                cache->cap = 0;
                e = cudaMallocAsync(reinterpret_cast<void**>(&cache->keys), cap * sizeof(uint32_t), s);
                if (e != cudaSuccess) return set_cuda_error(e, "select keys alloc");
                cache->cap = cap;
            }
            cache->wlo = static_cast<uint32_t>(wlo);
            cache->whi = static_cast<uint32_t>(whi);
            if (!cache->bcnt) {
                e = cudaMallocAsync(reinterpret_cast<void**>(&cache->bcnt), kHistBlocks * sizeof(unsigned long long), s);
                if (e != cudaSuccess) return set_cuda_error(e, "select counts alloc");
            }
            const uint64_t seg = cache->cap / kHistBlocks;
            e = cudaMemsetAsync(hist, 0, hb + 8, s);
            if (e == cudaSuccess) {
                if (vec && ld == width)
                    radix_hist_keep_lin<<<kHistBlocks, 512, 0, s>>>(reinterpret_cast<const float4*>(map), n / 4,
                                                                    cache->wlo, cache->whi, cache->keys, seg,
                                                                    cache->bcnt, hist);
                else
                    radix_hist_keep<<<kHistBlocks, 512, 0, s>>>(map, width, rows, ld, vec, cache->wlo, cache->whi,
                                                               cache->keys, seg, cache->bcnt, hist);
            }
            std::vector<unsigned long long> got(kHistBlocks);
            if (e == cudaSuccess) e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaMemcpyAsync(out_hist, hist, hb, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(got.data(), cache->bcnt, kHistBlocks * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) return set_cuda_error(e, "select pass 1");
            cache->valid = true;
            for (auto g : got) cache->valid = cache->valid && g <= seg;
            return TG_OK;
        }
    }
    const bool from_keys = cache && cache->valid && (mask & 0xffe00000u) == 0xffe00000u &&
                           (prefix >> 21) - cache->wlo <= cache->whi - cache->wlo;
    if (e == cudaSuccess) {
        SelectState init{prefix, mask, 0};
        SelectState* st = reinterpret_cast<SelectState*>(cnt + 1);  // 64 spare bytes after the histogram
        e = cudaMemcpyAsync(st, &init, sizeof(init), cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) {
            if (from_keys)
                radix_hist_keys<<<kHistBlocks, 512, 0, s>>>(cache->keys, cache->cap / kHistBlocks, cache->bcnt, prefix,
                                                            mask, shift, bits, hist);
            else if (ld == width)
                radix_hist<<<kHistBlocks, 512, 0, s>>>(map, n, st, shift, bits, hist);
            else
                radix_hist2d<<<hblocks, 512, 0, s>>>(map, width, rows, ld, st, shift, bits, hist);
            e = cudaGetLastError();
        }
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_hist, hist, (size_t{1} << bits) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_cuda_error(e, "select histogram");
    return TG_OK;
}

void select_cache_free(SelectCache* c, cudaStream_t s) {
    if (c->keys) cudaFreeAsync(c->keys, s);
    if (c->bcnt) cudaFreeAsync(c->bcnt, s);
    if (c->dev_hist) cudaFreeAsync(c->dev_hist, s);
    *c = SelectCache{};
}

}  // namespace tg

using namespace tg;

extern "C" {

int tg_median_f32(const float* dev_map, uint64_t n, float* out_median, void* stream) {
    if (!dev_map || !out_median || n == 0)
        return set_error(TG_EVALIDATION, "coastline_mask: empty heightmap");
    if (int st = check_device()) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // the map as rows of up to 2^20 keys (any n), ragged tail as its own window
    const int64_t W = n >= (uint64_t(1) << 20) ? (int64_t(1) << 20) : static_cast<int64_t>(n);
    const int64_t rows = static_cast<int64_t>(n / W), tail = static_cast<int64_t>(n - uint64_t(rows) * W);
    SelectCache cache;
    uint32_t prefix = 0, mask = 0;
    uint64_t k = n / 2;  // analysis.hpp:247 (upper median)
    const int digits[3][2] = {{21, 11}, {10, 11}, {0, 10}};
    std::vector<uint64_t> h(kBins), ht(kBins);
    int st = TG_OK;
    for (const auto& dg : digits) {
        const int shift = dg[0], bits = dg[1];
        st = select_hist(dev_map, W, rows, W, prefix, mask, shift, bits, h.data(), &cache, s);
        if (st == TG_OK && tail)
            st = select_hist(dev_map + uint64_t(rows) * W, tail, 1, tail, prefix, mask, shift, bits, ht.data(), nullptr,
                             s);
        if (st != TG_OK) break;
        uint64_t c = 0;
        int d = 0;
        for (; d < (1 << bits); ++d) {
            const uint64_t hd = h[d] + (tail ? ht[d] : 0);
            if (c + hd > k) break;
            c += hd;
        }
        if (d == (1 << bits)) {
            st = set_error(TG_ENUMERICAL, "median: select out of range");
            break;
        }
        k -= c;
        prefix |= static_cast<uint32_t>(d) << shift;
        mask |= ((1u << bits) - 1u) << shift;
    }
    select_cache_free(&cache, s);
    if (st != TG_OK) return st;
    const uint32_t b = (prefix & 0x80000000u) ? (prefix & 0x7fffffffu) : ~prefix;
    std::memcpy(out_median, &b, 4);
    return TG_OK;
}

static int coast_common(const float* dev_map, int64_t R, int64_t rows, int64_t ld, int has_top, int has_bot,
                        double sea, uint32_t* bits, uint8_t* mask8, unsigned long long* counts, cudaStream_t s) {
    const int64_t segs = ((R + 31) / 32 + 31) / 32;
    // strips of up to kCoastRows rows, shorter when the map offers fewer
    // than ~4 warps of work per SMSP
    const int srows = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kCoastRows, rows * segs / (148 * 16))));
    const int64_t warps = ((rows + srows - 1) / srows) * segs;
    const int64_t blocks = std::min<int64_t>((warps * 32 + 255) / 256, 148 * 16);
    // land test h >= sea with the fp32 map widened exactly: for a double sea
    // level, h >= sea  <=>  h >= the smallest float >= sea.
    float seaf = static_cast<float>(sea);
    if (static_cast<double>(seaf) < sea) seaf = nextafterf(seaf, INFINITY);
    coast_bits_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(dev_map, R, rows, ld, has_top, has_bot, seaf,
                                                                     srows, bits, mask8, counts);
    return cudaGetLastError() == cudaSuccess ? TG_OK : set_error(TG_EDEVICE, "coastline kernel launch");
}

static int check_sizes(int64_t R, const int32_t* sizes, int32_t n) {
    if (n < 3 || n > 64) return set_error(TG_EVALIDATION, "box_count: need at least 3 box sizes to fit");
    for (int i = 0; i < n; ++i) {  // analysis.hpp:272-278
        if (sizes[i] < 1 || sizes[i] > R)
            return set_error(TG_EVALIDATION, "box_count: box sizes must lie in [1, resolution]");
        if (i > 0 && sizes[i] <= sizes[i - 1])
            return set_error(TG_EVALIDATION, "box_count: box sizes must be strictly increasing");
    }
    return TG_OK;
}

static int boxcount_from_bits(const uint32_t* bits, int64_t R, int64_t rows, const int32_t* sizes, int32_t n,
                              unsigned long long* dcounts, int32_t* dsizes, cudaStream_t s) {
    cudaError_t e = cudaMemcpyAsync(dsizes, sizes, n * sizeof(int32_t), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return set_cuda_error(e, "boxcount sizes");
    dim3 grid(148 * 4, static_cast<unsigned>(n));
    bool any_other = false;
    for (int i = 0; i < n; ++i) any_other = any_other || (sizes[i] & (sizes[i] - 1)) != 0;
    Pow2Slots ps = {};
    bool big = false;
    for (int i = 0; i < n; ++i) {
        const int v = sizes[i];
        if (v > 0 && (v & (v - 1)) == 0 && v <= 32)
            ps.idx[__builtin_ctz(static_cast<unsigned>(v))] |= 1ull << i;
        else if (v > 32 && (v & (v - 1)) == 0)
            big = true;
    }
    boxcount_pow2_fused_kernel<<<148 * 4, 256, 0, s>>>(bits, R, rows, ps, dcounts);
    if (big) boxcount_pow2_kernel<<<grid, 256, 0, s>>>(bits, R, rows, dsizes, n, dcounts);
    if (any_other) boxcount_kernel<<<grid, 256, 0, s>>>(bits, R, rows, dsizes, n, dcounts);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "boxcount launch");
    return TG_OK;
}

int tg_coastline_mask(const float* dev_map, int64_t resolution, double sea_level, uint8_t* dev_mask,
                      int64_t* out_land_count, void* stream) {
    if (resolution < 2) return set_error(TG_EVALIDATION, "coastline_mask: resolution must be at least 2");
    if (!dev_map || !dev_mask) return set_error(TG_EVALIDATION, "coastline_mask: null pointer");
    if (int st = check_device()) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Scratch scr(s);
    cudaError_t e = scr.alloc(2 * sizeof(unsigned long long));
    if (e != cudaSuccess) return set_cuda_error(e, "coastline alloc");
    auto* counts = static_cast<unsigned long long*>(scr.p);
    e = cudaMemsetAsync(counts, 0, 2 * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return set_cuda_error(e, "coastline memset");
    if (int st = coast_common(dev_map, resolution, resolution, resolution, 0, 0, sea_level, nullptr, dev_mask,
                              counts, s))
        return st;
    unsigned long long h[2];
    e = cudaMemcpyAsync(h, counts, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_cuda_error(e, "coastline");
    if (out_land_count) *out_land_count = static_cast<int64_t>(h[0]);
    const unsigned long long total = static_cast<unsigned long long>(resolution) * resolution;
    if (h[0] == 0 || h[0] == total)  // analysis.hpp:237-238
        return set_error(TG_EVALIDATION, "coastline_mask: map is entirely land or entirely water");
    return TG_OK;
}

int tg_coastline_boxcount_band(const float* dev_rows, int64_t width, int64_t rows, int64_t ld, int32_t has_top,
                               int32_t has_bottom, double sea_level, const int32_t* sizes, int32_t n_sizes,
                               int64_t* out_counts, int64_t* out_coast_pixels, int64_t* out_land_count,
                               void* stream) {
    if (width < 2 || rows < 1 || ld < width) return set_error(TG_EVALIDATION, "coastline_mask: bad window");
    if (!dev_rows || !sizes || !out_counts) return set_error(TG_EVALIDATION, "coastline_boxcount: null pointer");
    if (int st = check_sizes(width, sizes, n_sizes)) return st;
    if (int st = check_device()) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t words = (width + 31) / 32;
    const size_t bits_bytes = static_cast<size_t>(rows * words) * 4;
    Scratch scr(s);
    const size_t hdr = 2 * 8 + 64 * 8 + 64 * 4;
    cudaError_t e = scr.alloc(hdr + bits_bytes);
    if (e != cudaSuccess) return set_cuda_error(e, "coastline_boxcount alloc");
    auto* counts = static_cast<unsigned long long*>(scr.p);
    auto* bcounts = counts + 2;
    auto* dsizes = reinterpret_cast<int32_t*>(bcounts + 64);
    auto* bits = reinterpret_cast<uint32_t*>(static_cast<char*>(scr.p) + hdr);
    e = cudaMemsetAsync(scr.p, 0, 2 * 8 + 64 * 8, s);
    if (e != cudaSuccess) return set_cuda_error(e, "coastline_boxcount memset");
    if (int st = coast_common(dev_rows, width, rows, ld, has_top, has_bottom, sea_level, bits, nullptr, counts, s))
        return st;
    if (int st = boxcount_from_bits(bits, width, rows, sizes, n_sizes, bcounts, dsizes, s)) return st;
    unsigned long long h[2 + 64];
    e = cudaMemcpyAsync(h, counts, (2 + n_sizes) * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_cuda_error(e, "coastline_boxcount");
    if (out_land_count) *out_land_count = static_cast<int64_t>(h[0]);
    if (out_coast_pixels) *out_coast_pixels = static_cast<int64_t>(h[1]);
    for (int i = 0; i < n_sizes; ++i) out_counts[i] = static_cast<int64_t>(h[2 + i]);
    return TG_OK;
}

int tg_coastline_boxcount(const float* dev_map, int64_t resolution, double sea_level, const int32_t* sizes,
                          int32_t n_sizes, int64_t* out_counts, int64_t* out_coast_pixels,
                          int64_t* out_land_count, void* stream) {
    if (resolution < 2) return set_error(TG_EVALIDATION, "coastline_mask: resolution must be at least 2");
    int64_t coast = 0, land = 0;
    if (int st = tg_coastline_boxcount_band(dev_map, resolution, resolution, resolution, 0, 0, sea_level, sizes,
                                            n_sizes, out_counts, &coast, &land, stream))
        return st;
    if (out_land_count) *out_land_count = land;
    if (out_coast_pixels) *out_coast_pixels = coast;
    const int64_t total = resolution * resolution;
    if (land == 0 || land == total)
        return set_error(TG_EVALIDATION, "coastline_mask: map is entirely land or entirely water");
    if (coast == 0) return set_error(TG_EVALIDATION, "box_count: empty coastline mask");
    return TG_OK;
}

int tg_boxcount_mask(const uint8_t* dev_mask, int64_t resolution, const int32_t* sizes, int32_t n_sizes,
                     int64_t* out_counts, void* stream) {
    if (resolution < 2) return set_error(TG_EVALIDATION, "box_count: invalid mask resolution");
    if (!dev_mask || !sizes || !out_counts) return set_error(TG_EVALIDATION, "box_count: null pointer");
    if (int st = check_sizes(resolution, sizes, n_sizes)) return st;
    if (int st = check_device()) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t words = (resolution + 31) / 32;
    const size_t bits_bytes = static_cast<size_t>(resolution * words) * 4;
    Scratch scr(s);
    const size_t hdr = 2 * 8 + 64 * 8 + 64 * 4;
    cudaError_t e = scr.alloc(hdr + bits_bytes);
    if (e != cudaSuccess) return set_cuda_error(e, "box_count alloc");
    auto* counts = static_cast<unsigned long long*>(scr.p);
    auto* bcounts = counts + 2;
    auto* dsizes = reinterpret_cast<int32_t*>(bcounts + 64);
    auto* bits = reinterpret_cast<uint32_t*>(static_cast<char*>(scr.p) + hdr);
    e = cudaMemsetAsync(scr.p, 0, 2 * 8 + 64 * 8, s);
    if (e != cudaSuccess) return set_cuda_error(e, "box_count memset");
    pack_mask_kernel<<<148 * 8, 256, 0, s>>>(dev_mask, resolution, bits, counts);
    if (int st = boxcount_from_bits(bits, resolution, resolution, sizes, n_sizes, bcounts, dsizes, s)) return st;
    unsigned long long h[2 + 64];
    e = cudaMemcpyAsync(h, counts, (2 + n_sizes) * 8, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_cuda_error(e, "box_count");
    for (int i = 0; i < n_sizes; ++i) out_counts[i] = static_cast<int64_t>(h[2 + i]);
    if (h[1] == 0) return set_error(TG_EVALIDATION, "box_count: empty coastline mask");
    return TG_OK;
}

int tg_variogram_band_f32(const float* dev_map, int64_t width, int64_t height, int64_t ld, int64_t pair_rows,
                          const int32_t* lags, int32_t n_lags, double* out_sum_sq, int64_t* out_pairs,
                          void* stream) {
    if (!dev_map || !lags || !out_sum_sq || !out_pairs) return set_error(TG_EVALIDATION, "variogram: null pointer");
    if (width < 1 || height < 1 || ld < width || pair_rows < 0 || pair_rows > height)
        return set_error(TG_EVALIDATION, "variogram: bad window");
    if (n_lags < 1 || n_lags > kMaxLags) return set_error(TG_EVALIDATION, "variogram: 1..32 lags");
    for (int i = 0; i < n_lags; ++i)
        if (lags[i] < 1) return set_error(TG_EVALIDATION, "variogram: lags must be >= 1");
    if (int st = check_device()) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Scratch scr(s);
    cudaError_t e = scr.alloc(2 * kMaxLags * sizeof(double));
    if (e != cudaSuccess) return set_cuda_error(e, "variogram alloc");
    auto* sums = static_cast<double*>(scr.p);
    e = cudaMemsetAsync(sums, 0, 2 * kMaxLags * sizeof(double), s);
    if (e != cudaSuccess) return set_cuda_error(e, "variogram setup");
    int sm = 148;
    {
        int dev = 0;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, dev);
    }
    const int64_t nseg = (width + kSegC - 1) / kSegC;
    const int seg_cap = static_cast<int>(std::min<int64_t>(width, kSegC + kApron));
    const size_t smem = std::max<size_t>(static_cast<size_t>(seg_cap), kFusedLags * (kVgThreads / 32)) * sizeof(double);
    using KX = void (*)(const float*, int64_t, int64_t, int64_t, LagSet, int64_t, int, double*);
    using KY = void (*)(const float*, int64_t, int64_t, int64_t, int64_t, LagSet, double*);
#define TG_VG_NL(K, B) K<2, B>, K<4, B>, K<6, B>, K<8, B>, K<10, B>, K<12, B>, K<14, B>, K<16, B>
    static const KX xt[2][8] = {{TG_VG_NL(variogram_x_kernel, false)}, {TG_VG_NL(variogram_x_kernel, true)}};
    static const KY yt[2][8] = {{TG_VG_NL(variogram_y_kernel, false)}, {TG_VG_NL(variogram_y_kernel, true)}};
#undef TG_VG_NL
    static PerDeviceOnce attr_set;  // >48 KiB dynamic smem opt-in, per device
    e = attr_set.run([&] {
        const int mx = static_cast<int>((kSegC + kApron) * sizeof(double));
        cudaError_t r = cudaSuccess;
        for (auto& row : xt)
            for (auto f : row)
                if (r == cudaSuccess) r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
        return r;
    });
    if (e != cudaSuccess) return set_cuda_error(e, "variogram smem opt-in");
    const int64_t xblocks =
        std::max<int64_t>(1, std::min<int64_t>(pair_rows * nseg, TG_VGX_GRID * static_cast<int64_t>(sm)));
    const int64_t nchunk = (width + kYC - 1) / kYC;
    // y: work items of (column strip of kYC) x (kYRows rows), one wave of resident CTAs
    const int64_t yitems = nchunk * ((pair_rows + kYRows - 1) / kYRows);
    const int64_t yblocks = std::max<int64_t>(1, std::min<int64_t>(yitems, TG_VGY_GRID * static_cast<int64_t>(sm)));
    // TG_VG_CONCURRENT: the y pass runs on a forked stream beside the x pass
    // (their sums are disjoint).  Off: measured no gain (8192^2: 0.610 vs
    // 0.618 ms; 32768^2: 10.20 vs 10.13 ms) since the x pass's shared loads and
    // the y pass's global loads share the L1 data pipe.
    cudaStream_t sy = s;
    cudaEvent_t fork = nullptr, join = nullptr;
    if (TG_VG_CONCURRENT) {
        thread_local cudaStream_t side[64] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 64 && (side[dev] || cudaStreamCreateWithFlags(&side[dev], cudaStreamNonBlocking) == cudaSuccess) &&
            cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&join, cudaEventDisableTiming) == cudaSuccess) {
            sy = side[dev];
            e = cudaEventRecord(fork, s);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(sy, fork, 0);
            if (e != cudaSuccess) return set_cuda_error(e, "variogram fork");
        }
    }
    const bool vec = (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(dev_map) & 15) == 0;
    // power-of-two lags up to 4096 (config 5's set): register-ring walks (vgring.cu)
    const int ring = vg_ring_enqueue(dev_map, width, height, ld, pair_rows, lags, n_lags, sums, sm, s, sy);
    if (ring < 0) return ring;
    for (int l0 = 0; ring && l0 < n_lags && e == cudaSuccess && pair_rows > 0; l0 += kFusedLags) {
        const int n = std::min(kFusedLags, n_lags - l0);
        LagSet Lx{}, Ly{};
        Lx.n = Ly.n = n;
        Lx.hmax = Ly.hmax = 0;
        bool long_x = false;
        for (int i = 0; i < kFusedLags; ++i) {
            const int64_t h = i < n ? lags[l0 + i] : 0;
            const bool pad = i >= n || h >= (int64_t(1) << 30);  // >= 2^30: no pair on either axis
            Lx.h[i] = Ly.h[i] = pad ? 0 : static_cast<int>(h);  // 0: the sample itself (d = 0)
            if (!pad) Lx.hmax = Ly.hmax = std::max(Lx.hmax, static_cast<int>(h));
            long_x = long_x || (!pad && h > kApron);
        }
        const int vi = (n - 1) / 2;
        // TG_VG_AXES (timing experiments only): 1 = x pass only, 2 = y pass only
        static const int axes = getenv("TG_VG_AXES") ? atoi(getenv("TG_VG_AXES")) : 3;
        if (axes & 1) xt[long_x ? 1 : 0][vi]<<<static_cast<unsigned>(xblocks), kVgThreads, smem, s>>>(
            dev_map, width, ld, pair_rows, Lx, nseg, seg_cap, sums + 2 * l0);
        if ((e = cudaGetLastError()) != cudaSuccess) break;
        if (axes & 2) yt[vec ? 1 : 0][vi]<<<static_cast<unsigned>(yblocks), kVgThreads, 0, sy>>>(dev_map, width, height, ld,
                                                                                  pair_rows, Ly, sums + 2 * l0);
        e = cudaGetLastError();
    }
    if (sy != s) {  // join (also on error: the scratch is freed in stream order on s)
        const cudaError_t ej = cudaEventRecord(join, sy);
        const cudaError_t ew = ej == cudaSuccess ? cudaStreamWaitEvent(s, join, 0) : ej;
        if (e == cudaSuccess) e = ew;
    }
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out_sum_sq, sums, 2 * n_lags * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_cuda_error(e, "variogram");
    for (int i = 0; ring == 0 && i < n_lags; ++i)  // the ring path sums a repeated lag once
        for (int j = 0; j < i; ++j)
            if (lags[j] == lags[i]) {
                out_sum_sq[2 * i] = out_sum_sq[2 * j];
                out_sum_sq[2 * i + 1] = out_sum_sq[2 * j + 1];
                break;
            }
    for (int i = 0; i < n_lags; ++i) {
        const int64_t h = lags[i];
        out_pairs[2 * i] = h < width ? (width - h) * pair_rows : 0;
        const int64_t ny = std::min<int64_t>(pair_rows, height - h);
        out_pairs[2 * i + 1] = ny > 0 ? width * ny : 0;
    }
    return TG_OK;
}

int tg_variogram_f32(const float* dev_map, int64_t width, int64_t height, int64_t ld, const int32_t* lags,
                     int32_t n_lags, double* out_sum_sq, int64_t* out_pairs, void* stream) {
    return tg_variogram_band_f32(dev_map, width, height, ld, height, lags, n_lags, out_sum_sq, out_pairs, stream);
}

// Local histogram of the radix-select digit (shift, bits) among keys whose
// fixed bits (mask) equal prefix — the per-rank step of a distributed upper
// median whose histograms are summed across GPUs.
int tg_histogram_f32(const float* dev_rows, int64_t width, int64_t rows, int64_t ld, uint32_t prefix,
                     uint32_t mask, int32_t shift, int32_t bits, uint64_t* out_hist, void* stream) {
    if (!dev_rows || !out_hist || width < 1 || rows < 1 || ld < width || bits < 1 || bits > 11 || shift < 0 ||
        shift + bits > 32)
        return set_error(TG_EVALIDATION, "histogram: bad arguments");
    if (int st = check_device()) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Scratch scr(s);
    cudaError_t e = scr.alloc(64 + kBins * sizeof(unsigned long long));
    if (e != cudaSuccess) return set_cuda_error(e, "histogram alloc");
    SelectState* state = static_cast<SelectState*>(scr.p);
    auto* hist = reinterpret_cast<unsigned long long*>(static_cast<char*>(scr.p) + 64);
    SelectState init{prefix, mask, 0};
    e = cudaMemcpyAsync(state, &init, sizeof(init), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(hist, 0, kBins * sizeof(unsigned long long), s);
    const int blocks = static_cast<int>(std::min<int64_t>(rows, kHistBlocks));
    if (e == cudaSuccess) {
        if (ld == width)
            radix_hist<<<kHistBlocks, 512, 0, s>>>(dev_rows, static_cast<uint64_t>(width * rows), state, shift, bits,
                                                   hist);
        else
            radix_hist2d<<<blocks, 512, 0, s>>>(dev_rows, width, rows, ld, state, shift, bits, hist);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(out_hist, hist, (size_t{1} << bits) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return set_cuda_error(e, "histogram");
    return TG_OK;
}

}  // extern "C"
