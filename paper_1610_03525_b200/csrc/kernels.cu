// kernels.cu — small device kernels behind the C-ABI: lattice probes
// (lattice.hpp parity), fp32->fp64 widening for the drop-in span<double>,
// min/max + rescale (normalize_map, fbm.hpp:638-656) and the FFMA-chain
// peak used as the FP32 roofline denominator.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/polyterrain_b200.h"
#include "fbm_params.h"
#include "lattice.cuh"

namespace tg {
int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
int check_device();

__global__ void lattice_kernel(int what, const tg_lattice_key* __restrict__ keys, uint64_t n,
                               uint64_t lane, void* __restrict__ out) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const tg_lattice_key k = keys[i];
        const uint64_t base = k.seed * kSeedMul + static_cast<uint64_t>(k.octave) * kOctMul;
        if (what == 0) {
            static_cast<uint64_t*>(out)[i] = mix64(pack_xy(base, k.ix, k.iy) ^ lane);
        } else if (what == 1) {
            static_cast<float*>(out)[i] = corner_height(base, k.ix, k.iy);
        } else {
            float c, s;
            corner_unit_gradient(base, k.ix, k.iy, &c, &s);
            static_cast<float*>(out)[2 * i] = c;
            static_cast<float*>(out)[2 * i + 1] = s;
        }
    }
}

cudaError_t lattice_launch(int what, const tg_lattice_key* keys, uint64_t n, uint64_t lane,
                           void* out, cudaStream_t st) {
    const uint64_t blocks = (n + 255) / 256;
    lattice_kernel<<<static_cast<unsigned>(blocks < 65535 * 16 ? blocks : 65535 * 16), 256, 0, st>>>(
        what, keys, n, lane, out);
    return cudaGetLastError();
}

// Row LUTs (kernels2d::build_row_lut at phase 0.5, kernels2d.hpp:214-239) for
// every power-of-two ppc up to 2^kLutLog2Max, both smoothstep orders, computed
// once per device in fp64 and rounded to fp32: entry (x, S(x), S(x)-x, x*S(x))
// at [ppc - 1 + r], followed by two planar copies, S(x) at float [ppc + r] and
// S(x) - x at float [kLutN4 + ppc + r] past the kLutN4-entry float4 block, so
// that 4 consecutive rows / columns are one aligned 16-byte load, then the
// pairs (S(x), S(x) - x) as float2 at [ppc + r] (one 8-byte load per column).
// Immutable after creation, so concurrent callers share it (like the
// reference's thread-local cached_row_lut, kernels2d.hpp:246-259).
const float4* row_lut(int order) {
    constexpr int kMaxDev = 64;
    static std::mutex mu;
    static float4* luts[kMaxDev][2] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
    const int oi = order == 5 ? 1 : 0;
    std::lock_guard<std::mutex> lock(mu);
    if (luts[dev][oi]) return luts[dev][oi];
    std::vector<float4> h(static_cast<size_t>(kLutN4 + 2 * kLutN4 / 4 + kLutN4 / 2), make_float4(0.f, 0.f, 0.f, 0.f));
    float* planes = reinterpret_cast<float*>(h.data() + kLutN4);
    float2* sd = reinterpret_cast<float2*>(h.data() + kLutN4 + kLutN4 / 2);  // (S, S - x) at [ppc + r]
    for (int k = 0; k <= kLutLog2Max; ++k) {
        const int ppc = 1 << k;
        for (int r = 0; r < ppc; ++r) {
            const double x = (static_cast<double>(r) + 0.5) / static_cast<double>(ppc);
            const double sv = order == 5 ? x * x * x * (10.0 + x * (6.0 * x - 15.0)) : x * x * (3.0 - 2.0 * x);
            h[static_cast<size_t>(ppc - 1 + r)] = make_float4(static_cast<float>(x), static_cast<float>(sv),
                                                              static_cast<float>(sv - x), static_cast<float>(x * sv));
            planes[ppc + r] = static_cast<float>(sv);
            planes[kLutN4 + ppc + r] = static_cast<float>(sv - x);
            sd[ppc + r] = make_float2(static_cast<float>(sv), static_cast<float>(sv - x));
        }
    }
    float4* d = nullptr;
    if (cudaMalloc(&d, sizeof(float4) * h.size()) != cudaSuccess) return nullptr;
    // A pageable cudaMemcpy may return before the DMA lands; the first
    // generation launch can go onto a non-blocking stream that does not wait
    // on the legacy stream, so complete the copy before publishing the LUT.
    if (cudaMemcpy(d, h.data(), sizeof(float4) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        cudaFree(d);
        return nullptr;
    }
    luts[dev][oi] = d;
    return d;
}

__global__ void widen_kernel(const float* __restrict__ in, double* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = static_cast<double>(in[i]);
}

// normalize_map (fbm.hpp:638-656) fused into the fp32 -> fp64 widening of
// the drop-in's host copy: -1 + 2 (v - lo) / span in fp64 on the exactly
// widened sample, the reference's expression and operation order (653).
__global__ void widen_normalize_kernel(const float* __restrict__ in, double* __restrict__ out, uint64_t n,
                                       double lo, double span, int norm) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double v = static_cast<double>(in[i]);
        out[i] = norm ? -1.0 + 2.0 * (v - lo) / span : v;
    }
}

cudaError_t widen_normalize_launch(const float* in, double* out, uint64_t n, double lo, double span, int norm,
                                   cudaStream_t st) {
    widen_normalize_kernel<<<148 * 8, 256, 0, st>>>(in, out, n, lo, span, norm);
    return cudaGetLastError();
}

cudaError_t widen_launch(const float* in, double* out, uint64_t n, cudaStream_t st) {
    widen_kernel<<<148 * 8, 256, 0, st>>>(in, out, n);
    return cudaGetLastError();
}

// Order-preserving float <-> uint32 key (for min/max atomics and radix select).
__device__ __forceinline__ uint32_t fkey(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float funkey(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__global__ void minmax_kernel(const float* __restrict__ x, uint64_t n, uint32_t* __restrict__ mm) {
    uint32_t lo = 0xffffffffu, hi = 0u;
    const uint64_t n4 = n / 4;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (aligned) {
        for (uint64_t i = i0; i < n4; i += stride) {
            const float4 v = x4[i];
            const uint32_t a = fkey(v.x), b = fkey(v.y), c = fkey(v.z), d = fkey(v.w);
            lo = min(lo, min(min(a, b), min(c, d)));
            hi = max(hi, max(max(a, b), max(c, d)));
        }
        for (uint64_t i = n4 * 4 + i0; i < n; i += stride) {
            const uint32_t a = fkey(x[i]);
            lo = min(lo, a);
            hi = max(hi, a);
        }
    } else {
        for (uint64_t i = i0; i < n; i += stride) {
            const uint32_t a = fkey(x[i]);
            lo = min(lo, a);
            hi = max(hi, a);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&mm[0], lo);
        atomicMax(&mm[1], hi);
    }
}

__global__ void rescale_kernel(float* __restrict__ x, uint64_t n, double lo, double span) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        x[i] = static_cast<float>(-1.0 + 2.0 * (static_cast<double>(x[i]) - lo) / span);  // fbm.hpp:653
}

// quantize16 (io.hpp:61-65): lround((v - lo)/(hi - lo) * 65535) in fp64 on
// the fp32 map widened exactly, written big-endian; with png_rows each row is
// prefixed by PNG filter byte 0 (io.hpp:228-239).  lround = round half away
// from zero; t >= 0 here so it is floor(x) + (frac >= 0.5).
__global__ void pack16_kernel(const float* __restrict__ m, int64_t W, int64_t H, int64_t ld, double lo,
                              double hi, int png_rows, unsigned char* __restrict__ out) {
    const int64_t row_bytes = 2 * W + (png_rows ? 1 : 0);
    for (int64_t y = blockIdx.x; y < H; y += gridDim.x) {
        unsigned char* o = out + y * row_bytes;
        if (png_rows && threadIdx.x == 0) o[0] = 0;
        unsigned char* os = o + (png_rows ? 1 : 0);
        for (int64_t x = threadIdx.x; x < W; x += blockDim.x) {
            uint32_t s = 0;
            if (hi != lo) {
                const double t = __ddiv_rn(__dsub_rn(static_cast<double>(m[y * ld + x]), lo), __dsub_rn(hi, lo));
                const double v = __dmul_rn(t, 65535.0);
                const double f = floor(v);
                s = static_cast<uint32_t>(f) + (__dsub_rn(v, f) >= 0.5 ? 1u : 0u);
            }
            os[2 * x] = static_cast<unsigned char>(s >> 8);
            os[2 * x + 1] = static_cast<unsigned char>(s & 0xFF);
        }
    }
}

// gradient / Hessian norm maps (terrain_cli.cpp:148-182): central
// differences inside, clamped at the borders, in fp64 on the fp32 map widened
// exactly, one rounding to fp32 at the end.
__global__ void stencil_kernel(const float* __restrict__ m, int64_t W, int64_t H, int hessian,
                               float* __restrict__ out) {
    for (int64_t y = blockIdx.x; y < H; y += gridDim.x) {
        const int64_t ym = y > 0 ? y - 1 : 0, yp = y + 1 < H ? y + 1 : H - 1;
        for (int64_t x = threadIdx.x; x < W; x += blockDim.x) {
            const int64_t xm = x > 0 ? x - 1 : 0, xp = x + 1 < W ? x + 1 : W - 1;
            const auto at = [&](int64_t xx, int64_t yy) { return static_cast<double>(m[yy * W + xx]); };
            double v;
            if (!hessian) {
                const double gx = 0.5 * (at(xp, y) - at(xm, y));
                const double gy = 0.5 * (at(x, yp) - at(x, ym));
                v = sqrt(gx * gx + gy * gy);
            } else {
                const double c = at(x, y);
                const double hxx = at(xp, y) - 2.0 * c + at(xm, y);
                const double hyy = at(x, yp) - 2.0 * c + at(x, ym);
                const double hxy = 0.25 * (at(xp, yp) - at(xm, yp) - at(xp, ym) + at(xm, ym));
                v = sqrt(hxx * hxx + 2.0 * hxy * hxy + hyy * hyy);
            }
            out[y * W + x] = static_cast<float>(v);
        }
    }
}

// Eight independent FFMA chains per thread: issue-bound FP32 peak.
__global__ void ffma_kernel(float* out, int iters) {
    float a0 = threadIdx.x * 1e-7f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
    float a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const float m = 0.9999999f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            a0 = fmaf(a0, m, c); a1 = fmaf(a1, m, c); a2 = fmaf(a2, m, c); a3 = fmaf(a3, m, c);
            a4 = fmaf(a4, m, c); a5 = fmaf(a5, m, c); a6 = fmaf(a6, m, c); a7 = fmaf(a7, m, c);
        }
    }
    const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (s == 123.456f) out[0] = s;
}

}  // namespace tg

extern "C" {

int tg_minmax_f32(const float* dev_map, uint64_t n, double* out_min, double* out_max,
                  void* stream) {
    if (!dev_map || !out_min || !out_max || n == 0)
        return tg::set_error(TG_EVALIDATION, "minmax: empty or null input");
    if (int st = tg::check_device()) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint32_t* mm = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&mm), 2 * sizeof(uint32_t), s);
    if (e != cudaSuccess) return tg::set_cuda_error(e, "minmax alloc");
    const uint32_t init[2] = {0xffffffffu, 0u};
    uint32_t res[2];
    e = cudaMemcpyAsync(mm, init, sizeof(init), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
        tg::minmax_kernel<<<148 * 4, 256, 0, s>>>(dev_map, n, mm);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(res, mm, sizeof(res), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(mm, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return tg::set_cuda_error(e, "minmax");
    const auto unkey = [](uint32_t k) {
        const uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
        float f;
        std::memcpy(&f, &b, 4);
        return static_cast<double>(f);
    };
    *out_min = unkey(res[0]);
    *out_max = unkey(res[1]);
    return TG_OK;
}

int tg_rescale_f32(float* dev_map, uint64_t n, double lo, double hi, void* stream) {
    if (!dev_map) return tg::set_error(TG_EVALIDATION, "rescale: null input");
    if (!(hi > lo)) return tg::set_error(TG_EVALIDATION, "rescale: empty range");
    if (n == 0) return TG_OK;
    if (int st = tg::check_device()) return st;
    tg::rescale_kernel<<<148 * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(dev_map, n, lo,
                                                                                 hi - lo);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return tg::set_cuda_error(e, "rescale");
    return TG_OK;
}

int tg_pack16_f32(const float* dev_map, int64_t width, int64_t height, int64_t ld, double lo, double hi,
                  int32_t png_rows, uint8_t* dev_out, void* stream) {
    if (!dev_map || !dev_out || width < 1 || height < 1 || ld < width)
        return tg::set_error(TG_EVALIDATION, "pack16: bad arguments");
    if (int st = tg::check_device()) return st;
    const int blocks = static_cast<int>(height < 148 * 8 ? height : 148 * 8);
    tg::pack16_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(dev_map, width, height, ld, lo, hi,
                                                                             png_rows, dev_out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return tg::set_cuda_error(e, "pack16");
    return TG_OK;
}

int tg_norm_map_f32(const float* dev_map, int64_t width, int64_t height, int32_t hessian, float* dev_out,
                    void* stream) {
    if (!dev_map || !dev_out || width < 1 || height < 1 || dev_map == dev_out)
        return tg::set_error(TG_EVALIDATION, "norm map: bad arguments");
    if (int st = tg::check_device()) return st;
    const int blocks = static_cast<int>(height < 148 * 8 ? height : 148 * 8);
    tg::stencil_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(dev_map, width, height,
                                                                              hessian ? 1 : 0, dev_out);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return tg::set_cuda_error(e, "norm map");
    return TG_OK;
}

int tg_measure_ffma_peak(double* out_tflops, double* out_ms) {
    if (int st = tg::check_device()) return st;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* sink = nullptr;
    cudaError_t e = cudaMalloc(&sink, sizeof(float));
    if (e != cudaSuccess) return tg::set_cuda_error(e, "ffma alloc");
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    tg::ffma_kernel<<<blocks, threads>>>(sink, 64);  // warm-up / clock ramp
    tg::ffma_kernel<<<blocks, threads>>>(sink, iters);
    cudaEventRecord(a);
    tg::ffma_kernel<<<blocks, threads>>>(sink, iters);
    cudaEventRecord(b);
    e = cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(sink);
    if (e != cudaSuccess) return tg::set_cuda_error(e, "ffma");
    const double flops = 2.0 * 8.0 * 16.0 * iters * static_cast<double>(blocks) * threads;
    *out_tflops = flops / (ms * 1e-3) / 1e12;
    if (out_ms) *out_ms = ms;
    return TG_OK;
}

}  // extern "C"
