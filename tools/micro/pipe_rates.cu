// Throughput of the integer / conversion instructions the lattice hash uses
// (B200, sm_100a): warp-instructions per SM per cycle for long independent
// chains.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_rates pipe_rates.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 4096, kChains = 8;

template <int OP>
__global__ void rate(uint32_t* out, uint32_t seed) {
    uint32_t a[kChains], b[kChains], ib[kChains];
    const float2 m2 = make_float2(__uint_as_float(seed) * 0.5f, 0.999f), k2 = make_float2(1e-3f, __uint_as_float(seed));
#pragma unroll
    for (int c = 0; c < kChains; ++c) { a[c] = seed + threadIdx.x * 7 + c; b[c] = a[c] * 3u + 1u; ib[c] = a[c]; }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if constexpr (OP == 0) {  // IMAD (mad.lo, immediate)
                asm volatile("mad.lo.u32 %0, %0, 0x1A85EC53, %1;" : "+r"(a[c]) : "r"(b[c]));
            } else if constexpr (OP == 1) {  // 64-bit multiply on halves: IMAD.WIDE.U32 + 2 IMAD
                asm volatile("{.reg .b64 p; mul.wide.u32 p, %0, 0xED558CCD; mov.b64 {%0, %1}, p;"
                             "mad.lo.u32 %1, %2, 0xED558CCD, %1; mad.lo.u32 %1, %3, 0xFF51AFD7, %1;}"
                             : "+r"(a[c]), "=r"(b[c]) : "r"(b[c]), "r"(a[c]));
            } else if constexpr (OP == 2) {  // IMAD.HI.U32
                asm volatile("mul.hi.u32 %0, %0, 0x1A85EC53;" : "+r"(a[c]));
                asm volatile("add.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(b[c]));
            } else if constexpr (OP == 3) {  // LOP3 + SHF: x ^= y >> 1
                asm volatile("{.reg .b32 t; shr.b32 t, %1, 1; xor.b32 %0, %0, t;}" : "+r"(a[c]) : "r"(b[c]));
                asm volatile("{.reg .b32 t; shr.b32 t, %1, 1; xor.b32 %0, %0, t;}" : "+r"(b[c]) : "r"(a[c]));
            } else if constexpr (OP == 4) {  // I2FP.F32.U32 then back (F2I on the other side)
                float f;
                asm volatile("cvt.rn.f32.u32 %0, %1;" : "=f"(f) : "r"(a[c]));
                asm volatile("mov.b32 %0, %1;" : "=r"(a[c]) : "f"(f));
            } else if constexpr (OP == 5) {  // FFMA 3-register
                float f = __uint_as_float(a[c]), g = __uint_as_float(b[c]);
                asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(f) : "f"(g));
                a[c] = __float_as_uint(f);
            } else if constexpr (OP == 7) {  // FFMA2 (fma.rn.f32x2): two fp32 FMAs per lane
                float2 x = make_float2(__uint_as_float(a[c]), __uint_as_float(b[c]));
                x = __ffma2_rn(x, m2, k2);
                a[c] = __float_as_uint(x.x); b[c] = __float_as_uint(x.y);
            } else if constexpr (OP == 8) {  // FFMA2 + IMAD interleaved (co-issue across pipes)
                float2 x = make_float2(__uint_as_float(a[c]), __uint_as_float(b[c]));
                x = __ffma2_rn(x, m2, k2);
                a[c] = __float_as_uint(x.x); b[c] = __float_as_uint(x.y);
                asm volatile("mad.lo.u32 %0, %0, 0x1A85EC53, %1;" : "+r"(ib[c]) : "r"(seed));
            } else if constexpr (OP == 9) {  // FRND.F32.FLOOR
                float f = __uint_as_float(a[c]);
                asm volatile("cvt.rmi.f32.f32 %0, %0;" : "+f"(f));
                a[c] = __float_as_uint(f) + 1u;
            } else if constexpr (OP == 10) {  // FADD.RM (floor via 1.5 * 2^23)
                float f = __uint_as_float(a[c]);
                asm volatile("add.rm.f32 %0, %0, 0f4B400000;" : "+f"(f));
                a[c] = __float_as_uint(f);
            } else if constexpr (OP == 11) {  // FFMA + IMAD interleaved
                float f = __uint_as_float(a[c]);
                asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(f));
                a[c] = __float_as_uint(f);
                asm volatile("mad.lo.u32 %0, %0, 0x1A85EC53, %1;" : "+r"(b[c]) : "r"(a[c]));
            } else if constexpr (OP == 6) {  // mul.wide alone, both halves consumed
                asm volatile("{.reg .b64 p; mul.wide.u32 p, %0, 0xED558CCD; mov.b64 {%0, %1}, p; xor.b32 %0, %0, %1;}"
                             : "+r"(a[c]), "=r"(b[c]));
            }
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s ^= a[c] ^ b[c] ^ ib[c];
    if (s == 0x12345678u) out[0] = s;
}

template <int OP>
void run(const char* name, int per_iter) {
    uint32_t* d;
    cudaMalloc(&d, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    dim3 grid(sms * 8), block(256);
    rate<OP><<<grid, block>>>(d, 1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    rate<OP><<<grid, block>>>(d, 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_instr = double(grid.x) * 8 * kIters * kChains * per_iter;  // 8 warps per block
    const double cycles = ms * 1e-3 * clk * 1e3;
    printf("%-28s %7.3f ms  %6.3f warp-instr/SM/cycle (at %d MHz max clock)\n", name, ms,
           warp_instr / cycles / sms, clk / 1000);
    cudaFree(d);
}

int main() {
    run<0>("IMAD imm", 1);
    run<1>("MUL64: WIDE + 2 IMAD", 3);
    run<2>("IMAD.HI.U32 (+addend)", 1);
    run<3>("SHF + LOP3", 4);
    run<4>("I2FP.F32.U32", 1);
    run<5>("FFMA 3-reg", 1);
    run<6>("IMAD.WIDE.U32 + LOP3", 2);
    run<7>("FFMA2 (f32x2)", 1);
    run<8>("FFMA2 + IMAD", 2);
    run<9>("FRND.F32.FLOOR (+IADD)", 2);
    run<10>("FADD.RM", 1);
    run<11>("FFMA + IMAD", 2);
    return 0;
}
