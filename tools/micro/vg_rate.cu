// Instruction rates behind the variogram (B200, sm_100a): DFMA / DADD,
// F2F.F64.F32, and the per-pair patterns (register pair, shared-memory fp32
// partner + conversion).  Reported as pairs (or ops) per SM per cycle.
// Measured (round 2): DFMA 60/SM/clk; LDS.64 partner + DADD + DFMA 15.2 pairs
// (shared-memory bandwidth: 8 B per pair); LDS.32 partner + F2F + DADD + DFMA
// 13.2 pairs.  The register-operand variants (OP 2, 3, 5, 6) read ~60 because
// the compiler hoists the toggled operand's conversion — not a real rate; ncu
// on the variogram kernels shows F2F.F64.F32 on the XU pipe (16 lanes/SM/clk).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o vg_rate vg_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kIters = 2048, kC = 8;

template <int OP>
__global__ void __launch_bounds__(256) k(float* out, float seed) {
    __shared__ float sm[4096];
    for (int i = threadIdx.x; i < 4096; i += 256) sm[i] = seed * i;
    __syncthreads();
    double acc[kC];
    double v[kC];
    float f[kC];
#pragma unroll
    for (int c = 0; c < kC; ++c) {
        acc[c] = 0.0;
        v[c] = seed + threadIdx.x + c;
        f[c] = seed * (threadIdx.x + c);
    }
    int idx = threadIdx.x;
    __shared__ double smd[2048];
    for (int i = threadIdx.x; i < 2048; i += 256) smd[i] = seed * i;
    __syncthreads();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int c = 0; c < kC; ++c) {
            if constexpr (OP == 0) {  // DFMA only
                acc[c] = fma(v[c], v[c], acc[c]);
            } else if constexpr (OP == 1) {  // register pair: DADD + DFMA
                const double d = v[(c + 1) % kC] - v[c];
                acc[c] = fma(d, d, acc[c]);
            } else if constexpr (OP == 2) {  // F2F.F64.F32 + DADD
                acc[c] += static_cast<double>(f[c]);
            } else if constexpr (OP == 3) {  // fp32 register partner: F2F + DADD + DFMA
                const double d = static_cast<double>(f[c]) - v[c];
                acc[c] = fma(d, d, acc[c]);
            } else if constexpr (OP == 4) {  // LDS.32 partner + F2F + DADD + DFMA
                const double d = static_cast<double>(sm[(idx + 32 * c) & 4095]) - v[c];
                acc[c] = fma(d, d, acc[c]);
            } else if constexpr (OP == 5) {  // fp32 difference squared (FADD + F2F + DFMA)
                const float s = f[(c + 1) % kC] - f[c];
                const double d = static_cast<double>(s);
                acc[c] = fma(d, d, acc[c]);
            } else if constexpr (OP == 6) {  // both operands converted: 2 F2F + DADD + DFMA
                const double d = static_cast<double>(f[(c + 1) % kC]) - static_cast<double>(f[c]);
                acc[c] = fma(d, d, acc[c]);
            } else if constexpr (OP == 7) {  // LDS.64 partner + DADD + DFMA
                const double d = smd[(idx + 32 * c) & 2047] - v[c];
                acc[c] = fma(d, d, acc[c]);
            }
        }
        idx += 7;
        // loop-carried operand changes on the ALU pipe (integer xor of a low bit)
#pragma unroll
        for (int c = 0; c < kC; ++c) {
            if constexpr (OP == 1) v[c] = __hiloint2double(__double2hiint(v[c]), __double2loint(v[c]) ^ it);
            if constexpr (OP == 2 || OP == 3 || OP == 5 || OP == 6) f[c] = __int_as_float(__float_as_int(f[c]) ^ (it & 1));
        }
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kC; ++c) s += acc[c];
    if (s == 1.2345) out[0] = static_cast<float>(s);
}

template <int OP>
void run(const char* name) {
    float* d;
    cudaMalloc(&d, 4);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    dim3 grid(sms * 8), block(256);
    k<OP><<<grid, block>>>(d, 1.0f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<grid, block>>>(d, 2.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double units = double(grid.x) * 256 * kIters * kC;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-44s %7.3f ms  %6.2f per SM per cycle\n", name, ms, units / cyc / sms);
    cudaFree(d);
}

int main() {
    run<0>("DFMA");
    run<1>("pair: DADD + DFMA (registers)");
    run<2>("F2F.F64.F32 (+DADD)");
    run<3>("pair: F2F + DADD + DFMA");
    run<4>("pair: LDS.32 + F2F + DADD + DFMA");
    run<5>("pair: FADD + F2F + DFMA (fp32 difference)");
    run<6>("pair: 2 F2F + DADD + DFMA");
    run<7>("pair: LDS.64 + DADD + DFMA");
    return 0;
}
