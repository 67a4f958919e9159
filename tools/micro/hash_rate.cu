// Achievable throughput of the map-path lattice hash (lattice.cuh) on B200,
// in the shapes the fBm kernel uses it: N independent chains per thread of
// (64-bit key add, fmix64 top word, I2FP, FFMA accumulate), 256-thread CTAs at
// 4 CTAs/SM (64 registers), optionally with extra independent FFMA work per
// hash to see how much FP work rides free beside the integer pipes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_1610_03525_b200/csrc -o hash_rate hash_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "lattice.cuh"

using namespace tg;

constexpr int kIters = 512;

template <int N, int XF>
__global__ void __launch_bounds__(256, 4) hash_chains(float* out, uint64_t k0, uint64_t kx) {
    uint64_t key = k0 + (blockIdx.x * 256ull + threadIdx.x) * 0x9E3779B97F4A7C15ULL;
    float acc[N];
    float x[XF > 0 ? XF : 1];
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = 0.f;
#pragma unroll
    for (int i = 0; i < (XF > 0 ? XF : 1); ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < kIters; ++it) {
        uint64_t p[N];
        p[0] = key;
#pragma unroll
        for (int i = 1; i < N; ++i) p[i] = add64(p[i - 1], kx);
        float h[N];
        map_heightN<N>(p, h);
#pragma unroll
        for (int i = 0; i < N; ++i) acc[i] = fmaf(0x1p-31f, h[i], acc[i]);
        if constexpr (XF > 0) {
#pragma unroll
            for (int j = 0; j < N; ++j)
#pragma unroll
                for (int i = 0; i < XF; ++i) x[i] = fmaf(x[i], 0.999f, acc[j]);
        }
        key = add64(p[N - 1], kx);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) s += acc[i];
#pragma unroll
    for (int i = 0; i < (XF > 0 ? XF : 1); ++i) s += x[i];
    if (s == 123.456f) out[0] = s;
}

template <int N, int XF>
void run(const char* name) {
    float* d;
    cudaMalloc(&d, 4);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    dim3 grid(sms * 4 * 4), block(256);
    hash_chains<N, XF><<<grid, block>>>(d, 1, 0x94D049BB133111EBULL * 2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    hash_chains<N, XF><<<grid, block>>>(d, 2, 0x94D049BB133111EBULL * 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_hashes = double(grid.x) * 8 * kIters * N;
    const double smsp_cycles = ms * 1e-3 * clk * 1e3 * sms * 4;
    printf("%-34s %7.3f ms  %6.2f SMSP-cycles per warp-hash  (%.3g hashes/s)\n", name, ms,
           smsp_cycles / warp_hashes, warp_hashes * 32 / (ms * 1e-3));
    cudaFree(d);
}

int main() {
    run<4, 0>("4 chains");
    run<8, 0>("8 chains");
    run<12, 0>("12 chains");
    run<16, 0>("16 chains");
    run<8, 1>("8 chains + 1 FFMA/hash");
    run<8, 2>("8 chains + 2 FFMA/hash");
    run<8, 4>("8 chains + 4 FFMA/hash");
    return 0;
}
