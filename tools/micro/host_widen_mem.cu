// Host fp32 -> fp64 widening throughput against the KIND of host memory on
// either side (no kernels): malloc with transparent huge pages, malloc with
// MADV_NOHUGEPAGE, cudaHostAlloc, and mmap + MADV_HUGEPAGE + cudaHostRegister.
//   nvcc -O3 -Xcompiler -pthread -o host_widen_mem host_widen_mem.cu && ./host_widen_mem [threads]
#include <cuda_runtime.h>
#include <immintrin.h>
#include <sys/mman.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

__attribute__((target("avx512f"))) static void widen_nt512(const float* s, double* d, size_t n) {
    for (size_t i = 0; i + 16 <= n; i += 16) {
        const __m512 a = _mm512_loadu_ps(s + i);
        _mm512_stream_pd(d + i, _mm512_cvtps_pd(_mm512_castps512_ps256(a)));
        _mm512_stream_pd(d + i + 8, _mm512_cvtps_pd(_mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castps_pd(a), 1))));
    }
    _mm_sfence();
}

static void* get(int kind, size_t bytes) {
    void* p = nullptr;
    if (kind == 0 || kind == 1) {
        p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        madvise(p, bytes, kind == 0 ? MADV_HUGEPAGE : MADV_NOHUGEPAGE);
    } else if (kind == 2) {
        if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
    } else {
        p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        madvise(p, bytes, MADV_HUGEPAGE);
        for (size_t i = 0; i < bytes; i += 4096) static_cast<char*>(p)[i] = 0;
        if (cudaHostRegister(p, bytes, cudaHostRegisterDefault) != cudaSuccess) return nullptr;
    }
    for (size_t i = 0; i < bytes; i += 64) static_cast<char*>(p)[i] = 1;
    return p;
}

int main(int argc, char** argv) {
    const int t = argc > 1 ? atoi(argv[1]) : 6;
    const size_t n = size_t(1) << 24;
    const char* names[4] = {"thp", "4k", "cudaHostAlloc", "thp+register"};
    cudaFree(0);
    for (int sk = 0; sk < 4; ++sk)
        for (int dk = 0; dk < 4; ++dk) {
            float* src = static_cast<float*>(get(sk, n * 4));
            double* dst = static_cast<double*>(get(dk, n * 8));
            if (!src || !dst) { printf("%s -> %s: alloc failed\n", names[sk], names[dk]); continue; }
            double best = 1e9;
            for (int rep = 0; rep < 8; ++rep) {
                std::atomic<int> go{0};
                std::vector<std::thread> th;
                const size_t per = n / t / 64 * 64;
                for (int k = 0; k < t; ++k)
                    th.emplace_back([&, k] {
                        while (!go.load()) {}
                        const size_t b = k * per, m = (k == t - 1) ? n - b : per;
                        widen_nt512(src + b, dst + b, m);
                    });
                const auto t0 = std::chrono::steady_clock::now();
                go.store(1);
                for (auto& x : th) x.join();
                const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                if (s < best) best = s;
            }
            printf("src %-14s dst %-14s threads=%d  %6.3f ms  %6.2f Gelem/s\n", names[sk], names[dk], t, best * 1e3,
                   n / best * 1e-9);
            // (buffers leak: one-shot probe)
        }
    // The same widening (cudaHostAlloc on both sides) while the copy engine
    // streams device -> host into another pinned buffer.
    {
        float* src = static_cast<float*>(get(2, n * 4));
        double* dst = static_cast<double*>(get(2, n * 8));
        float* land = static_cast<float*>(get(2, n * 4));
        float* dev = nullptr;
        cudaMalloc(&dev, n * 4);
        cudaStream_t st;
        cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        for (int dma = 0; dma < 2; ++dma)
            for (int tt : {4, 6, 8, 12}) {
                double best = 1e9;
                for (int rep = 0; rep < 6; ++rep) {
                    if (dma)
                        for (int k = 0; k < 4; ++k) cudaMemcpyAsync(land, dev, n * 4, cudaMemcpyDeviceToHost, st);
                    std::this_thread::sleep_for(std::chrono::microseconds(300));
                    std::atomic<int> go{0};
                    std::vector<std::thread> th;
                    const size_t per = n / tt / 64 * 64;
                    for (int k = 0; k < tt; ++k)
                        th.emplace_back([&, k] {
                            while (!go.load()) {}
                            const size_t b = k * per, m = (k == tt - 1) ? n - b : per;
                            widen_nt512(src + b, dst + b, m);
                        });
                    const auto t0 = std::chrono::steady_clock::now();
                    go.store(1);
                    for (auto& x : th) x.join();
                    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                    const bool still = dma && cudaStreamQuery(st) == cudaErrorNotReady;
                    cudaStreamSynchronize(st);
                    if (s < best && (!dma || still)) best = s;
                }
                printf("widen with%s D2H in flight, threads=%2d: %6.3f ms  %6.2f Gelem/s\n", dma ? "" : "out", tt,
                       best * 1e3, n / best * 1e-9);
            }
    }
    return 0;
}
