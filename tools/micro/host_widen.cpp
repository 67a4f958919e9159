// Host fp32 -> fp64 widening throughput against thread count (no GPU): what
// the host side of tg_fbm_generate_f64_host can sustain on this box.
//   g++ -O3 -pthread -o host_widen host_widen.cpp && ./host_widen
// Prints G elements/s (and GB/s read + written) for 1..16 threads, with
// non-temporal and regular stores, on a 64 MiB fp32 source (config 2).
#include <immintrin.h>

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
__attribute__((target("avx2"))) static void widen_nt256(const float* s, double* d, size_t n) {
    for (size_t i = 0; i + 8 <= n; i += 8) {
        const __m256 a = _mm256_loadu_ps(s + i);
        _mm256_stream_pd(d + i, _mm256_cvtps_pd(_mm256_castps256_ps128(a)));
        _mm256_stream_pd(d + i + 4, _mm256_cvtps_pd(_mm256_extractf128_ps(a, 1)));
    }
    _mm_sfence();
}
static void widen_plain(const float* s, double* d, size_t n) {
    for (size_t i = 0; i < n; ++i) d[i] = s[i];
}

int main() {
    const size_t n = size_t(1) << 24;
    float* src = static_cast<float*>(aligned_alloc(4096, n * 4));
    double* dst = static_cast<double*>(aligned_alloc(4096, n * 8));
    for (size_t i = 0; i < n; ++i) src[i] = float(i & 1023) * 0.25f;
    for (size_t i = 0; i < n; ++i) dst[i] = 0.0;
    const bool avx512 = __builtin_cpu_supports("avx512f");
    printf("avx512f=%d hw_threads=%u\n", int(avx512), std::thread::hardware_concurrency());
    for (int mode = 0; mode < 3; ++mode) {
        if (mode == 0 && !avx512) continue;
        for (int t : {1, 2, 4, 6, 8, 10, 12, 14, 16}) {
            double best = 1e9;
            for (int rep = 0; rep < 8; ++rep) {
                std::atomic<int> go{0};
                std::vector<std::thread> th;
                const size_t per = n / t / 64 * 64;
                for (int k = 0; k < t; ++k)
                    th.emplace_back([&, k] {
                        while (!go.load()) {}
                        const size_t b = k * per, m = (k == t - 1) ? n - b : per;
                        if (mode == 0) widen_nt512(src + b, dst + b, m);
                        else if (mode == 1) widen_nt256(src + b, dst + b, m);
                        else widen_plain(src + b, dst + b, m);
                    });
                const auto t0 = std::chrono::steady_clock::now();
                go.store(1);
                for (auto& x : th) x.join();
                const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                if (s < best) best = s;
            }
            printf("%-8s threads=%2d  %6.3f ms  %6.2f Gelem/s  %6.1f GB/s (r+w)\n",
                   mode == 0 ? "nt512" : mode == 1 ? "nt256" : "plain", t, best * 1e3, n / best * 1e-9,
                   12.0 * n / best * 1e-9);
        }
    }
    return 0;
}
