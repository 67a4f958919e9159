// hostpipe.cpp — persistent host worker pool + fp32->fp64 widening for the
// host-buffer entry points (tg_fbm_generate_f64_host / _f32_host).
//
// The reference's generate_into writes a caller-owned span<double>
// (fbm.hpp:541-628).  Moving doubles over PCIe doubles the bus bytes; the
// device computes fp32 anyway, so the path ships fp32 bands (4 B/sample) into
// pinned staging and the host widens them (exact) into the caller's buffer,
// overlapped with the next bands' generation and copies.
#include "hostpipe.h"

#include <emmintrin.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>

namespace tg {
namespace host {
namespace {

class Pool {
   public:
    explicit Pool(int n) : n_(n) {
        for (int i = 1; i < n_; ++i) std::thread([this] { loop(); }).detach();  // process lifetime
    }
    int size() const { return n_; }

    // Between begin_burst() and end_burst() idle workers poll for the next
    // job instead of sleeping on the condition variable: a futex wake of an
    // idle (halted) virtual CPU costs 50-130 us on the B200 host, once per
    // band and worker, which doubled the widening time of an 8 MiB band.
    void begin_burst() {
        {
            std::lock_guard<std::mutex> lk(m_);
            hot_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
    }
    void end_burst() { hot_.fetch_sub(1, std::memory_order_release); }

    // One submission.  A worker that wakes late holds an old job, whose index
    // counter is exhausted, so it can never run a stale function.
    struct Job {
        std::function<void(int)> fn;
        int total = 0;
        std::atomic<int> next{0}, done{0};
    };
    using Handle = std::shared_ptr<Job>;

    // Publishes f(0..n-1) to the workers and returns at once; the caller
    // joins it with finish().  The pool runs one job at a time: submitting
    // first completes (helping) whichever job is current, so a caller's jobs
    // finish in submission order.  Submissions from different threads
    // interleave job by job.
    Handle submit(int n, std::function<void(int)> f) {
        auto job = std::make_shared<Job>();
        job->fn = std::move(f);
        job->total = n;
        if (n_ <= 1 || n <= 1) {
            for (int i = 0; i < n; ++i) job->fn(i);
            job->done.store(n);
            return job;
        }
        std::lock_guard<std::mutex> submit(submit_);
        if (cur_) complete(*cur_);
        {
            std::lock_guard<std::mutex> lk(m_);
            job_ = job;
            gen_.fetch_add(1, std::memory_order_release);
        }
        cv_.notify_all();
        cur_ = job;
        return job;
    }
    void finish(const Handle& h) {
        if (h && h->done.load(std::memory_order_acquire) != h->total) complete(*h);
    }
    void run(int n, const std::function<void(int)>& f) { finish(submit(n, f)); }

   private:
    // help with the job's remaining pieces, then wait for the stragglers
    void complete(Job& j) {
        work(j);
        if (hot_.load(std::memory_order_acquire) > 0) {
            // mid-piece workers finish within microseconds: poll
            for (int spins = 0; j.done.load(std::memory_order_acquire) != j.total && spins < (1 << 22); ++spins)
                _mm_pause();
        }
        std::unique_lock<std::mutex> lk(m_);
        done_cv_.wait(lk, [&] { return j.done.load() == j.total; });
    }

    void work(Job& j) {
        int i, mine = 0;
        while ((i = j.next.fetch_add(1)) < j.total) {
            j.fn(i);
            ++mine;
        }
        if (mine && j.done.fetch_add(mine) + mine == j.total) {
            std::lock_guard<std::mutex> lk(m_);
            done_cv_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            // next job: poll while a burst is open, sleep otherwise
            while (gen_.load(std::memory_order_acquire) == seen) {
                if (hot_.load(std::memory_order_acquire) > 0) {
                    _mm_pause();
                    continue;
                }
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return gen_.load() != seen || hot_.load() > 0; });
            }
            std::shared_ptr<Job> j;
            {
                std::lock_guard<std::mutex> lk(m_);
                seen = gen_.load();
                j = job_;
            }
            if (j) work(*j);
        }
    }

    int n_;
    std::mutex submit_, m_;
    std::condition_variable cv_, done_cv_;
    std::shared_ptr<Job> job_;  // published to the workers (under m_)
    std::shared_ptr<Job> cur_;  // last submitted (under submit_)
    std::atomic<uint64_t> gen_{0};
    std::atomic<int> hot_{0};
};

Pool& pool() {
    static Pool* p = [] {
        // Streaming widen/copy: the workers are bound by the host's memory
        // system (reads of freshly DMA-written bands, streaming stores), so
        // more of them help up to a little over half the hardware threads
        // (16-thread B200 hosts, config 2 f64 drop-in: on the slower hosts of
        // the pool 6 workers 1.99 ms, 8: 1.87, 10: 1.80-1.83, 12 / 15: 1.83;
        // on the faster ones 1.34-1.39 ms from 6 workers up); the rest stay
        // free for the CUDA driver and the caller.  Shared among the ranks of
        // this node (LOCAL_WORLD_SIZE, set by torchrun), at most 10.
        int n = static_cast<int>(std::thread::hardware_concurrency());
        int ranks = 1;
        if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) ranks = std::max(1, std::atoi(e));
        n = std::min(std::max((n * 5 / 8) / ranks, 1), 10);
        if (const char* e = std::getenv("TG_HOST_THREADS")) n = std::max(1, std::atoi(e));
        return new Pool(n);
    }();
    return *p;
}

// AVX-512 form: 16 floats -> two 64-byte non-temporal stores of doubles (a
// whole cache line per store; the 16-byte SSE stores capped a core near
// 14 GB/s of read + write on the B200 host).
__attribute__((target("avx512f"))) void widen_avx512(const float* s, double* d, size_t n) {
    size_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 63); ++i) d[i] = s[i];
    // The source is a band the copy engine has just written: its lines come
    // from memory (or the IO agent's cache) at a latency the hardware
    // streamer, restarting at every 4 KiB page, does not cover while DMA is
    // still running; an L2 prefetch 16 KiB ahead does (B200 host, config 2,
    // 6 workers: 2.2 -> 2.0 ms; 10 workers 1.93 -> 1.80 ms).
    static const int pf = [] { const char* e = std::getenv("TG_HOST_PREFETCH"); return e ? std::atoi(e) : 16384; }();
    static const int hint = [] { const char* e = std::getenv("TG_HOST_PREFETCH_HINT"); return e ? std::atoi(e) : 0; }();
    for (; i + 16 <= n; i += 16) {
        if (pf) {
            if (hint == 1) _mm_prefetch(reinterpret_cast<const char*>(s + i) + pf, _MM_HINT_NTA);
            else if (hint == 2) _mm_prefetch(reinterpret_cast<const char*>(s + i) + pf, _MM_HINT_T0);
            else _mm_prefetch(reinterpret_cast<const char*>(s + i) + pf, _MM_HINT_T1);
        }
        const __m512 a = _mm512_loadu_ps(s + i);
        _mm512_stream_pd(d + i, _mm512_cvtps_pd(_mm512_castps512_ps256(a)));
        _mm512_stream_pd(d + i + 8, _mm512_cvtps_pd(_mm256_castpd_ps(_mm512_extractf64x4_pd(_mm512_castps_pd(a), 1))));
    }
    for (; i < n; ++i) d[i] = s[i];
    _mm_sfence();
}

// AVX2 form for hosts without AVX-512: 8 floats -> two 32-byte non-temporal
// stores, the same L2 prefetch ahead of the loads.
__attribute__((target("avx2"))) void widen_avx2(const float* s, double* d, size_t n) {
    size_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = s[i];
    static const int pf = [] { const char* e = std::getenv("TG_HOST_PREFETCH"); return e ? std::atoi(e) : 16384; }();
    for (; i + 8 <= n; i += 8) {
        if (pf && (i & 15) == 0) _mm_prefetch(reinterpret_cast<const char*>(s + i) + pf, _MM_HINT_T1);
        const __m256 a = _mm256_loadu_ps(s + i);
        _mm256_stream_pd(d + i, _mm256_cvtps_pd(_mm256_castps256_ps128(a)));
        _mm256_stream_pd(d + i + 4, _mm256_cvtps_pd(_mm256_extractf128_ps(a, 1)));
    }
    for (; i < n; ++i) d[i] = s[i];
    _mm_sfence();
}

bool have_avx2() {
    static const bool v = [] {
        if (const char* e = std::getenv("TG_HOST_AVX2")) return std::atoi(e) != 0;
        return __builtin_cpu_supports("avx2") != 0;
    }();
    return v;
}

bool have_avx512() {
    static const bool v = [] {
        if (const char* e = std::getenv("TG_HOST_AVX512")) return std::atoi(e) != 0;
        return __builtin_cpu_supports("avx512f") != 0;
    }();
    return v;
}

void widen_serial(const float* s, double* d, size_t n, bool stream) {
    if (stream && have_avx512()) return widen_avx512(s, d, n);
    if (stream && have_avx2()) return widen_avx2(s, d, n);
    size_t i = 0;
    if (stream) {
        for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 15); ++i) d[i] = s[i];
        for (; i + 8 <= n; i += 8) {
            const __m128 a = _mm_loadu_ps(s + i), b = _mm_loadu_ps(s + i + 4);
            _mm_stream_pd(d + i, _mm_cvtps_pd(a));
            _mm_stream_pd(d + i + 2, _mm_cvtps_pd(_mm_movehl_ps(a, a)));
            _mm_stream_pd(d + i + 4, _mm_cvtps_pd(b));
            _mm_stream_pd(d + i + 6, _mm_cvtps_pd(_mm_movehl_ps(b, b)));
        }
    }
    for (; i < n; ++i) d[i] = s[i];
    if (stream) _mm_sfence();
}

void copy_serial(const float* s, float* d, size_t n, bool stream) {
    size_t i = 0;
    if (stream) {
        for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 15); ++i) d[i] = s[i];
        for (; i + 8 <= n; i += 8) {
            _mm_stream_ps(d + i, _mm_loadu_ps(s + i));
            _mm_stream_ps(d + i + 4, _mm_loadu_ps(s + i + 4));
        }
        for (; i < n; ++i) d[i] = s[i];
        _mm_sfence();
        return;
    }
    std::memcpy(d, s, n * sizeof(float));
}

#ifndef TG_HOST_PIECES
#define TG_HOST_PIECES 4
#endif
constexpr size_t kPiecesPerWorker = TG_HOST_PIECES;

// n elements in pieces of >= 64 KiB of input on 64-element boundaries, a few
// pieces per worker (dynamic hand-out): a worker that starts late or shares
// its core does not hold the whole band back.  f(begin, count) is copied
// into the job.
template <class F>
Pool::Handle split(size_t n, F f) {
    const int t = pool().size();
    const size_t min_piece = 16384;
    int pieces = static_cast<int>(std::min<size_t>(static_cast<size_t>(t) * kPiecesPerWorker, (n + min_piece - 1) / min_piece));
    pieces = std::max(pieces, 1);
    size_t per = (n + pieces - 1) / pieces;
    per = (per + 63) / 64 * 64;
    return pool().submit(pieces, [f, per, n](int k) {
        const size_t b = static_cast<size_t>(k) * per;
        if (b >= n) return;
        f(b, std::min(per, n - b));
    });
}

}  // namespace

int threads() { return pool().size(); }

Burst::Burst() { pool().begin_burst(); }
Burst::~Burst() { pool().end_burst(); }

void parallel_for(int n, const std::function<void(int)>& f) { pool().run(n, f); }

struct Pending::Impl {
    std::shared_ptr<void> h;  // Pool::Handle
};
Pending::Pending() = default;
Pending::~Pending() { wait(); }
Pending::Pending(Pending&& o) noexcept : impl_(std::move(o.impl_)) {}
Pending& Pending::operator=(Pending&& o) noexcept {
    if (this != &o) {
        wait();
        impl_ = std::move(o.impl_);
    }
    return *this;
}
void Pending::wait() {
    if (impl_) pool().finish(std::static_pointer_cast<Pool::Job>(impl_->h));
    impl_.reset();
}

Pending widen_async(const float* src, double* dst, size_t n, bool stream) {
    Pending p;
    p.impl_.reset(new Pending::Impl{split(n, [=](size_t b, size_t m) { widen_serial(src + b, dst + b, m, stream); })});
    return p;
}

Pending copy_async(const float* src, float* dst, size_t n, bool stream) {
    Pending p;
    p.impl_.reset(new Pending::Impl{split(n, [=](size_t b, size_t m) { copy_serial(src + b, dst + b, m, stream); })});
    return p;
}

void widen(const float* src, double* dst, size_t n, bool stream) { widen_async(src, dst, n, stream).wait(); }

void copy(const float* src, float* dst, size_t n, bool stream) { copy_async(src, dst, n, stream).wait(); }

}  // namespace host
}  // namespace tg
