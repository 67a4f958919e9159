// CPU-only test of the host side of the drop-in path (csrc/hostpipe.cpp): the
// worker pool's asynchronous submit / join, the burst (polling) mode, and the
// widening / copying kernels on ragged, misaligned ranges, from several
// caller threads at once.  No CUDA: hostpipe.cpp has no device dependency.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "../../paper_1610_03525_b200/csrc/hostpipe.h"

static int failures = 0;
#define CHECK(c)                                                     \
    do {                                                             \
        if (!(c)) {                                                  \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);  \
            ++failures;                                              \
        }                                                            \
    } while (0)

static float val(size_t i, int salt) { return static_cast<float>(static_cast<int>((i * 2654435761u + salt) % 2000003u) - 1000001) * 0.125f; }

static void check_widen(size_t n, size_t off, bool stream, int salt) {
    std::vector<float> src(n + 8);
    std::vector<double> dst(n + off + 8, -7.0);
    for (size_t i = 0; i < n; ++i) src[i] = val(i, salt);
    tg::host::widen(src.data(), dst.data() + off, n, stream);
    bool ok = true;
    for (size_t i = 0; i < n; ++i) ok = ok && dst[off + i] == static_cast<double>(src[i]);
    for (size_t i = 0; i < off; ++i) ok = ok && dst[i] == -7.0;  // nothing before the range
    ok = ok && dst[off + n] == -7.0;                             // nothing after it
    CHECK(ok);
}

static void check_copy(size_t n, size_t off, bool stream, int salt) {
    std::vector<float> src(n + 8), dst(n + off + 8, -7.0f);
    for (size_t i = 0; i < n; ++i) src[i] = val(i, salt);
    tg::host::copy(src.data(), dst.data() + off, n, stream);
    bool ok = true;
    for (size_t i = 0; i < n; ++i) ok = ok && dst[off + i] == src[i];
    ok = ok && dst[off + n] == -7.0f;
    CHECK(ok);
}

int main() {
    std::printf("pool threads: %d\n", tg::host::threads());
    // ragged sizes, misaligned destinations, both store kinds
    for (size_t n : {size_t(0), size_t(1), size_t(15), size_t(16), size_t(17), size_t(1000), size_t(16384), size_t(100003),
                     size_t(1) << 20})
        for (size_t off : {size_t(0), size_t(1), size_t(3)})
            for (bool stream : {true, false}) {
                check_widen(n, off, stream, 1);
                check_copy(n, off, stream, 2);
            }
    // parallel_for covers every index exactly once
    {
        std::vector<std::atomic<int>> hits(1000);
        tg::host::parallel_for(1000, [&](int i) { hits[i].fetch_add(1); });
        bool ok = true;
        for (auto& h : hits) ok = ok && h.load() == 1;
        CHECK(ok);
    }
    // asynchronous jobs: a caller's submissions complete in order, with and
    // without a burst open, while other threads submit their own
    auto caller = [&](int salt, bool burst) {
        const size_t n = (size_t(1) << 18) + 37 * salt;
        std::vector<float> src(n);
        for (size_t i = 0; i < n; ++i) src[i] = val(i, salt);
        std::vector<std::vector<double>> out(6, std::vector<double>(n, 0.0));
        {
            std::unique_ptr<tg::host::Burst> b;
            if (burst) b.reset(new tg::host::Burst);
            tg::host::Pending pending;
            for (int k = 0; k < 6; ++k) {
                pending = tg::host::widen_async(src.data(), out[k].data(), n, (k & 1) != 0);
                // the job before the one just joined by this submission is complete
                if (k >= 1) {
                    bool ok = true;
                    for (size_t i = 0; i < n; i += 997) ok = ok && out[k - 1][i] == static_cast<double>(src[i]);
                    if (!ok) {
                        std::printf("FAIL job %d of caller %d not complete after the next submission\n", k - 1, salt);
                        ++failures;
                    }
                }
            }
            pending.wait();
        }
        bool ok = true;
        for (int k = 0; k < 6; ++k)
            for (size_t i = 0; i < n; ++i) ok = ok && out[k][i] == static_cast<double>(src[i]);
        if (!ok) {
            std::printf("FAIL caller %d\n", salt);
            ++failures;
        }
    };
    {
        std::vector<std::thread> th;
        for (int t = 0; t < 4; ++t) th.emplace_back(caller, t + 1, (t & 1) != 0);
        for (auto& t : th) t.join();
    }
    // a Pending that is never waited on joins in its destructor
    {
        std::vector<float> src(1 << 16, 2.5f);
        std::vector<double> dst(1 << 16, 0.0);
        { tg::host::Pending p = tg::host::widen_async(src.data(), dst.data(), src.size(), true); }
        bool ok = true;
        for (double d : dst) ok = ok && d == 2.5;
        CHECK(ok);
    }
    std::printf(failures ? "FAILED (%d)\n" : "ok\n", failures);
    return failures ? 1 : 0;
}
