// hostpipe.h — host side of the drop-in generate_into(span<double>) path
// (fbm.hpp:630-634): a persistent worker pool that widens/copies fp32 bands
// from pinned staging into the caller's buffer while later bands are still
// being generated and copied over PCIe.
#pragma once
#include <cstddef>
#include <functional>
#include <memory>

namespace tg {
namespace host {

// Number of host threads the pool uses (TG_HOST_THREADS, default
// min(hardware_concurrency, 8): widening is host-memory-bound well before that); 1 means the caller's thread alone.
int threads();

// Runs f(i) for i in [0, n) on the pool and the calling thread; returns when
// all are done.  Calls from different threads are serialised.
void parallel_for(int n, const std::function<void(int)>& f);

// While a Burst is alive the pool's idle workers poll for the next job
// instead of sleeping (a sleeping worker's wake-up costs more than widening
// its share of a band); one per host-buffer call.
struct Burst {
    Burst();
    ~Burst();
    Burst(const Burst&) = delete;
    Burst& operator=(const Burst&) = delete;
};

// dst[i] = (double)src[i] / dst[i] = src[i], parallel over the pool;
// streaming stores when `stream` (no read-for-ownership of dst).
void widen(const float* src, double* dst, size_t n, bool stream);
void copy(const float* src, float* dst, size_t n, bool stream);

// The same, returning at once: the pool's workers start on the band while the
// caller queues the next band's device work; wait() (or the destructor, or
// the next submission) joins it, the caller helping with what is left.  A
// caller's submissions complete in order.
class Pending {
   public:
    Pending();
    ~Pending();
    Pending(Pending&&) noexcept;
    Pending& operator=(Pending&&) noexcept;
    void wait();

   private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
    friend Pending widen_async(const float*, double*, size_t, bool);
    friend Pending copy_async(const float*, float*, size_t, bool);
};
Pending widen_async(const float* src, double* dst, size_t n, bool stream);
Pending copy_async(const float* src, float* dst, size_t n, bool stream);

}  // namespace host
}  // namespace tg
