// devattr.h — per-device one-shot kernel attribute opt-in.
//
// cudaFuncSetAttribute acts on the current device's context, so a process
// that drives several GPUs must opt in once per device (a process-wide bool
// would leave every device but the first without the >48 KiB shared-memory
// opt-in).  One bit per device ordinal, set atomically after a successful call.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

namespace tg {

class PerDeviceOnce {
   public:
    // Runs f() (returning cudaError_t) the first time it is called on the
    // current device; later calls on that device return cudaSuccess.
    template <class F>
    cudaError_t run(F&& f) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        const uint64_t bit = dev >= 0 && dev < 64 ? (uint64_t(1) << dev) : 0;
        if (bit && (bits_.load(std::memory_order_acquire) & bit)) return cudaSuccess;
        e = f();
        if (e == cudaSuccess && bit) bits_.fetch_or(bit, std::memory_order_acq_rel);
        return e;
    }

   private:
    std::atomic<uint64_t> bits_{0};
};

}  // namespace tg
