// select.h — the radix-select pass shared by tg_median_f32 (analysis.cu) and
// the multi-GPU terrain driver (terrain.cpp): one digit histogram per call,
// with a per-caller cache of candidate keys kept by the first pass.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace tg {

struct SelectCache {
    double rank_frac = 0.5;  // expected relative rank of the selected key in this window
    double delta = 0.005;    // kept window: sample ranks rank_frac +- delta (5 sigma of a 2^18 sample)
    uint32_t* keys = nullptr;
    uint64_t cap = 0;                 // kept-key capacity (kHistBlocks equal segments)
    unsigned long long* bcnt = nullptr;  // kept keys per block segment
    unsigned long long* dev_hist = nullptr;
    uint32_t wlo = 0, whi = 0;  // first-digit window of the kept keys
    bool valid = false;
};

// Digit histogram (shift, bits) of the keys matching prefix/mask in a
// width x rows window (pitch ld), to the host (1 << bits entries).
int select_hist(const float* map, int64_t width, int64_t rows, int64_t ld, uint32_t prefix, uint32_t mask, int shift,
                int bits, uint64_t* out_hist, SelectCache* cache, cudaStream_t s);
void select_cache_free(SelectCache* c, cudaStream_t s);

}  // namespace tg
