// fbm_params.h — launch parameters shared by the host planner (capi.cu) and
// the fused-octave kernels (fbm2d.cu, fbm3d.cu).  Passed by value as a
// __grid_constant__ kernel argument: no mutable __constant__ globals, so
// calls stay reentrant across streams and host threads (fbm.hpp:529-534).
#pragma once

#include <cstdint>

namespace tg {

// Per-octave sampling class, a function of the configuration only (never of
// the window), so any window reproduces the full-map pixels bit-for-bit
// (fbm.hpp:7-8).
enum OctaveClass : int32_t {
    kClsFast = 0,     // integer cell count dividing R: x = (r + 0.5)/ppc (fbm.hpp:160-166)
    kClsSubInt = 1,   // freq = k*R, k even, R = 2^n: u = (g+0.5)*k is an exact
                      // integer, so cx = cy = 0 and the cell value is h(ix, iy)
                      // exactly (render_general, fbm.hpp:468-489)
    kClsGeneral = 2,  // render_general: u = ((g + 0.5)/R)*freq in fp64 (fbm.hpp:468,474)
};

enum KernelKind : int32_t { kZgPaper = 0, kZgSeparable = 1, kGeneric = 2, kPerlin = 3 };

constexpr int kMaxOctaves = 32;
constexpr int kMaxBatch = 64;

struct OctDev {
    uint64_t oct_key;  // octave * K2 (lattice.hpp:47); seed term added per map
    double freq;       // f0 * ratio^i by repeated multiplication (fbm.hpp:155-158)
    float amp;         // h0 * p^i, rounded to fp32
    float w;           // generic gradient weight (fbm.hpp:62-64)
    float inv_ppc;     // 1 / ppc (fast)
    int32_t cls;       // OctaveClass
    int32_t ppc;       // pixels per cell (fast)
    int32_t shift;     // log2(ppc) when ppc is a power of two, else -1
    int64_t k;         // freq / R (sub-integer class)
};

struct FbmArgs {
    int64_t ox, oy;          // window origin, global pixels
    int64_t tile_x0, tile_y0;  // tile-grid origin (aligned to the tile size in global px)
    int64_t width, height;   // window size
    int64_t ld;              // output row pitch (elements)
    int64_t map_stride;      // elements between batched maps
    double R;                // resolution
    int32_t octaves;
    int32_t zero;            // ZeroSource
    int32_t n_maps;
    int32_t pad;
    uint64_t seed_key[kMaxBatch];  // seed * K1 per map (lattice.hpp:47)
    OctDev oct[kMaxOctaves];
};

struct Fbm3Args {
    int64_t ox, oy, oz;
    int64_t tile_x0, tile_y0, tile_z0;
    int64_t nx, ny, nz;
    double R;
    int32_t octaves;
    int32_t zero;
    uint64_t seed_key;
    OctDev oct[kMaxOctaves];
};

}  // namespace tg
