// fbm_params.h — launch parameters shared by the host planner (capi.cu) and
// the fused-octave kernels (fbm2d.cu, fbm3d.cu).  Passed by value as a
// __grid_constant__ kernel argument: no mutable __constant__ globals, so
// calls stay reentrant across streams and host threads (fbm.hpp:529-534).
#pragma once

#include <cstdint>

#include <vector_types.h>

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

enum KernelKind : int32_t { kZgPaper = 0, kZgSeparable = 1, kGeneric = 2, kPerlin = 3, kOpenSimplex = 4, kPerlinPerm = 5 };

constexpr int kMaxOctaves = 32;
constexpr int kMaxCellSlots = 10;  // kGBlkT octaves with per-tile cell parameters (8 cells each)
constexpr int kMaxBatch = 64;

// 2D tile geometry and per-CTA shared-memory budget (fbm2d.cu).
#ifndef TG_RPT
#define TG_RPT 8                   // pixel rows per thread (4 or 8)
#endif
constexpr int kRPT = TG_RPT;
constexpr int kTileW = 128;        // 32 lanes x 4 columns
constexpr int kTileH = 8 * kRPT;   // 8 warps x kRPT rows
constexpr int kGridCap = kRPT == 8 ? 12288 : 6656;  // lattice-corner floats per channel per CTA
constexpr int kTabSlots = 4;       // per-CTA sampling tables (general octaves)
constexpr int kLutLog2Max = 13;    // device row LUT covers ppc = 1 .. 8192
constexpr int kLutN4 = 2 << kLutLog2Max;  // float4 entries before the planar S / S-x copies

// Per-octave evaluation mode: a function of the configuration only (never of
// the window), so every window reproduces the full-map bits.
enum Mode : int32_t {
    kModeSubInt = 0,  // samples on lattice points: v = h(ix, iy), one hash per pixel
    kModePpc1 = 1,    // zg, 1 px per cell: v = 0.25*((h00+h10) + (h01+h11))
    kModeBlock2 = 2,  // zg, 2 px per cell: 2 x 4 cells per thread block
    kModeBlock = 3,   // power-of-two ppc >= 4: one cell per 4-column group
    kModeGrid = 4,    // shared corner grid + per-CTA sampling tables
    kModeDirect = 5,  // corners hashed per pixel (over the CTA budget)
};

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
    // static per-CTA plan, computed on the host (capi.cu plan_octaves)
    int32_t mode;      // Mode
    int32_t ncx, ncy;  // corner grid shape (exact when aligned, upper bound otherwise)
    int32_t pitch;     // grid row stride (floats, multiple of 4)
    int32_t goff;      // grid offset (floats per channel, multiple of 4)
    int32_t tslot;     // sampling-table slot (kModeGrid) or -1
    int32_t lut_off;   // offset of this ppc's row LUT (aligned modes) or -1
    int32_t pad;       // 3D: corner grid depth (ncz)
    int32_t cslot;     // kGBlkT: slot of the octave's per-tile cell parameters, else -1
    int32_t cdiv;      // 2D coarse grids: ceil(2^16 / ncx), so lane / ncx = (lane * cdiv) >> 16 for lane < 32
    // per-launch lattice-key constants (2D, build_args): the packed key of a
    // tile's first corner / lattice point is seed*K1 + key0 + bx*kx + by*ky
    //   lattice-point octaves: key0 = oct*K2 + (tile_x0*k + k/2)*K3 + (tile_y0*k + k/2)*K4,
    //                          kx = k*K3 (per pixel column), ky = k*K4 (per pixel row)
    //   aligned ppc <= 16:     key0 = oct*K2 + (tile_x0 >> s)*K3 + (tile_y0 >> s)*K4,
    //                          kx = (128 >> s)*K3 (per tile), ky = (64 >> s)*K4 (per tile)
    uint64_t key0, kx, ky;
    uint64_t kz;       // 3D lattice-point octaves: k*K5 per voxel slice (fbm3d_plan)
    double ratio;      // freq / R (OpenSimplex sample spacing), set by its launcher
};

// Octave lists built by the host planner (capi.cu): the kernel loops over
// mode-homogeneous lists instead of dispatching per octave.  Accumulation
// order is therefore group order — fixed per configuration, so results stay
// a pure function of (config, pixel).
enum OctGroup : int32_t {
    kGProCoarse = 0,  // aligned grids of <= 32 corners: one warp per octave
    kGProFine = 1,    // other grids / sampling tables
    kGBlk8 = 2,       // zg, power-of-two ppc >= 8
    kGBlk4 = 3,       // zg, ppc == 4
    kGBlk2 = 4,       // zg, ppc == 2
    kGPpc1 = 5,       // zg, ppc == 1
    kGSub = 6,        // lattice-point octaves
    kGGen = 7,        // everything else (Perlin/generic cells, general octaves)
    kGBlkT = 8,       // zg paper, power-of-two ppc >= 32: column / row terms built once per tile
    kNumGroups = 9
};

// Aligned power-of-two corner grids with ppc = 2^s <= 16, one slot per s
// (distinct octaves never share a ppc): the kernel visits the five slots with
// compile-time shapes and per-slot constants at fixed parameter offsets
// (no per-octave list walk).  goff < 0: slot unused.
struct FineDev {
    uint64_t key0, kx, ky;  // as OctDev::key0 / kx / ky
    int32_t goff, pitch;    // grid offset / row stride (floats)
    int32_t rot;            // starting warp (list position & 7)
    int32_t oct;            // octave index (corner data of Perlin / generic grids)
    int32_t blk;            // zg paper ppc 4 / 8 / 16: grid stored amplitude-scaled and the
                            // octave evaluated by its slot with compile-time shape (not listed)
    int32_t pad_;
};
constexpr int kFineSlots = 5;

// kGBlkT octave q (ppc = 2^shift >= 32): per-slot constants of the per-tile
// column / row terms, indexed by list position (cell parameters at slot q).
struct BlkTDev {
    const float2* sd;          // (S, S - x) row LUT of this ppc (row_lut's float2 plane at [ppc])
    int32_t shift, ncx1, mask;  // log2 ppc, cell columns per tile (ncx - 1), ppc - 1
    float inv;                  // 1 / ppc
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
    int32_t epilogue;        // 0 none, 1 marble, 2 wood (texture.hpp:50-72, fused into the store)
    int32_t tma;             // set by the launcher: tile store through the output tensor map
    float hoff;              // -sum of the octave amplitudes (map_height offset, lattice.cuh)
    float tex_freq2pi;       // 2*pi*pattern_frequency
    float tex_gain;          // turbulence gain
    // Row LUT of the smoothstep order in use: for ppc = 2^k, entries
    // lut[2^k - 1 + r] = (x, S(x), S(x) - x, x*S(x)) with x = (r + 0.5)/ppc
    // (kernels2d.hpp:214-239 at phase 0.5), computed in fp64 and rounded.
    const float4* lut;
    int32_t ngroup[kNumGroups];
    int8_t group[kNumGroups][kMaxOctaves];
    uint64_t seed_key[kMaxBatch];  // seed * K1 per map (lattice.hpp:47)
    OctDev oct[kMaxOctaves];
    FineDev fine[kFineSlots];  // kGProFine octaves taken out of the list (see FineDev)
    BlkTDev blkt[kMaxCellSlots];
    int32_t stage_pairs;       // the ppc-1 grid sits at offset 0 and no other grid below
                               // kTileW * kTileH floats: the tile store's staging only
                               // waits for the neighbouring warp (fbm2d.cu)
    int32_t pad_;
};

struct Fbm3Args {
    int64_t ox, oy, oz;
    int64_t tile_x0, tile_y0, tile_z0;
    int64_t nx, ny, nz;
    double R;
    int32_t octaves;
    int32_t zero;
    uint64_t seed_key;
    float hoff;         // -sum of the octave amplitudes (map_height offset, lattice.cuh)
    int32_t pad;
    const float4* lut;  // row LUT (see FbmArgs)
    OctDev oct[kMaxOctaves];
};

}  // namespace tg
