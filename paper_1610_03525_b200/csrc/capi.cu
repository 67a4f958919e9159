// capi.cu — C-ABI entry points (include/polyterrain_b200.h), validation and
// the per-call octave planner.
//
// Host logic restated from terrain/fbm.hpp:
//   FbmConfig::validate        fbm.hpp:71-88   -> tg_fbm_validate
//   detail::octave_spec        fbm.hpp:151-168 -> tg_fbm_octave_spec / plan()
//   window checks              fbm.hpp:546-558 -> tg_fbm_validate_window
//   generate_into_with_source  fbm.hpp:541-628 -> tg_fbm_generate_*_f32
// Errors map onto terrain/errors.hpp through the tg_status codes.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "hostpipe.h"

#include "../../include/polyterrain_b200.h"
#include "fbm_params.h"
#include "lattice.cuh"

namespace tg {
cudaError_t fbm2d_launch(int kind, int order, const FbmArgs& a, float* out, cudaStream_t st);
int fbm2d_tile_h();
cudaError_t fbm3d_launch(int order, const Fbm3Args& a, float* out, cudaStream_t st);
void fbm3d_tile(int* tx, int* ty, int* tz);
void fbm3d_plan(Fbm3Args* a, int zg_sep_only);
cudaError_t lattice_launch(int what, const tg_lattice_key* keys, uint64_t n, uint64_t lane,
                           void* out, cudaStream_t st);
cudaError_t widen_normalize_launch(const float* in, double* out, uint64_t n, double lo, double span, int norm,
                                   cudaStream_t st);
cudaError_t widen_launch(const float* in, double* out, uint64_t n, cudaStream_t st);
const float4* row_lut(int order);
}  // namespace tg

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(TG_EDEVICE, std::string(where) + ": " + cudaGetErrorString(e));
}

#define TG_CUDA(call)                                  \
    do {                                               \
        cudaError_t e_ = (call);                       \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

int64_t floor_div(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
    return q;
}

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

int order_of(const tg_fbm_config* c) {
    if (c->smoothstep) return c->smoothstep;
    return c->method == TG_METHOD_PERLIN5 || c->method == TG_METHOD_PERLIN_PERM ? 5 : 3;  // fbm.hpp:66-69
}

int kind_of(const tg_fbm_config* c) {
    switch (c->method) {
        case TG_METHOD_ZG_PAPER: return tg::kZgPaper;
        case TG_METHOD_ZG_SEPARABLE: return tg::kZgSeparable;
        case TG_METHOD_GENERIC: return tg::kGeneric;
        case TG_METHOD_OPENSIMPLEX: return tg::kOpenSimplex;
        case TG_METHOD_PERLIN_PERM: return tg::kPerlinPerm;
        default: return tg::kPerlin;
    }
}

void octave_spec(const tg_fbm_config* c, int octave, tg_octave_spec* os) {
    os->freq = static_cast<double>(c->base_frequency);
    os->amp = c->base_amplitude;
    for (int k = 0; k < octave; ++k) {  // repeated multiplication, fbm.hpp:155-158
        os->freq *= c->frequency_ratio;
        os->amp *= c->persistence;
    }
    os->fast = 0;
    os->cells = 0;
    os->ppc = 0;
    const double rounded = std::floor(os->freq);
    if (rounded == os->freq && rounded >= 1.0 && rounded <= static_cast<double>(c->resolution) &&
        c->resolution % static_cast<long long>(rounded) == 0) {
        os->fast = 1;
        os->cells = static_cast<int64_t>(rounded);
        os->ppc = static_cast<int32_t>(c->resolution / os->cells);
    }
}

// Fill the per-octave device plan for windows whose global coordinates stay
// within |g| <= gmax: sampling class, evaluation mode and the per-CTA
// shared-memory layout (fbm2d.cu).  Every decision depends on the
// configuration only, so all windows of one map evaluate each octave the same
// way (fbm.hpp:7-8).
void plan_octaves(const tg_fbm_config* c, int64_t gmax, tg::OctDev* out, bool plan_2d) {
    const double R = static_cast<double>(c->resolution);
    const double w = c->has_gradient_weight ? c->gradient_weight : c->base_amplitude / 100.0;
    const bool zg = c->method == TG_METHOD_ZG_PAPER || c->method == TG_METHOD_ZG_SEPARABLE;
    int goff = 0, slot = 0;
    // The aligned ppc-1 grid (the largest) goes first, at offset 0: the tile
    // store stages each warp's rows over it (fbm2d.cu, FbmArgs::stage_pairs).
    int o1 = -1;
    int64_t size1 = 0;
    if (plan_2d) {
        for (int o = 0; o < c->octaves && o1 < 0; ++o) {
            tg_octave_spec os;
            octave_spec(c, o, &os);
            if (os.fast && os.ppc == 1) {
                o1 = o;
                size1 = ((tg::kTileW + 1 + 3) & ~3) * static_cast<int64_t>(tg::kTileH + 1);
                if (size1 > tg::kGridCap) o1 = -1;
            }
        }
        if (o1 >= 0) goff = static_cast<int>(size1);
    }
    for (int o = 0; o < c->octaves; ++o) {
        tg_octave_spec os;
        octave_spec(c, o, &os);
        tg::OctDev& d = out[o];
        std::memset(&d, 0, sizeof(d));
        d.oct_key = static_cast<uint64_t>(static_cast<uint32_t>(o)) * tg::kOctMul;
        d.freq = os.freq;
        // ZeroSource (fbm.hpp:125-133): every corner datum 0 <=> amp = w = 0
        d.amp = c->zero_lattice ? 0.0f : static_cast<float>(os.amp);
        d.w = c->zero_lattice ? 0.0f : static_cast<float>(w);
        d.shift = -1;
        d.tslot = -1;
        d.lut_off = -1;
        if (os.fast) {
            d.cls = tg::kClsFast;
            d.ppc = os.ppc;
            d.inv_ppc = 1.0f / static_cast<float>(os.ppc);
            if (is_pow2(os.ppc)) {
                int s = 0;
                while ((1LL << s) < os.ppc) ++s;
                d.shift = s;
            }
        } else {
            d.cls = tg::kClsGeneral;
            // Exact lattice-point sampling: R = 2^n and freq = k*R with k even make
            // ((g + 0.5)/R)*freq = g*k + k/2 exactly in fp64 (no rounding while
            // |g*k| < 2^52), so render_general sees cx = cy = 0 (fbm.hpp:468-489).
            if (is_pow2(c->resolution)) {
                const double kd = os.freq / R;
                if (kd >= 2.0 && kd < 9.0e15 && std::floor(kd) == kd && kd * R == os.freq) {
                    const int64_t k = static_cast<int64_t>(kd);
                    const double bound = (static_cast<double>(gmax) + 1.0) * kd + kd;
                    if ((k & 1) == 0 && bound < 4.0e15) {
                        d.cls = tg::kClsSubInt;
                        d.k = k;
                    }
                }
            }
        }
        if (!plan_2d) continue;
        if (d.cls == tg::kClsSubInt) {
            d.mode = tg::kModeSubInt;
            continue;
        }
        int64_t ncx, ncy;
        int mode;
        if (d.cls == tg::kClsFast && d.shift >= 0 && d.shift <= tg::kLutLog2Max) {
            d.lut_off = (1 << d.shift) - 1;
            ncx = std::max<int64_t>(tg::kTileW >> d.shift, 1) + 1;
            ncy = std::max<int64_t>(tg::kTileH >> d.shift, 1) + 1;
            const bool perlin = c->method == TG_METHOD_PERLIN3 || c->method == TG_METHOD_PERLIN5;
            if ((zg || perlin) && d.ppc == 1) mode = tg::kModePpc1;
            else if (d.ppc == 2) mode = tg::kModeBlock2;
            else if (d.ppc >= 4) mode = tg::kModeBlock;
            else mode = tg::kModeGrid;
        } else if (d.cls == tg::kClsFast) {
            // tile spans at most floor(127/ppc) + 2 cells
            ncx = (tg::kTileW - 1) / d.ppc + 3;
            ncy = (tg::kTileH - 1) / d.ppc + 3;
            mode = tg::kModeGrid;
        } else {
            const double span = d.freq / R;
            const double bx = std::ceil((tg::kTileW - 1) * span) + 3.0;
            const double by = std::ceil((tg::kTileH - 1) * span) + 3.0;
            ncx = bx > 1.0e6 ? 1000000 : static_cast<int64_t>(bx);
            ncy = by > 1.0e6 ? 1000000 : static_cast<int64_t>(by);
            mode = tg::kModeGrid;
        }
        const int64_t pitch = (ncx + 3) & ~int64_t(3);
        const int64_t size = pitch * ncy;
        const bool needs_tab = mode == tg::kModeGrid;
        if (o == o1 && ncx * ncy <= tg::kGridCap && size == size1 && !(needs_tab && slot >= tg::kTabSlots)) {
            d.mode = mode;  // the reserved slot at offset 0
            d.ncx = static_cast<int32_t>(ncx);
            d.ncy = static_cast<int32_t>(ncy);
            d.pitch = static_cast<int32_t>(pitch);
            d.goff = 0;
            d.cdiv = static_cast<int32_t>((65536 + ncx - 1) / ncx);
            if (needs_tab) d.tslot = slot++;
            continue;
        }
        if (ncx * ncy > tg::kGridCap || goff + size > tg::kGridCap || (needs_tab && slot >= tg::kTabSlots)) {
            d.mode = tg::kModeDirect;
            continue;
        }
        d.mode = mode;
        d.ncx = static_cast<int32_t>(ncx);
        d.ncy = static_cast<int32_t>(ncy);
        d.pitch = static_cast<int32_t>(pitch);
        d.goff = goff;
        d.cdiv = static_cast<int32_t>((65536 + ncx - 1) / ncx);
        goff += static_cast<int>(size);
        if (needs_tab) d.tslot = slot++;
    }
}

int validate_cfg(const tg_fbm_config* c) {
    if (!c) return fail(TG_EVALIDATION, "fbm config: null");
    if (c->octaves < 1 || c->octaves > TG_MAX_OCTAVES)
        return fail(TG_EVALIDATION, "fbm config: octaves must be in [1, 32]");
    if (c->resolution < 1 || c->resolution > TG_MAX_RESOLUTION)
        return fail(TG_EVALIDATION, "fbm config: resolution must be in [1, 4194304]");
    if (c->base_frequency < 1 || c->base_frequency > TG_MAX_RESOLUTION)
        return fail(TG_EVALIDATION, "fbm config: base_frequency must be in [1, 4194304]");
    if (!(c->frequency_ratio > 1.0) || !std::isfinite(c->frequency_ratio))
        return fail(TG_EVALIDATION, "fbm config: frequency_ratio must be > 1");
    if (!(c->persistence > 0.0 && c->persistence <= 1.0))
        return fail(TG_EVALIDATION, "fbm config: persistence must lie in (0, 1]");
    if (!(c->base_amplitude > 0.0) || !std::isfinite(c->base_amplitude))
        return fail(TG_EVALIDATION, "fbm config: base_amplitude must be positive");
    if (c->has_gradient_weight && (!(c->gradient_weight >= 0.0) || !std::isfinite(c->gradient_weight)))
        return fail(TG_EVALIDATION, "fbm config: gradient_weight must be non-negative");
    if (c->threads < 0 || c->threads > 256)
        return fail(TG_EVALIDATION, "fbm config: threads must be in [0, 256]");
    if (c->method < TG_METHOD_ZG_PAPER || c->method > TG_METHOD_PERLIN_PERM)
        return fail(TG_EVALIDATION, "fbm config: unknown method");
    if (c->smoothstep != 0 && c->smoothstep != 3 && c->smoothstep != 5)
        return fail(TG_EVALIDATION, "fbm config: smoothstep must be 0, 3 or 5");
    return TG_OK;
}

int validate_window(const tg_fbm_config* c, int64_t ox, int64_t oy, int64_t width,
                    int64_t height, bool require_alignment = true) {
    if (width < 1 || width > TG_MAX_EXTENT || height < 1 || height > TG_MAX_EXTENT)
        return fail(TG_EVALIDATION, "generate: extent must be in [1, 131072]");
    const int64_t origin[2] = {ox, oy};
    for (const int64_t o : origin) {  // fbm.hpp:551-558
        if (o < -(1LL << 40) || o > (1LL << 40))
            return fail(TG_EVALIDATION, "generate: origin out of supported range");
        const int64_t prod = o * c->base_frequency;
        if (require_alignment && ((prod % c->resolution) + c->resolution) % c->resolution != 0)
            return fail(TG_EVALIDATION, "generate: origin must be aligned to octave-0 cell boundaries");
    }
    return TG_OK;
}

// Scratch buffers come from the device's default stream-ordered pool; keep
// freed blocks cached in the pool (default release threshold 0 would unmap
// them at every synchronisation and remap on the next call).
void keep_pool(int dev) {
    static std::atomic<uint64_t> done{0};
    if (dev < 0 || dev >= 64 || (done.load() >> dev) & 1ULL) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
    done.fetch_or(1ULL << dev);
}

int device_ready() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(TG_EDEVICE, "no CUDA device: the B200 path has no CPU fallback");
    }
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) keep_pool(dev);
    return TG_OK;
}

// -sum of the octave amplitudes: the kernels' map_height values carry +1 per
// corner height (lattice.cuh), and each cell blends its corners affinely, so
// every octave's contribution is off by exactly +amp (removed once per pixel).
static float amp_offset(const tg::OctDev* oct, int n) {
    double s = 0.0;
    for (int o = 0; o < n; ++o) s += static_cast<double>(oct[o].amp);
    return static_cast<float>(-s);
}

int build_args(const tg_fbm_config* c, int64_t ox, int64_t oy, int64_t width, int64_t height,
               int64_t ld, tg::FbmArgs* a) {
    std::memset(a, 0, sizeof(*a));
    a->ox = ox;
    a->oy = oy;
    a->width = width;
    a->height = height;
    a->ld = ld;
    a->map_stride = ld * height;
    a->tile_x0 = floor_div(ox, 128) * 128;
    a->tile_y0 = floor_div(oy, tg::fbm2d_tile_h()) * tg::fbm2d_tile_h();
    a->R = static_cast<double>(c->resolution);
    a->octaves = c->octaves;
    a->zero = c->zero_lattice ? 1 : 0;
    a->n_maps = 1;
    a->seed_key[0] = c->seed * tg::kSeedMul + tg::kMapKeyBias;
    int64_t gmax = 0;
    const int64_t cand[4] = {ox - 256, ox + width + 256, oy - 256, oy + height + 256};
    for (int64_t v : cand) gmax = std::max<int64_t>(gmax, v < 0 ? -v : v);
    plan_octaves(c, gmax, a->oct, true);
    a->hoff = amp_offset(a->oct, c->octaves);
    for (int o = 0; o < c->octaves; ++o) {  // per-launch key constants (fbm_params.h OctDev::key0)
        tg::OctDev& d = a->oct[o];
        const uint64_t tx = static_cast<uint64_t>(a->tile_x0), ty = static_cast<uint64_t>(a->tile_y0);
        if (d.mode == tg::kModeSubInt) {
            const uint64_t k = static_cast<uint64_t>(d.k), h = k >> 1;
            d.kx = k * tg::kIxMul;
            d.ky = k * tg::kIyMul;
            d.key0 = d.oct_key + (tx * k + h) * tg::kIxMul + (ty * k + h) * tg::kIyMul;
        } else if (d.lut_off >= 0 && d.shift >= 0 && d.shift <= 4) {
            const int sh = d.shift;
            d.kx = static_cast<uint64_t>(tg::kTileW >> sh) * tg::kIxMul;
            d.ky = static_cast<uint64_t>(tg::fbm2d_tile_h() >> sh) * tg::kIyMul;
            d.key0 = d.oct_key + static_cast<uint64_t>(a->tile_x0 >> sh) * tg::kIxMul +
                     static_cast<uint64_t>(a->tile_y0 >> sh) * tg::kIyMul;
        }
    }
    // mode-homogeneous octave lists (fbm_params.h OctGroup)
    const bool zg = c->method == TG_METHOD_ZG_PAPER || c->method == TG_METHOD_ZG_SEPARABLE;
    const bool paper = c->method == TG_METHOD_ZG_PAPER;
    for (int o = 0; o < c->octaves; ++o) a->oct[o].cslot = -1;
    for (int o = 0; o < c->octaves; ++o) {
        const tg::OctDev& d = a->oct[o];
        auto push = [&](int g) { a->group[g][a->ngroup[g]++] = static_cast<int8_t>(o); };
        const bool has_grid = d.mode == tg::kModePpc1 || d.mode == tg::kModeBlock2 || d.mode == tg::kModeBlock ||
                              d.mode == tg::kModeGrid;
        if (has_grid) push(d.lut_off >= 0 && d.mode != tg::kModeGrid && d.ncx * d.ncy <= 32 ? tg::kGProCoarse
                                                                                            : tg::kGProFine);
        if (d.mode == tg::kModeSubInt) push(tg::kGSub);
        else if (zg && d.mode == tg::kModeBlock && d.shift >= 3) {
            // ppc >= 32 on a 128 x 64 tile: at most 4 x 2 cells, 15 corners
            const bool tile_terms = paper && d.shift >= 5 && tg::fbm2d_tile_h() == 64 && d.ncx * d.ncy <= 32 &&
                                    a->ngroup[tg::kGBlkT] < tg::kMaxCellSlots;
            if (tile_terms) {
                const int q = a->ngroup[tg::kGBlkT];
                a->oct[o].cslot = q;
                a->blkt[q] = {nullptr, d.shift, d.ncx - 1, d.ppc - 1, d.inv_ppc};  // sd: below
            }
            push(tile_terms ? tg::kGBlkT : tg::kGBlk8);
        }
        else if (zg && d.mode == tg::kModeBlock && d.shift == 2) push(tg::kGBlk4);
        else if (d.mode == tg::kModeBlock2) push(tg::kGBlk2);
        else if (d.mode == tg::kModePpc1) push(tg::kGPpc1);
        else push(tg::kGGen);
    }
    // aligned ppc <= 16 grids leave the kGProFine list for the per-ppc slots
    for (int sl = 0; sl < tg::kFineSlots; ++sl) a->fine[sl].goff = -1;
    {
        int n = 0, nspec = 0;
        for (int q = 0; q < a->ngroup[tg::kGProFine]; ++q) {
            const int o = a->group[tg::kGProFine][q];
            const tg::OctDev& d = a->oct[o];
            const int sh = d.shift;
            if (c->method != TG_METHOD_GENERIC && d.mode != tg::kModeGrid && d.lut_off >= 0 && sh >= 0 && sh < tg::kFineSlots &&
                a->fine[sh].goff < 0) {  // (grid-mode octaves also build sampling tables)
                tg::FineDev& f = a->fine[sh];
                f.key0 = d.key0;
                f.kx = d.kx;
                f.ky = d.ky;
                f.goff = d.goff;
                f.pitch = d.pitch;
                f.rot = (nspec++) & 7;
                f.oct = o;
            } else {
                a->group[tg::kGProFine][n++] = static_cast<int8_t>(o);
            }
        }
        a->ngroup[tg::kGProFine] = n;
    }
    // zg paper ppc 4 / 8 / 16 block octaves: evaluated by their fine slot with
    // compile-time shapes (fbm2d.cu blk_slot) instead of the kGBlk4 / kGBlk8 lists
    if (paper && tg::fbm2d_tile_h() == 64) {
        for (int sh = 2; sh <= 4; ++sh) {
            tg::FineDev& f = a->fine[sh];
            if (f.goff < 0) continue;
            const int g = sh == 2 ? tg::kGBlk4 : tg::kGBlk8;
            int n = 0;
            for (int q = 0; q < a->ngroup[g]; ++q) {
                if (a->group[g][q] == f.oct) f.blk = 1;
                else a->group[g][n++] = a->group[g][q];
            }
            a->ngroup[g] = n;
        }
    }
    // tile-store staging over the ppc-1 grid (plan_octaves puts it at offset 0)
    a->stage_pairs = 0;
    if (tg::fbm2d_tile_h() == 64) {
        int below = 0, p1 = 0;
        for (int o = 0; o < c->octaves; ++o) {
            const tg::OctDev& d = a->oct[o];
            const bool grid = d.mode == tg::kModePpc1 || d.mode == tg::kModeBlock2 || d.mode == tg::kModeBlock ||
                              d.mode == tg::kModeGrid;
            if (!grid) continue;
            if (d.goff == 0 && d.lut_off == 0 && d.pitch >= tg::kTileW + 1 && d.pitch <= tg::kTileW + 4) p1 = 1;
            else if (d.goff < tg::kTileW * 64) below = 1;
        }
        a->stage_pairs = p1 && !below;
    }
    a->lut = tg::row_lut(order_of(c));
    if (!a->lut) return fail(TG_EDEVICE, "row LUT allocation failed");
    for (int q = 0; q < a->ngroup[tg::kGBlkT]; ++q)  // (S, S - x) plane of row_lut at [ppc]
        a->blkt[q].sd = reinterpret_cast<const float2*>(a->lut + tg::kLutN4 + tg::kLutN4 / 2) + (a->blkt[q].mask + 1);
    return TG_OK;
}

}  // namespace

extern "C" {

int tg_abi_version(void) { return TG_ABI_VERSION; }

const char* tg_last_error(void) { return g_err.c_str(); }

int tg_fbm_validate(const tg_fbm_config* cfg) { return validate_cfg(cfg); }

int tg_fbm_octave_spec(const tg_fbm_config* cfg, int32_t octave, tg_octave_spec* out) {
    if (int st = validate_cfg(cfg)) return st;
    if (!out || octave < 0 || octave >= cfg->octaves)
        return fail(TG_EVALIDATION, "octave_spec: octave out of range");
    octave_spec(cfg, octave, out);
    return TG_OK;
}

int tg_fbm_validate_window(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t width,
                           int64_t height) {
    if (int st = validate_cfg(cfg)) return st;
    return validate_window(cfg, ox, oy, width, height);
}

int tg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int tg_fbm_generate_rect_f32(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t width,
                             int64_t height, float* dev_out, int64_t ld, void* stream) {
    if (int st = validate_cfg(cfg)) return st;
    // The chunk/band primitive accepts any origin: every value is a pure
    // function of (cfg, global pixel), so halo rows can be regenerated.
    if (int st = validate_window(cfg, ox, oy, width, height, false)) return st;
    if (!dev_out) return fail(TG_EVALIDATION, "generate: null output");
    if (ld < width) return fail(TG_EVALIDATION, "generate: row pitch smaller than width");
    if (int st = device_ready()) return st;
    tg::FbmArgs a;
    if (int st = build_args(cfg, ox, oy, width, height, ld, &a)) return st;
    TG_CUDA(tg::fbm2d_launch(kind_of(cfg), order_of(cfg), a, dev_out,
                             static_cast<cudaStream_t>(stream)));
    return TG_OK;
}

int tg_fbm_generate_f32(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t extent,
                        float* dev_out, uint64_t n_out, void* stream) {
    if (int st = validate_cfg(cfg)) return st;
    if (extent < 1 || extent > TG_MAX_EXTENT)
        return fail(TG_EVALIDATION, "generate: extent must be in [1, 131072]");
    if (n_out != static_cast<uint64_t>(extent) * static_cast<uint64_t>(extent))
        return fail(TG_EVALIDATION, "generate: output buffer size mismatch");  // fbm.hpp:549
    if (int st = validate_window(cfg, ox, oy, extent, extent)) return st;  // fbm.hpp:551-558
    return tg_fbm_generate_rect_f32(cfg, ox, oy, extent, extent, dev_out, extent, stream);
}

// generate_region / generate_heightmap with cfg.normalize (fbm.hpp:638-685)
// on the device: the map generated in fp32, its min / max reduced on the
// device (exact: the extremes of the fp32 samples are those of the widened
// doubles), then widened and normalised in fp64 band by band on the way to
// the host — the same doubles as normalize_map on the host-widened map.
int tg_fbm_generate_normalized_f64_host(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int32_t extent,
                                        double* host_out, uint64_t n_out, double* out_min, double* out_max,
                                        int32_t* constant_source) {
    if (int st = validate_cfg(cfg)) return st;
    if (!host_out || !out_min || !out_max || !constant_source) return fail(TG_EVALIDATION, "generate: null output");
    if (extent < 1 || extent > TG_MAX_EXTENT) return fail(TG_EVALIDATION, "generate: extent must be in [1, 131072]");
    const uint64_t n = static_cast<uint64_t>(extent) * static_cast<uint64_t>(extent);
    if (n_out != n) return fail(TG_EVALIDATION, "generate: output buffer size mismatch");
    if (int st = validate_window(cfg, ox, oy, extent, extent)) return st;
    if (int st = device_ready()) return st;
    cudaStream_t s = nullptr;
    TG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    float* map = nullptr;
    double* band = nullptr;
    const uint64_t rows = std::max<uint64_t>(1, (uint64_t(8) << 20) / static_cast<uint64_t>(extent));
    int st = TG_OK;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&map), sizeof(float) * n, s);
    if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&band), sizeof(double) * rows * extent, s);
    if (e != cudaSuccess) st = cuda_fail(e, "normalized generate alloc");
    if (st == TG_OK) st = tg_fbm_generate_f32(cfg, ox, oy, extent, map, n, s);
    double lo = 0, hi = 0;
    if (st == TG_OK) st = tg_minmax_f32(map, n, &lo, &hi, s);
    const int norm = lo != hi;
    for (uint64_t r0 = 0; st == TG_OK && r0 < static_cast<uint64_t>(extent); r0 += rows) {
        const uint64_t m = std::min<uint64_t>(rows, extent - r0) * extent;
        e = tg::widen_normalize_launch(map + r0 * extent, band, m, lo, hi - lo, norm, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(host_out + r0 * extent, band, sizeof(double) * m,
                                                  cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) st = cuda_fail(e, "normalized generate");
    }
    if (map) cudaFreeAsync(map, s);
    if (band) cudaFreeAsync(band, s);
    e = cudaStreamSynchronize(s);
    if (st == TG_OK && e != cudaSuccess) st = cuda_fail(e, "normalized generate sync");
    cudaStreamDestroy(s);
    if (st != TG_OK) return st;
    *out_min = lo;
    *out_max = hi;
    *constant_source = norm ? 0 : 1;
    return TG_OK;
}

// Per-octave device time (generate_into's octave_seconds, fbm.hpp:564,
// 624-626): the fused kernel renders every octave in one pass, so octave k's
// time is measured as the increment T(k+1) - T(k) between diagnostic launches
// of the octave prefixes 0..k over the same window (CUDA events, median of 3
// after a warm-up; clamped at 0).  Costs about 4 (N + 1) extra launches.
int tg_fbm_octave_times(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int32_t extent, double* seconds_out,
                        void* stream) {
    if (int st = validate_cfg(cfg)) return st;
    if (!seconds_out) return fail(TG_EVALIDATION, "octave_times: null output");
    if (extent < 1 || extent > TG_MAX_EXTENT) return fail(TG_EVALIDATION, "generate: extent must be in [1, 131072]");
    if (int st = validate_window(cfg, ox, oy, extent, extent)) return st;
    if (int st = device_ready()) return st;
    // The times depend on the configuration's shape, not on the seed or the
    // (aligned) origin: measured once per shape and device, then reused.
    static std::mutex mu;
    static std::map<std::string, std::vector<double>> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    char keyb[256];
    snprintf(keyb, sizeof(keyb), "%d|%d|%d|%d|%lld|%d|%.17g|%.17g|%.17g|%d|%lld", dev, cfg->method, cfg->smoothstep,
             cfg->octaves, static_cast<long long>(cfg->resolution), cfg->base_frequency, cfg->frequency_ratio,
             cfg->persistence, cfg->base_amplitude, cfg->zero_lattice, static_cast<long long>(extent));
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(keyb);
        if (it != cache.end()) {
            std::copy(it->second.begin(), it->second.end(), seconds_out);
            return TG_OK;
        }
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    float* buf = nullptr;
    TG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), sizeof(float) * extent * extent, s));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    std::vector<double> prefix_ms(static_cast<size_t>(cfg->octaves) + 1, 0.0);
    int st = TG_OK;
    for (int k = 1; k <= cfg->octaves && st == TG_OK; ++k) {
        tg_fbm_config c = *cfg;
        c.octaves = k;  // octaves 0..k-1: the same specs (repeated multiplication from octave 0)
        double ms[3];
        for (int r = -1; r < 3 && st == TG_OK; ++r) {
            cudaEventRecord(e0, s);
            st = tg_fbm_generate_rect_f32(&c, ox, oy, extent, extent, buf, extent, s);
            cudaEventRecord(e1, s);
            if (st == TG_OK && cudaEventSynchronize(e1) != cudaSuccess) st = fail(TG_EDEVICE, "octave_times sync");
            float f = 0.f;
            cudaEventElapsedTime(&f, e0, e1);
            if (r >= 0) ms[r] = f;
        }
        if (st == TG_OK) prefix_ms[k] = std::max(std::min(ms[0], ms[1]), std::min(std::max(ms[0], ms[1]), ms[2]));
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFreeAsync(buf, s);
    if (st != TG_OK) return st;
    std::vector<double> t(static_cast<size_t>(cfg->octaves));
    for (int k = 0; k < cfg->octaves; ++k) t[k] = std::max(0.0, prefix_ms[k + 1] - prefix_ms[k]) * 1e-3;
    std::copy(t.begin(), t.end(), seconds_out);
    std::lock_guard<std::mutex> lock(mu);
    cache[keyb] = std::move(t);
    return TG_OK;
}

// texture::render (texture.hpp:50-72): marble / wood fused into the fBm
// store; cloud = the noise normalised to [-1, 1] (device min/max + rescale).
int tg_texture_generate_f32(const tg_fbm_config* cfg, int32_t kind, double gain, double pattern_frequency,
                            float* dev_out, void* stream) {
    if (int st = validate_cfg(cfg)) return st;
    if (kind < 0 || kind > 2) return fail(TG_EVALIDATION, "texture: unknown kind");
    if (!(pattern_frequency > 0.0) || !std::isfinite(pattern_frequency))
        return fail(TG_EVALIDATION, "TextureSpec: pattern frequency must be positive");
    if (!std::isfinite(gain)) return fail(TG_EVALIDATION, "TextureSpec: non-finite gain");
    if (!dev_out) return fail(TG_EVALIDATION, "texture: null output");
    if (cfg->resolution > TG_MAX_EXTENT) return fail(TG_EVALIDATION, "texture: resolution above the extent cap");
    if (int st = device_ready()) return st;
    const int64_t R = cfg->resolution;
    tg::FbmArgs a;
    if (int st = build_args(cfg, 0, 0, R, R, R, &a)) return st;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (kind != 2) {  // TG texture kinds: 0 marble, 1 wood, 2 cloud
        a.epilogue = kind == 0 ? 1 : 2;
        a.tex_freq2pi = static_cast<float>(2.0 * 3.14159265358979323846 * pattern_frequency);
        a.tex_gain = static_cast<float>(gain);
    }
    TG_CUDA(tg::fbm2d_launch(kind_of(cfg), order_of(cfg), a, dev_out, s));
    if (kind == 2) {
        double lo = 0, hi = 0;
        if (int st = tg_minmax_f32(dev_out, static_cast<uint64_t>(R * R), &lo, &hi, stream)) return st;
        if (hi > lo)
            if (int st = tg_rescale_f32(dev_out, static_cast<uint64_t>(R * R), lo, hi, stream)) return st;
    }
    return TG_OK;
}

int tg_fbm_generate_batch_f32(const tg_fbm_config* cfg, const uint64_t* seeds, int32_t n_seeds,
                              int64_t ox, int64_t oy, int64_t width, int64_t height,
                              float* dev_out, void* stream) {
    if (int st = validate_cfg(cfg)) return st;
    if (int st = validate_window(cfg, ox, oy, width, height)) return st;
    if (!seeds || n_seeds < 1 || !dev_out) return fail(TG_EVALIDATION, "batch: bad arguments");
    if (int st = device_ready()) return st;
    tg::FbmArgs a;
    if (int st = build_args(cfg, ox, oy, width, height, width, &a)) return st;
    for (int32_t b0 = 0; b0 < n_seeds; b0 += tg::kMaxBatch) {
        const int nb = std::min<int32_t>(tg::kMaxBatch, n_seeds - b0);
        a.n_maps = nb;
        for (int i = 0; i < nb; ++i) a.seed_key[i] = seeds[b0 + i] * tg::kSeedMul + tg::kMapKeyBias;
        TG_CUDA(tg::fbm2d_launch(kind_of(cfg), order_of(cfg), a,
                                 dev_out + static_cast<int64_t>(b0) * width * height,
                                 static_cast<cudaStream_t>(stream)));
    }
    return TG_OK;
}

// Host-buffer forms: the drop-in for generate_into(cfg, origin, extent,
// std::span<double>) (fbm.hpp:630-634).  Device work is fp32; the result is
// produced in row bands so the next band's generation overlaps the previous
// band's device->host copy.
// Host-buffer generation (the drop-in generate_into(span<double>),
// fbm.hpp:630-634).  Bands of whole tile rows are generated on two streams
// and copied over PCIe as fp32 into a ring of pinned staging slots; the host
// pool widens (exact) / copies each landed band into the caller's buffer while
// later bands are in flight, so the bus carries 4 B/sample, not 8.  A pinned
// fp32 destination takes the copy directly.  Staging is cached per device.
namespace {

constexpr int kSlots = 16;
#ifndef TG_BAND_LOG2
#define TG_BAND_LOG2 20
#endif
// 4 MiB of fp32 per full band in a ring of 8 slots.  Config 2, f64 drop-in,
// workers joined asynchronously: 2 MiB bands 1.89-2.03 ms in a 5-slot ring but
// 1.40-1.45 in 16 slots (a slot rewritten by DMA while its lines still sit in
// the workers' caches slows both sides), 4 MiB 1.38-1.45 in 8 slots, 8 MiB
// 1.44-1.54 on a quiet host and 1.96 where the host is the slower side.


struct HostStage {
    int dev = -1;
    size_t cap = 0;  // elements per band slot
    int nslots = 0;  // pinned slots allocated
    cudaStream_t st[2] = {nullptr, nullptr};
    float* dbuf[2] = {nullptr, nullptr};
    double* dwide[2] = {nullptr, nullptr};  // device-widened bands (pinned f64 destinations)
    float* pin[kSlots] = {};
    cudaEvent_t ev[kSlots] = {};
};

std::mutex g_stage_m;
std::vector<HostStage*> g_stage_free;

void stage_free_buffers(HostStage* s) {
    for (auto& d : s->dbuf) if (d) cudaFree(d), d = nullptr;
    for (auto& d : s->dwide) if (d) cudaFree(d), d = nullptr;
    for (auto& p : s->pin) if (p) cudaFreeHost(p), p = nullptr;
    s->cap = 0;
    s->nslots = 0;
}

HostStage* stage_acquire(int dev, size_t cap, int nslots) {
    HostStage* s = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_stage_m);
        for (size_t i = 0; i < g_stage_free.size(); ++i)
            if (g_stage_free[i]->dev == dev) {
                s = g_stage_free[i];
                g_stage_free.erase(g_stage_free.begin() + i);
                break;
            }
    }
    if (!s) {
        s = new HostStage;
        s->dev = dev;
        for (auto& st : s->st)
            if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) st = nullptr;
        for (auto& e : s->ev)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) e = nullptr;
        if (!s->st[0] || !s->st[1] || !s->ev[kSlots - 1]) {
            cudaGetLastError();
            return nullptr;  // leaks the half-built stage; only on a broken device
        }
    }
    if (s->cap < cap || s->nslots < nslots) {
        cap = std::max(cap, s->cap);
        stage_free_buffers(s);
        bool ok = true;
        for (auto& d : s->dbuf) ok = ok && cudaMalloc(reinterpret_cast<void**>(&d), cap * sizeof(float)) == cudaSuccess;
        for (auto& d : s->dwide) ok = ok && cudaMalloc(reinterpret_cast<void**>(&d), cap * sizeof(double)) == cudaSuccess;
        for (int k = 0; k < nslots; ++k)
            ok = ok && cudaHostAlloc(reinterpret_cast<void**>(&s->pin[k]), cap * sizeof(float), cudaHostAllocDefault) == cudaSuccess;
        s->nslots = nslots;
        if (!ok) {
            cudaGetLastError();
            stage_free_buffers(s);
            std::lock_guard<std::mutex> lk(g_stage_m);
            g_stage_free.push_back(s);
            return nullptr;
        }
        s->cap = cap;
    }
    return s;
}

void stage_release(HostStage* s) {
    std::lock_guard<std::mutex> lk(g_stage_m);
    g_stage_free.push_back(s);
}

bool is_pinned(const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

bool env_flag(const char* name, bool dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) != 0 : dflt;
}

double env_double(const char* name, double dflt) {
    const char* e = std::getenv(name);
    return e ? std::atof(e) : dflt;
}

}  // namespace

static int generate_host(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t extent,
                         void* host_out, uint64_t n_out, bool f64) {
    if (int st = validate_cfg(cfg)) return st;
    if (extent < 1 || extent > TG_MAX_EXTENT)
        return fail(TG_EVALIDATION, "generate: extent must be in [1, 131072]");
    if (n_out != static_cast<uint64_t>(extent) * static_cast<uint64_t>(extent))
        return fail(TG_EVALIDATION, "generate: output buffer size mismatch");
    if (!host_out) return fail(TG_EVALIDATION, "generate: null output");
    if (int st = validate_window(cfg, ox, oy, extent, extent)) return st;
    if (int st = device_ready()) return st;
    int dev = 0;
    TG_CUDA(cudaGetDevice(&dev));

    const int64_t th = tg::fbm2d_tile_h();
    const bool pinned = is_pinned(host_out);
    const bool direct32 = !f64 && pinned;  // fp32 into pinned: one DMA per band
    // full bands: an eighth of the map, between 0.5 MiB and 4 MiB of fp32 (8 MiB
    // when the band is DMA'd straight into the destination: larger copies
    // move 2 % faster and no host work hides behind them)
    const int64_t band_log2 = static_cast<int64_t>(env_double("TG_HOST_BAND_LOG2", TG_BAND_LOG2));
    const int64_t band_base = int64_t(1) << std::min<int64_t>(std::max<int64_t>(band_log2, 16), 26);
    const int64_t band_elems = direct32 ? 2 * band_base : band_base;
    const int64_t hi = std::max<int64_t>(th, band_elems / extent / th * th);
    const int64_t lo = ((band_elems / 8 + extent - 1) / extent + th - 1) / th * th;
    int64_t band = std::min(std::max(extent / 8 / th * th, lo), hi);
    band = std::min<int64_t>(std::max<int64_t>(band, th), extent);
    // Band schedule: uniform bands of whole tile rows, the remainder last.
    // (Short bands at both ends — 1, 1, 2, 4 tile rows, so that widening starts
    // and ends on a tile row — measured slower once the pool joined
    // asynchronously: 1.40 vs 1.34 ms at config 2, 0.23 vs 0.19 ms at 1024^2;
    // every extra copy costs more than the shorter fill and tail save.)
    std::vector<int64_t> band_h;
    for (int64_t rest = extent; rest > 0; rest -= band) band_h.push_back(std::min(band, rest));
    const int64_t nb = static_cast<int64_t>(band_h.size());
    std::vector<int64_t> band_y(band_h.size());
    for (int64_t k = 0, y = 0; k < nb; y += band_h[k++]) band_y[k] = y;
    const int64_t band_cap = *std::max_element(band_h.begin(), band_h.end());
    // f64 destinations: bands cross PCIe as fp32 (4 B/sample) into the pinned
    // staging ring and the host pool widens them into the caller's buffer
    // while later bands are in flight.  With a pinned destination a fraction
    // TG_HOST_WIDEN_FRAC of the bands may instead be widened on the device and
    // DMA'd as f64 straight into it (8 B/sample, no host work): the default is
    // all-host when the pool has >= 4 workers (config 2 on the B200 host:
    // 1.5-1.6 ms vs 2.45 ms device-widened), all-device otherwise.  Pageable
    // destinations always take the host route (a pageable DMA is
    // driver-staged anyway).
    // Mixing the two routes per band (host-widening a fraction 2P / (P + H)
    // of the bands, P / H the PCIe / host time of a band) measured no better
    // than all-host even when the host was the slower side (B200 host,
    // 1.98 ms all-host vs 2.06-2.28 ms at fractions 0.875-0.5): the f64 DMA
    // slows the host workers as much as it relieves them.
    const double frac_dflt = tg::host::threads() >= 4 ? 1.0 : 0.0;
    double frac = f64 ? (pinned ? env_double("TG_HOST_WIDEN_FRAC", frac_dflt) : 1.0) : 1.0;
    frac = std::min(1.0, std::max(0.0, frac));
    auto host_widened = [&](int64_t i) {
        return std::floor(static_cast<double>(i + 1) * frac) > std::floor(static_cast<double>(i) * frac);
    };
    const bool nt = env_flag("TG_HOST_STREAM_STORES", true);

    int rc = TG_OK;
    // ring of ns staging slots (TG_HOST_SLOTS, default 8): kLook bands
    // generated / copied ahead of the one the pool is widening, one slot being
    // widened, one whose widening the next submission joins.  The depth keeps
    // a slot from being rewritten by DMA while its lines are still in the
    // workers' caches.
    const int ns = std::min(kSlots, std::max(3, static_cast<int>(env_double("TG_HOST_SLOTS", 8))));
    const int kLook = std::min(ns - 2, std::max(1, static_cast<int>(env_double("TG_HOST_LOOK", ns - 2))));
    HostStage* s = stage_acquire(dev, static_cast<size_t>(band_cap) * static_cast<size_t>(extent), ns);
    if (!s) return fail(TG_EDEVICE, "generate: staging allocation failed");
    const bool dbg = env_flag("TG_HOST_DEBUG", false);
    // workers poll between bands for the length of this call (direct fp32
    // DMA into a pinned destination has no host work)
    std::unique_ptr<tg::host::Burst> burst;
    if (!direct32 && env_flag("TG_HOST_SPIN", true)) burst.reset(new tg::host::Burst);
    // The pool widens band j while this thread queues the device work of the
    // bands after it (launch + copy + event: ~15 us per band that used to sit
    // on the host-bound critical path); a submission first joins the previous
    // band's job, so a slot's widening is complete two submissions later,
    // before its slot is copied into again.
    tg::host::Pending pending;
    auto drain = [&](int64_t j) {
        const int slot = static_cast<int>(j % ns);
        const auto tw0 = std::chrono::steady_clock::now();
        if (cudaError_t e = cudaEventSynchronize(s->ev[slot])) {
            if (rc == TG_OK) rc = cuda_fail(e, "generate_host");
            pending.wait();
            return;
        }
        if (direct32 || rc != TG_OK || (f64 && !host_widened(j))) {
            pending.wait();
            return;
        }
        const size_t n = static_cast<size_t>(band_h[j]) * static_cast<size_t>(extent);
        const size_t off = static_cast<size_t>(band_y[j]) * static_cast<size_t>(extent);
        const auto t0 = std::chrono::steady_clock::now();
        if (f64) pending = tg::host::widen_async(s->pin[slot], static_cast<double*>(host_out) + off, n, nt);
        else pending = tg::host::copy_async(s->pin[slot], static_cast<float*>(host_out) + off, n, nt);
        if (dbg)  // TG_HOST_DEBUG=1: per band, the wait for its copy and the join of the previous band's job
            std::fprintf(stderr, "band %lld rows %lld wait %.1f us join+submit %.1f us\n", static_cast<long long>(j),
                         static_cast<long long>(band_h[j]), std::chrono::duration<double, std::micro>(t0 - tw0).count(),
                         std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    };
    tg::FbmArgs a;
    int64_t issued = 0;
    for (int64_t i = 0; i < nb && rc == TG_OK; ++i) {
        const int64_t y0 = band_y[i], h = band_h[i];
        const int b = static_cast<int>(i & 1), slot = static_cast<int>(i % ns);
        if (build_args(cfg, ox, oy + y0, extent, h, extent, &a) != TG_OK) {
            rc = TG_EDEVICE;
            break;
        }
        const size_t n = static_cast<size_t>(h) * static_cast<size_t>(extent);
        const size_t off = static_cast<size_t>(y0) * static_cast<size_t>(extent);
        cudaError_t e = tg::fbm2d_launch(kind_of(cfg), order_of(cfg), a, s->dbuf[b], s->st[b]);
        if (e == cudaSuccess) {
            if (f64 && !host_widened(i)) {
                e = tg::widen_launch(s->dbuf[b], s->dwide[b], n, s->st[b]);
                if (e == cudaSuccess)
                    e = cudaMemcpyAsync(static_cast<double*>(host_out) + off, s->dwide[b], n * sizeof(double),
                                        cudaMemcpyDeviceToHost, s->st[b]);
            } else {
                void* dst = direct32 ? static_cast<void*>(static_cast<float*>(host_out) + off) : s->pin[slot];
                e = cudaMemcpyAsync(dst, s->dbuf[b], n * sizeof(float), cudaMemcpyDeviceToHost, s->st[b]);
            }
        }
        if (e == cudaSuccess) e = cudaEventRecord(s->ev[slot], s->st[b]);
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "generate_host");
            break;
        }
        issued = i + 1;
        if (i >= kLook) drain(i - kLook);
    }
    for (int64_t j = std::max<int64_t>(0, issued - kLook); j < issued; ++j) drain(j);
    pending.wait();
    for (auto st : s->st) {
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess && rc == TG_OK) rc = cuda_fail(e, "generate_host sync");
    }
    stage_release(s);
    return rc;
}

int tg_fbm_generate_f64_host(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t extent,
                             double* host_out, uint64_t n_out) {
    return generate_host(cfg, ox, oy, extent, host_out, n_out, true);
}

int tg_fbm_generate_f32_host(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t extent,
                             float* host_out, uint64_t n_out) {
    return generate_host(cfg, ox, oy, extent, host_out, n_out, false);
}

int tg_fbm3d_generate_f32(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t oz,
                          int64_t nx, int64_t ny, int64_t nz, float* dev_out, void* stream) {
    if (int st = validate_cfg(cfg)) return st;
    if (cfg->method != TG_METHOD_ZG_SEPARABLE)
        return fail(TG_EVALIDATION, "fbm3d: only the separable zero-gradient cell is defined in 3D");
    if (nx < 1 || ny < 1 || nz < 1 || nx > TG_MAX_EXTENT || ny > TG_MAX_EXTENT || nz > TG_MAX_EXTENT)
        return fail(TG_EVALIDATION, "fbm3d: extent out of range");
    if (int st = validate_window(cfg, ox, oy, 1, 1)) return st;
    if (int st = validate_window(cfg, oz, 0, 1, 1)) return st;
    if (!dev_out) return fail(TG_EVALIDATION, "fbm3d: null output");
    if (int st = device_ready()) return st;
    tg::Fbm3Args a;
    std::memset(&a, 0, sizeof(a));
    int tx, ty, tz;
    tg::fbm3d_tile(&tx, &ty, &tz);
    a.ox = ox;
    a.oy = oy;
    a.oz = oz;
    a.nx = nx;
    a.ny = ny;
    a.nz = nz;
    a.tile_x0 = floor_div(ox, tx) * tx;
    a.tile_y0 = floor_div(oy, ty) * ty;
    a.tile_z0 = floor_div(oz, tz) * tz;
    a.R = static_cast<double>(cfg->resolution);
    a.octaves = cfg->octaves;
    a.zero = cfg->zero_lattice ? 1 : 0;
    a.seed_key = cfg->seed * tg::kSeedMul + tg::kMapKeyBias;
    int64_t gmax = 0;
    const int64_t cand[6] = {ox - 64, ox + nx + 64, oy - 64, oy + ny + 64, oz - 64, oz + nz + 64};
    for (int64_t v : cand) gmax = std::max<int64_t>(gmax, v < 0 ? -v : v);
    plan_octaves(cfg, gmax, a.oct, false);
    a.hoff = amp_offset(a.oct, cfg->octaves);
    tg::fbm3d_plan(&a, 1);
    a.lut = tg::row_lut(order_of(cfg));
    if (!a.lut) return fail(TG_EDEVICE, "row LUT allocation failed");
    TG_CUDA(tg::fbm3d_launch(order_of(cfg), a, dev_out, static_cast<cudaStream_t>(stream)));
    return TG_OK;
}

int tg_lattice_hash(const tg_lattice_key* dev_keys, uint64_t n, uint64_t lane, uint64_t* dev_out,
                    void* stream) {
    if (n == 0) return TG_OK;
    if (!dev_keys || !dev_out) return fail(TG_EVALIDATION, "lattice_hash: null pointer");
    if (int st = device_ready()) return st;
    TG_CUDA(tg::lattice_launch(0, dev_keys, n, lane, dev_out, static_cast<cudaStream_t>(stream)));
    return TG_OK;
}

int tg_lattice_height_f32(const tg_lattice_key* dev_keys, uint64_t n, float* dev_out,
                          void* stream) {
    if (n == 0) return TG_OK;
    if (!dev_keys || !dev_out) return fail(TG_EVALIDATION, "lattice_height: null pointer");
    if (int st = device_ready()) return st;
    TG_CUDA(tg::lattice_launch(1, dev_keys, n, 0, dev_out, static_cast<cudaStream_t>(stream)));
    return TG_OK;
}

int tg_lattice_unit_gradient_f32(const tg_lattice_key* dev_keys, uint64_t n, float* dev_out,
                                 void* stream) {
    if (n == 0) return TG_OK;
    if (!dev_keys || !dev_out) return fail(TG_EVALIDATION, "lattice_unit_gradient: null pointer");
    if (int st = device_ready()) return st;
    TG_CUDA(tg::lattice_launch(2, dev_keys, n, 0, dev_out, static_cast<cudaStream_t>(stream)));
    return TG_OK;
}

}  // extern "C"

// Error helpers for the other translation units.
namespace tg {
int set_error(int code, const char* msg) { return fail(code, msg); }
int set_cuda_error(cudaError_t e, const char* where) { return cuda_fail(e, where); }
int check_device() { return device_ready(); }
}  // namespace tg
