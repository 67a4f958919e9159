// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference
// headers (/root/reference/proj/include/terrain/*.hpp), compiled by
// oracle/Makefile into oracle/_ref/libtgref.so.  TEST INFRASTRUCTURE ONLY:
// used to pin the C restatement (oracle.c), to generate tests/golden/, and as
// the CPU baseline / `bench.py --impl reference` arm.  No reference source is
// copied into this repository; this file only calls the reference's API.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <sstream>
#include <string>
#include <vector>

#include "terrain/analysis.hpp"
#include "terrain/bench.hpp"
#include "terrain/fbm.hpp"
#include "terrain/io.hpp"
#include "terrain/kernels2d.hpp"
#include "terrain/lattice.hpp"
#include "terrain/texture.hpp"

#include "../include/polyterrain_b200.h"

using namespace terrain;

namespace {

thread_local std::string g_err;

// tg_fbm_config -> FbmConfig.  zg with an explicit S5 is not expressible in
// the reference FbmConfig: rejected here.
bool to_ref(const tg_fbm_config* c, fbm::FbmConfig& out) {
    out = {};
    out.seed = c->seed;
    out.method = static_cast<fbm::Method>(c->method);
    out.octaves = c->octaves;
    out.resolution = static_cast<int>(c->resolution);
    out.base_frequency = static_cast<int>(c->base_frequency);
    out.frequency_ratio = c->frequency_ratio;
    out.persistence = c->persistence;
    out.base_amplitude = c->base_amplitude;
    if (c->has_gradient_weight) out.gradient_weight = c->gradient_weight;
    out.normalize = c->normalize != 0;
    out.threads = c->threads;
    const int def = c->method == TG_METHOD_PERLIN5 ? 5 : 3;
    if (c->smoothstep != 0 && c->smoothstep != def) {
        g_err = "smoothstep order not expressible in the reference FbmConfig";
        return false;
    }
    return true;
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return TG_OK;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return TG_EVALIDATION;
    } catch (const NumericalError& e) {
        g_err = e.what();
        return TG_ENUMERICAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        return TG_EDEVICE;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_hash(uint64_t seed, uint32_t octave, int64_t ix, int64_t iy, uint64_t lane) {
    return lattice::detail::mix(lattice::detail::pack({seed, octave, ix, iy}) ^ lane);
}

void ref_hash_keys(const tg_lattice_key* keys, uint64_t n, uint64_t lane, uint64_t* out) {
    for (uint64_t i = 0; i < n; ++i)
        out[i] = ref_hash(keys[i].seed, keys[i].octave, keys[i].ix, keys[i].iy, lane);
}

void ref_corner_heights(const tg_lattice_key* keys, uint64_t n, double* out) {
    for (uint64_t i = 0; i < n; ++i)
        out[i] = lattice::corner_height({keys[i].seed, keys[i].octave, keys[i].ix, keys[i].iy});
}

void ref_corner_angles(const tg_lattice_key* keys, uint64_t n, double* out) {
    for (uint64_t i = 0; i < n; ++i)
        out[i] = lattice::corner_angle({keys[i].seed, keys[i].octave, keys[i].ix, keys[i].iy});
}

void ref_corner_unit_gradients(const tg_lattice_key* keys, uint64_t n, double* out) {
    for (uint64_t i = 0; i < n; ++i) {
        const auto g =
            lattice::corner_unit_gradient({keys[i].seed, keys[i].octave, keys[i].ix, keys[i].iy});
        out[2 * i] = g[0];
        out[2 * i + 1] = g[1];
    }
}

void ref_corner_gradients(const tg_lattice_key* keys, uint64_t n, double w, double* out) {
    for (uint64_t i = 0; i < n; ++i) {
        const auto g = lattice::corner_gradient(
            {keys[i].seed, keys[i].octave, keys[i].ix, keys[i].iy}, lattice::GradientWeight{w});
        out[2 * i] = g[0];
        out[2 * i + 1] = g[1];
    }
}

int ref_validate(const tg_fbm_config* c) {
    fbm::FbmConfig cfg;
    if (!to_ref(c, cfg)) return TG_EVALIDATION;
    return guard([&] { cfg.validate(); });
}

int ref_octave_spec(const tg_fbm_config* c, int octave, tg_octave_spec* out) {
    fbm::FbmConfig cfg;
    if (!to_ref(c, cfg)) return TG_EVALIDATION;
    const auto os = fbm::detail::octave_spec(cfg, octave);
    out->freq = os.freq;
    out->amp = os.amp;
    out->fast = os.fast;
    out->cells = os.cells;
    out->ppc = os.ppc;
    return TG_OK;
}

// fbm::generate_into / generate_into_with_source<ZeroSource> (fbm.hpp:541-634).
int ref_generate_into(const tg_fbm_config* c, int64_t ox, int64_t oy, int32_t extent,
                      double* out, uint64_t n_out, int32_t* n_warnings) {
    fbm::FbmConfig cfg;
    if (!to_ref(c, cfg)) return TG_EVALIDATION;
    return guard([&] {
        std::vector<std::string> warnings;
        std::span<double> span(out, n_out);
        if (c->zero_lattice)
            fbm::generate_into_with_source<fbm::ZeroSource>(cfg, {ox, oy}, extent, span, nullptr,
                                                            &warnings);
        else
            fbm::generate_into(cfg, {ox, oy}, extent, span, nullptr, &warnings);
        if (n_warnings) *n_warnings = static_cast<int32_t>(warnings.size());
    });
}

// fbm::generate_region (fbm.hpp:658-685), including normalize; metadata out.
int ref_generate_region(const tg_fbm_config* c, int64_t ox, int64_t oy, int32_t extent,
                        double* out, double* src_min, double* src_max, int32_t* normalized,
                        int32_t* constant_source, char* warnings, int32_t warnings_len) {
    fbm::FbmConfig cfg;
    if (!to_ref(c, cfg)) return TG_EVALIDATION;
    return guard([&] {
        const auto hm = fbm::generate_region(cfg, {ox, oy}, extent);
        std::copy(hm.data.begin(), hm.data.end(), out);
        *src_min = hm.source_min;
        *src_max = hm.source_max;
        *normalized = hm.normalized;
        *constant_source = hm.constant_source;
        std::string all;
        for (const auto& w : hm.warnings) all += w + "\n";
        if (warnings && warnings_len > 0) {
            std::strncpy(warnings, all.c_str(), static_cast<size_t>(warnings_len - 1));
            warnings[warnings_len - 1] = 0;
        }
    });
}

// The per-pixel oracle pattern of tests/test_fbm.cpp:20-80 over the
// reference's own primitives, with an explicit smoothstep order for zg (the
// only way to express zg+S5).
int ref_oracle_pixels(const tg_fbm_config* c, int64_t ox, int64_t oy, int32_t width,
                      int32_t height, double* out) {
    const int order_i = c->smoothstep ? c->smoothstep : (c->method == TG_METHOD_PERLIN5 ? 5 : 3);
    const auto order = order_i == 5 ? kernels2d::SmoothstepOrder::s5 : kernels2d::SmoothstepOrder::s3;
    const double w = c->has_gradient_weight ? c->gradient_weight : c->base_amplitude / 100.0;
    const double R = static_cast<double>(c->resolution);
    for (int32_t ly = 0; ly < height; ++ly)
        for (int32_t lx = 0; lx < width; ++lx) {
            const long long gx = ox + lx, gy = oy + ly;
            double total = 0.0, freq = static_cast<double>(c->base_frequency),
                   amp = c->base_amplitude;
            for (int oct = 0; oct < c->octaves; ++oct) {
                const double u = (static_cast<double>(gx) + 0.5) / R * freq;
                const double v = (static_cast<double>(gy) + 0.5) / R * freq;
                const long long ix = static_cast<long long>(std::floor(u));
                const long long iy = static_cast<long long>(std::floor(v));
                const double x = u - static_cast<double>(ix), y = v - static_cast<double>(iy);
                const auto key = [&](long long dx, long long dy) {
                    return lattice::LatticeKey{c->seed, static_cast<std::uint32_t>(oct), ix + dx,
                                               iy + dy};
                };
                switch (c->method) {
                    case TG_METHOD_ZG_PAPER:
                    case TG_METHOD_ZG_SEPARABLE: {
                        const auto p = kernels2d::zg_params(amp * lattice::corner_height(key(0, 0)),
                                                            amp * lattice::corner_height(key(1, 0)),
                                                            amp * lattice::corner_height(key(0, 1)),
                                                            amp * lattice::corner_height(key(1, 1)));
                        total += kernels2d::zg_eval(p, x, y,
                                                    c->method == TG_METHOD_ZG_PAPER
                                                        ? kernels2d::ZgVariant::paper
                                                        : kernels2d::ZgVariant::separable,
                                                    order);
                        break;
                    }
                    case TG_METHOD_GENERIC: {
                        std::array<kernels2d::Corner2D, 4> corners;
                        const long long off[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
                        for (int q = 0; q < 4; ++q) {
                            const auto g = lattice::corner_gradient(key(off[q][0], off[q][1]),
                                                                    lattice::GradientWeight{w});
                            corners[static_cast<size_t>(q)] = {
                                amp * lattice::corner_height(key(off[q][0], off[q][1])), g[0], g[1]};
                        }
                        total += kernels2d::generic_eval(kernels2d::generic_coeffs(corners), x, y);
                        break;
                    }
                    default: {
                        kernels2d::PerlinCellParams p;
                        p.order = order;
                        const long long off[4][2] = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
                        for (int q = 0; q < 4; ++q) {
                            const auto g = lattice::corner_unit_gradient(key(off[q][0], off[q][1]));
                            p.f[static_cast<size_t>(q)] = amp * g[0];
                            p.g[static_cast<size_t>(q)] = amp * g[1];
                        }
                        total += kernels2d::perlin_cell_eval(p, x, y);
                        break;
                    }
                }
                freq *= c->frequency_ratio;
                amp *= c->persistence;
            }
            out[static_cast<size_t>(ly) * static_cast<size_t>(width) + static_cast<size_t>(lx)] =
                total;
        }
    return TG_OK;
}

// kernels2d::zg_eval with explicit variant/order (kernels2d.hpp:70-76).
double ref_zg_eval(double h00, double h10, double h01, double h11, double x, double y,
                   int separable, int order) {
    return kernels2d::zg_eval(kernels2d::zg_params(h00, h10, h01, h11), x, y,
                              separable ? kernels2d::ZgVariant::separable
                                        : kernels2d::ZgVariant::paper,
                              order == 5 ? kernels2d::SmoothstepOrder::s5
                                         : kernels2d::SmoothstepOrder::s3);
}

// normalize_map (fbm.hpp:638-656) on a caller buffer.
int ref_normalize(double* data, int64_t n, double* lo, double* hi, int32_t* constant_source,
                  int32_t* normalized) {
    fbm::Heightmap hm;
    hm.data.assign(data, data + n);
    const auto out = fbm::normalize_map(hm);
    std::copy(out.data.begin(), out.data.end(), data);
    *lo = out.source_min;
    *hi = out.source_max;
    *constant_source = out.constant_source;
    *normalized = out.normalized;
    return TG_OK;
}

// coastline_mask (+ median) and box_count (analysis.hpp:213-310).
// use_median != 0 -> sea level = upper median (analysis.hpp:244-250).
int ref_coastline_boxcount(const double* data, int32_t R, int32_t use_median, double sea,
                           const int32_t* sizes, int32_t n_sizes, int64_t* counts, double* d,
                           double* k, double* r2, double* land_fraction, double* sea_out,
                           int64_t* coast_pixels, uint8_t* mask_out) {
    return guard([&] {
        fbm::Heightmap hm;
        hm.resolution = R;
        hm.data.assign(data, data + static_cast<size_t>(R) * static_cast<size_t>(R));
        const auto mask =
            use_median ? analysis::coastline_mask(hm) : analysis::coastline_mask(hm, sea);
        *land_fraction = mask.land_fraction;
        *sea_out = mask.sea_level;
        *coast_pixels = mask.pixel_count();
        if (mask_out) std::copy(mask.coast.begin(), mask.coast.end(), mask_out);
        if (n_sizes > 0) {
            std::vector<int> sz(sizes, sizes + n_sizes);
            const auto rep = analysis::box_count(mask, sz);
            for (int32_t i = 0; i < n_sizes; ++i) counts[i] = rep.counts[static_cast<size_t>(i)];
            *d = rep.d;
            *k = rep.k;
            *r2 = rep.r2;
        }
    });
}

// box_count on an explicit mask (analysis.hpp:269-305).
int ref_box_count_mask(const uint8_t* mask, int32_t R, const int32_t* sizes, int32_t n_sizes,
                       int64_t* counts, double* d, double* k, double* r2) {
    return guard([&] {
        analysis::CoastlineMask m;
        m.resolution = R;
        m.coast.assign(mask, mask + static_cast<size_t>(R) * static_cast<size_t>(R));
        std::vector<int> sz(sizes, sizes + n_sizes);
        const auto rep = analysis::box_count(m, sz);
        for (int32_t i = 0; i < n_sizes; ++i) counts[i] = rep.counts[static_cast<size_t>(i)];
        *d = rep.d;
        *k = rep.k;
        *r2 = rep.r2;
    });
}

// write_pgm16 / write_png16 (io.hpp:91-111, 203-257) into a caller buffer;
// returns the byte count (or -1 when it does not fit / on error).
static int64_t put_bytes(const std::string& b, uint8_t* out, int64_t cap) {
    if (static_cast<int64_t>(b.size()) > cap) return -1;
    std::memcpy(out, b.data(), b.size());
    return static_cast<int64_t>(b.size());
}

int64_t ref_encode_pgm16(const double* data, int32_t width, int32_t height, uint8_t* out, int64_t cap) {
    try {
        std::ostringstream os;
        io::write_pgm16(os, std::span<const double>(data, static_cast<size_t>(width) * height), width, height);
        return put_bytes(os.str(), out, cap);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int64_t ref_encode_png16(const double* data, int32_t width, int32_t height, uint8_t* out, int64_t cap) {
    try {
        std::ostringstream os;
        io::write_png16(os, std::span<const double>(data, static_cast<size_t>(width) * height), width, height);
        return put_bytes(os.str(), out, cap);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// texture::render (texture.hpp:50-72): full R x R map into out.
int ref_texture(const tg_fbm_config* c, int32_t kind, double gain, double pattern_frequency, double* out) {
    fbm::FbmConfig cfg;
    if (!to_ref(c, cfg)) return TG_EVALIDATION;
    return guard([&] {
        texture::TextureSpec spec;
        spec.kind = static_cast<texture::Kind>(kind);
        spec.fbm = cfg;
        spec.gain = gain;
        spec.pattern_frequency = pattern_frequency;
        const auto hm = texture::render(spec);
        std::copy(hm.data.begin(), hm.data.end(), out);
    });
}

// linear_fit (analysis.hpp:29-63).
int ref_linear_fit(const double* xs, const double* ys, int32_t n, double* slope,
                   double* intercept, double* r2) {
    return guard([&] {
        const auto f = analysis::linear_fit(std::span<const double>(xs, static_cast<size_t>(n)),
                                            std::span<const double>(ys, static_cast<size_t>(n)));
        *slope = f.slope;
        *intercept = f.intercept;
        *r2 = f.r2;
    });
}

// bench::run_bench (bench.hpp:54-78): the reference's own timing protocol.
// Returns median/min seconds per generate_into of the full map.
int ref_run_bench(const tg_fbm_config* c, int32_t reps, int32_t warmup, double* median_s,
                  double* min_s, double* mean_s) {
    fbm::FbmConfig cfg;
    if (!to_ref(c, cfg)) return TG_EVALIDATION;
    return guard([&] {
        const auto run = bench::run_bench(cfg, reps, warmup);
        *median_s = run.median;
        *min_s = run.min;
        *mean_s = run.mean;
    });
}

}  // extern "C"
