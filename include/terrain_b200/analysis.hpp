#pragma once

// terrain_b200/analysis.hpp — drop-in for the reference's fractal analysis
// (/root/reference/proj/include/terrain/analysis.hpp:20-346) on the B200:
// the median sea level, coastline mask and box counts run as device kernels
// through the C-ABI; the log-log fit (a handful of points) stays on the host.
//
// Deviation: the device pass works on fp32 maps, so host
// Heightmaps must hold fp32-representable values — true for every map this
// library generates (they are fp32 results widened exactly).  Other values
// are rejected with ValidationError instead of being silently rounded.

#include <cmath>
#include <cstdint>
#include <span>
#include <vector>

#include <cuda_runtime.h>

#include "fbm.hpp"

namespace terrain_b200::analysis {

struct LinearFit {  // analysis.hpp:20-24
    double slope = 0.0;
    double intercept = 0.0;
    double r2 = 1.0;
};

inline LinearFit linear_fit(std::span<const double> xs, std::span<const double> ys) {  // 29-63
    if (xs.size() != ys.size()) throw ValidationError("linear_fit: mismatched series lengths");
    const std::size_t n = xs.size();
    if (n < 2) throw ValidationError("linear_fit: need at least two points");
    double mx = 0.0, my = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        mx += xs[i];
        my += ys[i];
    }
    mx /= static_cast<double>(n);
    my /= static_cast<double>(n);
    double sxx = 0.0, sxy = 0.0, syy = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        const double dx = xs[i] - mx, dy = ys[i] - my;
        sxx += dx * dx;
        sxy += dx * dy;
        syy += dy * dy;
    }
    if (sxx == 0.0) throw ValidationError("linear_fit: x values are all equal");
    LinearFit fit;
    fit.slope = sxy / sxx;
    fit.intercept = my - fit.slope * mx;
    if (syy == 0.0) {
        fit.r2 = 1.0;
        return fit;
    }
    double ssr = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        const double r = ys[i] - (fit.slope * xs[i] + fit.intercept);
        ssr += r * r;
    }
    fit.r2 = 1.0 - ssr / syy;
    return fit;
}

struct BoxCountReport {  // analysis.hpp:252-259
    std::vector<int> sizes;
    std::vector<long long> counts;
    std::vector<double> lengths;
    double d = 0.0;
    double k = 0.0;
    double r2 = 0.0;
    double sea_level = 0.0;
    double land_fraction = 0.0;
    long long coast_pixels = 0;
};

inline std::vector<int> default_box_sizes() { return {2, 4, 8, 16, 32, 64}; }  // 261

namespace detail {
struct DeviceMap {
    float* ptr = nullptr;
    explicit DeviceMap(const fbm::Heightmap& hm) {
        const std::size_t n = hm.data.size();
        std::vector<float> f(n);
        for (std::size_t i = 0; i < n; ++i) {
            f[i] = static_cast<float>(hm.data[i]);
            if (static_cast<double>(f[i]) != hm.data[i])
                throw ValidationError("analysis: heightmap values must be fp32-representable");
        }
        if (cudaMalloc(&ptr, n * sizeof(float)) != cudaSuccess) throw DeviceError("analysis: cudaMalloc failed");
        if (cudaMemcpy(ptr, f.data(), n * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
            throw DeviceError("analysis: upload failed");
    }
    ~DeviceMap() { cudaFree(ptr); }
};

inline BoxCountReport fit_report(const std::vector<int>& sizes, const std::vector<long long>& counts) {
    BoxCountReport rep;
    rep.sizes = sizes;
    rep.counts = counts;
    std::vector<double> le, lc;
    for (std::size_t i = 0; i < sizes.size(); ++i) {
        rep.lengths.push_back(static_cast<double>(counts[i]) * static_cast<double>(sizes[i]));
        le.push_back(std::log(static_cast<double>(sizes[i])));
        lc.push_back(std::log(static_cast<double>(counts[i])));
    }
    const auto fit = linear_fit(le, lc);  // analysis.hpp:300-304
    rep.d = -fit.slope;
    rep.k = std::exp(fit.intercept);
    rep.r2 = fit.r2;
    return rep;
}
}  // namespace detail

// Upper median of a device map (analysis.hpp:244-250).
inline float upper_median(const float* dev_map, std::uint64_t n, void* stream = nullptr) {
    float m = 0.f;
    check(tg_median_f32(dev_map, n, &m, stream));
    return m;
}

// coastline_mask + box_count fused on a device map (analysis.hpp:213-305);
// sea level = upper median when not given.
inline BoxCountReport box_count_device(const float* dev_map, int resolution,
                                       std::span<const int> sizes,
                                       std::optional<double> sea_level = std::nullopt,
                                       void* stream = nullptr) {
    const double sea = sea_level ? *sea_level
                                 : upper_median(dev_map, static_cast<std::uint64_t>(resolution) * resolution, stream);
    std::vector<int32_t> sz(sizes.begin(), sizes.end());
    std::vector<long long> counts(sizes.size());
    std::vector<int64_t> c64(sizes.size());
    int64_t coast = 0, land = 0;
    check(tg_coastline_boxcount(dev_map, resolution, sea, sz.data(), static_cast<int32_t>(sz.size()), c64.data(),
                                &coast, &land, stream));
    for (std::size_t i = 0; i < c64.size(); ++i) counts[i] = c64[i];
    auto rep = detail::fit_report(std::vector<int>(sizes.begin(), sizes.end()), counts);
    rep.sea_level = sea;
    rep.land_fraction = static_cast<double>(land) / (static_cast<double>(resolution) * resolution);
    rep.coast_pixels = coast;
    return rep;
}

// Host-Heightmap forms of the reference pipeline: box_count(coastline_mask(hm))
inline BoxCountReport box_count(const fbm::Heightmap& hm, std::span<const int> sizes,
                                std::optional<double> sea_level = std::nullopt) {
    if (hm.data.empty()) throw ValidationError("coastline_mask: empty heightmap");
    detail::DeviceMap dm(hm);
    return box_count_device(dm.ptr, hm.resolution, sizes, sea_level);
}

inline BoxCountReport box_count(const fbm::Heightmap& hm) {
    const auto s = default_box_sizes();
    return box_count(hm, s);
}

struct SweepRow {  // analysis.hpp:312-317
    int octaves = 0;
    double persistence = 0.0;
    double d = 0.0;
    double r2 = 0.0;
};

// dimension_vs_octaves (analysis.hpp:320-340): generate -> median coastline ->
// box count per (N, p), maps kept on the device.
inline std::vector<SweepRow> dimension_vs_octaves(const fbm::FbmConfig& base, int n_min, int n_max,
                                                  std::span<const double> persistences,
                                                  std::span<const int> sizes) {
    if (n_min < 1 || n_max < n_min) throw ValidationError("dimension_vs_octaves: need 1 <= n_min <= n_max");
    if (persistences.empty()) throw ValidationError("dimension_vs_octaves: need at least one persistence value");
    const std::size_t n = static_cast<std::size_t>(base.resolution) * base.resolution;
    float* d = nullptr;
    if (cudaMalloc(&d, n * sizeof(float)) != cudaSuccess) throw DeviceError("sweep: cudaMalloc failed");
    std::vector<SweepRow> rows;
    try {
        for (const double p : persistences)
            for (int k = n_min; k <= n_max; ++k) {
                fbm::FbmConfig cfg = base;
                cfg.octaves = k;
                cfg.persistence = p;
                cfg.validate();
                fbm::generate_device(cfg, {0, 0}, cfg.resolution, cfg.resolution, d, cfg.resolution);
                const auto rep = box_count_device(d, cfg.resolution, sizes);
                rows.push_back({k, p, rep.d, rep.r2});
            }
    } catch (...) {
        cudaFree(d);
        throw;
    }
    cudaFree(d);
    return rows;
}

}  // namespace terrain_b200::analysis
