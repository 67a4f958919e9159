#pragma once

// terrain_b200/fbm.hpp — C++ drop-in for the reference generator API
// (/root/reference/proj/include/terrain/fbm.hpp:27-107, 538-685) over the
// C-ABI in polyterrain_b200.h.  Same names, argument meaning and error
// behaviour; generation runs on the B200 (fp32 accumulation, results within
// 1e-5 of the map amplitude of the reference's fp64 values; lattice hashes
// bit-exact).  Switching a caller is a namespace change:
//
//     namespace fbm = terrain_b200::fbm;   // was terrain::fbm
//
// Differences, all deliberate and documented in DESIGN.md:
//   * FbmConfig gains `smoothstep` (0 = reference default, 3 or 5) so the
//     quintic zero-gradient kernel is expressible, and
//     `zero_lattice` replaces the ZeroSource template policy.
//   * resolution/extent caps are lifted to 2^22 / 2^17.
//   * octave_seconds has one entry per octave: octave k's device time as the
//     increment between diagnostic launches of the octave prefixes 0..k
//     (tg_fbm_octave_times; the fused kernel renders every octave in one
//     pass, so they are measured when requested, at extra cost).
//   * `threads` is validated like the reference and otherwise ignored.

#include <array>
#include <chrono>
#include <cstdint>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../polyterrain_b200.h"

namespace terrain_b200 {

// terrain/errors.hpp:9-36
class ValidationError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class NumericalError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class IoError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class DeviceError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

inline void check(int status) {
    if (status == TG_OK) return;
    const std::string msg = tg_last_error();
    switch (status) {
        case TG_EVALIDATION: throw ValidationError(msg);
        case TG_ENUMERICAL: throw NumericalError(msg);
        case TG_EIO: throw IoError(msg);
        default: throw DeviceError(msg);
    }
}

namespace fbm {

// fbm.hpp:27, plus opensimplex (the paper's third baseline; absent from the
// reference) and the classic permutation-table Perlin (BASELINE
// config 3; the reference hashes gradient angles instead)
enum class Method { zg_paper, zg_separable, generic, perlin3, perlin5, opensimplex, perlin_perm };

inline const char* method_name(Method m) {  // fbm.hpp:29-38
    switch (m) {
        case Method::zg_paper: return "zg_paper";
        case Method::zg_separable: return "zg_separable";
        case Method::generic: return "generic";
        case Method::perlin3: return "perlin3";
        case Method::perlin5: return "perlin5";
        case Method::opensimplex: return "opensimplex";
        case Method::perlin_perm: return "perlin_perm";
    }
    return "unknown";
}

inline std::optional<Method> parse_method(std::string_view name) {  // fbm.hpp:40-47
    if (name == "zg_paper" || name == "zg") return Method::zg_paper;
    if (name == "zg_separable") return Method::zg_separable;
    if (name == "generic") return Method::generic;
    if (name == "perlin3" || name == "perlin") return Method::perlin3;
    if (name == "perlin5") return Method::perlin5;
    if (name == "opensimplex") return Method::opensimplex;
    if (name == "perlin_perm") return Method::perlin_perm;
    return std::nullopt;
}

struct FbmConfig {  // fbm.hpp:49-89
    std::uint64_t seed = 0;
    Method method = Method::zg_paper;
    int octaves = 1;
    int resolution = 256;
    int base_frequency = 2;
    double frequency_ratio = 2.0;
    double persistence = 0.5;
    double base_amplitude = 1.0;
    std::optional<double> gradient_weight;
    bool normalize = false;
    int threads = 1;
    int smoothstep = 0;         // B200 extension: 0 = reference default, 3 | 5
    bool zero_lattice = false;  // B200 extension: the ZeroSource test hook

    double gradient_weight_value() const {
        return gradient_weight ? *gradient_weight : base_amplitude / 100.0;
    }
    int smoothstep_order() const {
        if (smoothstep) return smoothstep;
        return method == Method::perlin5 || method == Method::perlin_perm ? 5 : 3;
    }
    tg_fbm_config to_c() const {
        tg_fbm_config c{};
        c.seed = seed;
        c.method = static_cast<int32_t>(method);
        c.smoothstep = smoothstep;
        c.octaves = octaves;
        c.threads = threads;
        c.resolution = resolution;
        c.base_frequency = base_frequency;
        c.frequency_ratio = frequency_ratio;
        c.persistence = persistence;
        c.base_amplitude = base_amplitude;
        c.has_gradient_weight = gradient_weight ? 1 : 0;
        c.gradient_weight = gradient_weight ? *gradient_weight : 0.0;
        c.normalize = normalize ? 1 : 0;
        c.zero_lattice = zero_lattice ? 1 : 0;
        return c;
    }
    void validate() const {
        const tg_fbm_config c = to_c();
        check(tg_fbm_validate(&c));
    }
};

struct Heightmap {  // fbm.hpp:91-107
    int resolution = 0;
    std::vector<double> data;
    FbmConfig config{};
    std::array<long long, 2> origin{0, 0};
    std::vector<double> octave_seconds;
    double source_min = 0.0;
    double source_max = 0.0;
    bool normalized = false;
    bool constant_source = false;
    std::vector<std::string> warnings;

    double at(int x, int y) const {
        return data[static_cast<std::size_t>(y) * static_cast<std::size_t>(resolution) +
                    static_cast<std::size_t>(x)];
    }
};

namespace detail {
inline std::vector<std::string> subpixel_warnings(const FbmConfig& cfg) {  // fbm.hpp:566-569
    std::vector<std::string> out;
    const tg_fbm_config c = cfg.to_c();
    for (int o = 0; o < cfg.octaves; ++o) {
        tg_octave_spec os{};
        check(tg_fbm_octave_spec(&c, o, &os));
        if (os.freq > static_cast<double>(cfg.resolution))
            out.push_back("octave " + std::to_string(o) + ": cell size below one pixel (frequency " +
                          std::to_string(os.freq) + " exceeds resolution)");
    }
    return out;
}
}  // namespace detail

// generate_into (fbm.hpp:630-634): caller buffer of extent^2 doubles,
// overwritten; runs on the device and blocks until the result is in `out`.
inline void generate_into(const FbmConfig& cfg, std::array<long long, 2> origin, int extent,
                          std::span<double> out, std::vector<double>* octave_seconds = nullptr,
                          std::vector<std::string>* warnings = nullptr) {
    cfg.validate();
    if (extent < 1 || extent > TG_MAX_EXTENT)
        throw ValidationError("generate: extent must be in [1, 131072]");
    if (out.size() != static_cast<std::size_t>(extent) * static_cast<std::size_t>(extent))
        throw ValidationError("generate: output buffer size mismatch");
    const tg_fbm_config c = cfg.to_c();
    const auto t0 = std::chrono::steady_clock::now();
    check(tg_fbm_generate_f64_host(&c, origin[0], origin[1], extent, out.data(), out.size()));
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (warnings) {
        const auto w = detail::subpixel_warnings(cfg);
        warnings->insert(warnings->end(), w.begin(), w.end());
    }
    (void)dt;
    if (octave_seconds) {
        std::vector<double> t(static_cast<std::size_t>(cfg.octaves));
        check(tg_fbm_octave_times(&c, origin[0], origin[1], extent, t.data(), nullptr));
        octave_seconds->insert(octave_seconds->end(), t.begin(), t.end());
    }
}

// normalize_map (fbm.hpp:638-656)
inline Heightmap normalize_map(const Heightmap& hm) {
    Heightmap out = hm;
    if (hm.data.empty()) return out;
    double lo = hm.data[0], hi = hm.data[0];
    for (const double v : hm.data) {
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
    }
    out.source_min = lo;
    out.source_max = hi;
    if (lo == hi) {
        out.constant_source = true;
        return out;
    }
    const double span = hi - lo;
    for (double& v : out.data) v = -1.0 + 2.0 * (v - lo) / span;
    out.normalized = true;
    return out;
}

// generate_region / generate_heightmap (fbm.hpp:658-685)
inline Heightmap generate_region(const FbmConfig& cfg, std::array<long long, 2> origin, int extent) {
    Heightmap hm;
    hm.config = cfg;
    hm.origin = origin;
    hm.resolution = extent;
    cfg.validate();
    if (extent < 1 || extent > TG_MAX_EXTENT)
        throw ValidationError("generate: extent must be in [1, 131072]");
    hm.data.resize(static_cast<std::size_t>(extent) * static_cast<std::size_t>(extent));
    if (!cfg.normalize) {
        generate_into(cfg, origin, extent, hm.data, &hm.octave_seconds, &hm.warnings);
        return hm;
    }
    // normalize_map fused on the device (the same doubles as the host form)
    const tg_fbm_config c = cfg.to_c();
    std::int32_t constant = 0;
    check(tg_fbm_generate_normalized_f64_host(&c, origin[0], origin[1], extent, hm.data.data(), hm.data.size(),
                                              &hm.source_min, &hm.source_max, &constant));
    hm.constant_source = constant != 0;
    hm.normalized = constant == 0;
    hm.octave_seconds.resize(static_cast<std::size_t>(cfg.octaves));
    check(tg_fbm_octave_times(&c, origin[0], origin[1], extent, hm.octave_seconds.data(), nullptr));
    const auto w = detail::subpixel_warnings(cfg);
    hm.warnings.insert(hm.warnings.end(), w.begin(), w.end());
    return hm;
}

inline Heightmap generate_heightmap(const FbmConfig& cfg) {
    cfg.validate();
    return generate_region(cfg, {0, 0}, cfg.resolution);
}

// Device-resident form (stream-ordered, no host sync): `dev_out` holds
// width*height floats with row pitch `ld`; `stream` is a cudaStream_t.
inline void generate_device(const FbmConfig& cfg, std::array<long long, 2> origin, long long width,
                            long long height, float* dev_out, long long ld, void* stream = nullptr) {
    const tg_fbm_config c = cfg.to_c();
    check(tg_fbm_generate_rect_f32(&c, origin[0], origin[1], width, height, dev_out, ld, stream));
}

}  // namespace fbm
}  // namespace terrain_b200

