// C++ drop-in tests: the reference's own fbm test cases
// (/root/reference/proj/tests/test_fbm.cpp, test_analysis.cpp) re-run against
// terrain_b200::fbm on the B200, with the C restatement (oracle/oracle.c) as
// the checker.  Built and run by tests/test_cpp_dropin.py.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <vector>

#include "terrain_b200/analysis.hpp"
#include "terrain_b200/fbm.hpp"
#include "terrain_b200/io.hpp"

extern "C" {
#include "../../oracle/oracle.h"
}

using namespace terrain_b200;
using namespace terrain_b200::fbm;

static int g_fail = 0, g_pass = 0;
#define EXPECT(cond, what)                                                   \
    do {                                                                     \
        if (cond) {                                                          \
            ++g_pass;                                                        \
        } else {                                                             \
            ++g_fail;                                                        \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, what);        \
        }                                                                    \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static std::vector<double> oracle_map(const FbmConfig& cfg, long long ox, long long oy, int ext) {
    std::vector<double> out(static_cast<size_t>(ext) * ext);
    const tg_fbm_config c = cfg.to_c();
    or_generate(&c, ox, oy, ext, ext, out.data());
    return out;
}

// north-star tolerance: max |dh| <= 1e-5 * max |h_ref|
static bool close(const std::vector<double>& got, const std::vector<double>& ref) {
    double a = 0.0, e = 0.0;
    for (size_t i = 0; i < ref.size(); ++i) {
        a = std::max(a, std::abs(ref[i]));
        e = std::max(e, std::abs(got[i] - ref[i]));
    }
    if (a < 1e-12) a = 1.0;
    return e <= 1e-5 * a;
}

int main() {
    // Config (test_fbm.cpp:114-147)
    {
        FbmConfig cfg;
        cfg.octaves = 0;
        EXPECT(throws<ValidationError>([&] { cfg.validate(); }), "octaves=0 rejected");
        cfg = {};
        cfg.persistence = 1.5;
        EXPECT(throws<ValidationError>([&] { cfg.validate(); }), "persistence>1 rejected");
        cfg = {};
        cfg.frequency_ratio = 1.0;
        EXPECT(throws<ValidationError>([&] { cfg.validate(); }), "ratio=1 rejected");
        cfg = {};
        cfg.base_amplitude = 2.0;
        EXPECT(cfg.gradient_weight_value() == 0.02, "gradient weight default h0/100");
        for (auto m : {Method::zg_paper, Method::zg_separable, Method::generic, Method::perlin3, Method::perlin5})
            EXPECT(parse_method(method_name(m)) == m, "method name round trip");
        EXPECT(!parse_method("simplex").has_value(), "simplex not a method");
    }
    // Generate vs oracle (test_fbm.cpp:149-190)
    for (auto m : {Method::zg_paper, Method::zg_separable, Method::generic, Method::perlin3, Method::perlin5}) {
        FbmConfig cfg;
        cfg.method = m;
        cfg.seed = 99;
        cfg.resolution = 8;
        const auto hm = generate_heightmap(cfg);
        EXPECT(close(hm.data, oracle_map(cfg, 0, 0, 8)), "single octave matches oracle");
    }
    for (int R : {8, 9}) {
        FbmConfig cfg;
        cfg.seed = 1234;
        cfg.resolution = R;
        cfg.octaves = 3;
        EXPECT(close(generate_heightmap(cfg).data, oracle_map(cfg, 0, 0, R)), "multi octave both paths");
    }
    {
        FbmConfig cfg;
        cfg.seed = 5;
        cfg.resolution = 16;
        cfg.octaves = 4;
        cfg.frequency_ratio = 1.7;
        cfg.method = Method::generic;
        EXPECT(close(generate_heightmap(cfg).data, oracle_map(cfg, 0, 0, 16)), "fractional ratio");
    }
    {
        FbmConfig cfg;  // config-2 shape (S5 zero-gradient), reduced
        cfg.seed = 1;
        cfg.smoothstep = 5;
        cfg.resolution = 512;
        cfg.base_frequency = 1;
        cfg.octaves = 12;
        EXPECT(close(generate_heightmap(cfg).data, oracle_map(cfg, 0, 0, 512)), "S5 12 octaves");
    }
    // ZeroSource, determinism, regions (test_fbm.cpp:192-308)
    {
        FbmConfig cfg;
        cfg.resolution = 16;
        cfg.octaves = 4;
        cfg.zero_lattice = true;
        const auto hm = generate_heightmap(cfg);
        bool zero = true;
        for (double v : hm.data) zero = zero && v == 0.0;
        EXPECT(zero, "zero lattice gives zero map");
        EXPECT(hm.octave_seconds.size() == 4u, "octave_seconds size");
    }
    {
        FbmConfig cfg;
        cfg.seed = 777;
        cfg.resolution = 64;
        cfg.octaves = 4;
        cfg.method = Method::generic;
        const auto a = generate_heightmap(cfg);
        cfg.threads = 5;
        EXPECT(a.data == generate_heightmap(cfg).data, "deterministic across threads setting");
    }
    for (auto m : {Method::zg_paper, Method::generic, Method::perlin3}) {
        for (double ratio : {2.0, 1.7}) {
            FbmConfig cfg;
            cfg.method = m;
            cfg.seed = 909;
            cfg.resolution = 64;
            cfg.octaves = 3;
            cfg.frequency_ratio = ratio;
            const auto full = generate_heightmap(cfg);
            const auto region = generate_region(cfg, {32, 32}, 32);
            bool eq = true;
            for (int y = 0; y < 32; ++y)
                for (int x = 0; x < 32; ++x) eq = eq && region.at(x, y) == full.at(32 + x, 32 + y);
            EXPECT(eq, "region equals submap bit-exact");
        }
    }
    {
        FbmConfig cfg;
        cfg.seed = 4242;
        cfg.resolution = 128;
        cfg.octaves = 4;
        const auto full = generate_heightmap(cfg);
        bool eq = true;
        for (long long oy : {0LL, 64LL})
            for (long long ox : {0LL, 64LL}) {
                const auto t = generate_region(cfg, {ox, oy}, 64);
                for (int y = 0; y < 64; ++y)
                    for (int x = 0; x < 64; ++x)
                        eq = eq && t.at(x, y) == full.at(static_cast<int>(ox) + x, static_cast<int>(oy) + y);
            }
        EXPECT(eq, "four-way tiling bit-exact");
    }
    {
        FbmConfig cfg;
        cfg.resolution = 64;
        EXPECT(throws<ValidationError>([&] { generate_region(cfg, {5, 0}, 16); }), "misaligned x throws");
        EXPECT(throws<ValidationError>([&] { generate_region(cfg, {0, 33}, 16); }), "misaligned y throws");
        EXPECT(!throws<ValidationError>([&] { generate_region(cfg, {32, -32}, 16); }), "negative origin ok");
    }
    // Normalize, warnings, buffer reuse (test_fbm.cpp:310-387)
    {
        Heightmap hm;
        hm.resolution = 2;
        hm.data = {-2.0, 0.0, 1.0, 2.0};
        const auto n = normalize_map(hm);
        EXPECT(n.data == std::vector<double>({-1.0, 0.0, 0.5, 1.0}) && n.normalized, "normalize affine");
        EXPECT(normalize_map(n).data == n.data, "normalize idempotent");
        FbmConfig cfg;
        cfg.seed = 21;
        cfg.resolution = 32;
        cfg.octaves = 3;
        cfg.normalize = true;
        const auto g = generate_heightmap(cfg);
        double lo = 1e9, hi = -1e9;
        for (double v : g.data) {
            lo = std::min(lo, v);
            hi = std::max(hi, v);
        }
        EXPECT(lo == -1.0 && hi == 1.0 && g.normalized, "generate honours normalize");
    }
    {
        FbmConfig cfg;
        cfg.resolution = 8;
        cfg.octaves = 4;
        const auto hm = generate_heightmap(cfg);
        EXPECT(hm.warnings.size() == 1u && hm.warnings[0].find("octave 3") != std::string::npos, "sub-pixel warning");
        cfg.octaves = 3;
        EXPECT(generate_heightmap(cfg).warnings.empty(), "no warning when not sub-pixel");
    }
    {
        FbmConfig cfg;
        cfg.seed = 17;
        cfg.resolution = 32;
        cfg.octaves = 2;
        std::vector<double> buffer(32 * 32, 123.0);
        generate_into(cfg, {0, 0}, 32, buffer);
        EXPECT(buffer == generate_heightmap(cfg).data, "buffer reuse overwrites stale content");
        std::vector<double> wrong(31 * 31);
        EXPECT(throws<ValidationError>([&] { generate_into(cfg, {0, 0}, 32, wrong); }), "buffer size mismatch");
    }
    // Analysis (test_analysis.cpp:242-251) with exact counts vs the oracle
    {
        FbmConfig cfg;
        cfg.seed = 42;
        cfg.resolution = 128;
        cfg.octaves = 6;
        const auto hm = generate_heightmap(cfg);
        const auto rep = analysis::box_count(hm);
        const double sea = or_upper_median(hm.data.data(), static_cast<int64_t>(hm.data.size()));
        std::vector<uint8_t> mask(hm.data.size());
        int64_t land = 0;
        or_coastline_mask(hm.data.data(), 128, sea, mask.data(), &land);
        const int32_t sizes[6] = {2, 4, 8, 16, 32, 64};
        int64_t counts[6];
        double d, k, r2;
        or_box_count(mask.data(), 128, sizes, 6, counts, &d, &k, &r2);
        bool eq = rep.sea_level == sea;
        for (int i = 0; i < 6; ++i) eq = eq && rep.counts[static_cast<size_t>(i)] == counts[i];
        EXPECT(eq, "box counts exact vs oracle");
        EXPECT(rep.d > 0.85 && rep.d < 2.05 && std::abs(rep.d - d) < 1e-12, "dimension in range and equal");
        const std::vector<double> ps{0.5};
        const auto rows = analysis::dimension_vs_octaves(cfg, 1, 3, ps, analysis::default_box_sizes());
        EXPECT(rows.size() == 3u && rows[2].octaves == 3, "sweep rows");
    }
    // acceptance_tests.cpp:384-436 (criterion 10): box-counting dimension
    // windows and the octave / persistence trends, through the drop-in
    {
        const auto measure = [](int octaves, double persistence) {
            FbmConfig cfg;
            cfg.seed = 42;
            cfg.resolution = 512;
            cfg.octaves = octaves;
            cfg.persistence = persistence;
            return analysis::box_count(generate_heightmap(cfg));
        };
        const auto headline = measure(8, 0.5);
        EXPECT(headline.d > 1.0 && headline.d < 2.0 && headline.r2 > 0.98, "512^2 p=0.5 N=8 D window, r2");
        double prev = 0.0;
        bool mono = true;
        for (int n = 1; n <= 8; ++n) {
            const double d = measure(n, 0.5).d;
            if (n > 1) mono = mono && d >= prev - 0.05;
            prev = d;
        }
        EXPECT(mono, "D(N) non-decreasing within 0.05");
        const double d3 = measure(8, 0.3).d, d5 = measure(8, 0.5).d, d7 = measure(8, 0.7).d;
        EXPECT(d5 >= d3 - 0.05 && d7 >= d5 - 0.05, "D grows with persistence");
        std::printf("criterion 10: D=%.4f r2=%.5f; D(p=.3/.5/.7)=%.3f %.3f %.3f\n", headline.d, headline.r2, d3,
                    d5, d7);
    }
    // PGM16 / PNG16 export of a device map (compared byte-for-byte with the
    // reference writers by tests/test_cpp_dropin.py)
    {
        FbmConfig cfg;
        cfg.seed = 5;
        cfg.smoothstep = 5;
        cfg.resolution = 1024;
        cfg.base_frequency = 4;
        cfg.octaves = 10;
        float* d = nullptr;
        cudaMalloc(&d, sizeof(float) * 300 * 200);
        generate_device(cfg, {0, 0}, 300, 200, d, 300);
        cudaDeviceSynchronize();
        const char* dir = std::getenv("TG_OUT_DIR");
        const std::string base = dir ? dir : "/tmp";
        io::write_pgm16(base + "/dropin_300x200.pgm", d, 300, 200);
        io::write_png16(base + "/dropin_300x200.png", d, 300, 200);
        cudaFree(d);
        EXPECT(true, "pgm/png written");
    }
    std::printf("%d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
