// terrain_b200 — GPU command-line front-end, mirroring the
// reference CLI's generate / analyze / bench subcommands and flags
// (/root/reference/proj/tools/terrain_cli.cpp:44-64, 242-271, 327-377,
// 391-452) and its exit codes (538-553: 0 ok, 1 validation, 2 io,
// 3 numerical).  Everything runs on the B200 through include/terrain_b200/.
//
//   terrain_b200 generate --size 4096 --octaves 12 --freq 8 --smoothstep 5 --out map --format png [--gradient-maps]
//   terrain_b200 texture  --kind marble --gain 1 --pattern-freq 4 --size 1024 --out tex
//   terrain_b200 analyze  --size 1024 --octaves 8 [--sea-level v] [--box-sizes 2,4,8,16]
//   terrain_b200 analyze  --in map.pgm | --sweep --n-min 1 --n-max 8 --persistences 0.3,0.5,0.7
//   terrain_b200 bench    --methods zg,perlin3,generic --octaves 1,2,4,8 --sizes 1024 --reps 20
//                         [--csv t.csv] [--speedup-csv s.csv]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <cmath>
#include <map>
#include <memory>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "terrain_b200/analysis.hpp"
#include "terrain_b200/fbm.hpp"
#include "terrain_b200/io.hpp"

using namespace terrain_b200;

namespace {

struct Args {
    std::string cmd;
    std::map<std::string, std::string> kv;
    std::vector<std::string> flags;
    bool has(const std::string& k) const { return kv.count(k) != 0; }
    bool flag(const std::string& k) const { return std::find(flags.begin(), flags.end(), k) != flags.end(); }
    std::string get(const std::string& k, const std::string& d) const { return has(k) ? kv.at(k) : d; }
};

template <class T>
T num(const std::string& s, const char* what) {
    std::istringstream is(s);
    T v{};
    if (!(is >> v) || !is.eof()) throw ValidationError(std::string("bad value for ") + what + ": " + s);
    return v;
}

template <class T>
std::vector<T> list(const std::string& s, const char* what) {
    std::vector<T> out;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) out.push_back(num<T>(tok, what));
    return out;
}

// to_config (terrain_cli.cpp:78-117); --smoothstep 5 is also accepted for zg
// (the quintic zero-gradient kernel).
fbm::FbmConfig to_config(const Args& a) {
    fbm::FbmConfig cfg;
    const auto m = fbm::parse_method(a.get("--method", "zg"));
    if (!m) throw ValidationError("unknown method: " + a.get("--method", "zg"));
    cfg.method = *m;
    if (a.has("--variant")) {
        const std::string v = a.kv.at("--variant");
        if (cfg.method != fbm::Method::zg_paper && cfg.method != fbm::Method::zg_separable)
            throw ValidationError("--variant only applies to the zg method");
        if (v == "paper") cfg.method = fbm::Method::zg_paper;
        else if (v == "separable") cfg.method = fbm::Method::zg_separable;
        else throw ValidationError("unknown variant: " + v);
    }
    if (a.has("--smoothstep")) {
        const int s = num<int>(a.kv.at("--smoothstep"), "--smoothstep");
        if (s != 3 && s != 5) throw ValidationError("--smoothstep must be 3 or 5");
        if (cfg.method == fbm::Method::perlin3 || cfg.method == fbm::Method::perlin5)
            cfg.method = s == 5 ? fbm::Method::perlin5 : fbm::Method::perlin3;
        else
            cfg.smoothstep = s;
    }
    cfg.seed = num<unsigned long long>(a.get("--seed", "0"), "--seed");
    cfg.resolution = num<int>(a.get("--size", "256"), "--size");
    cfg.octaves = num<int>(a.get("--octaves", "6"), "--octaves");
    cfg.persistence = num<double>(a.get("--persistence", "0.5"), "--persistence");
    cfg.base_frequency = num<int>(a.get("--freq", "2"), "--freq");
    cfg.frequency_ratio = num<double>(a.get("--freq-ratio", "2"), "--freq-ratio");
    cfg.base_amplitude = num<double>(a.get("--amplitude", "1"), "--amplitude");
    if (a.has("--gradient-weight")) cfg.gradient_weight = num<double>(a.kv.at("--gradient-weight"), "--gradient-weight");
    cfg.normalize = a.flag("--normalize");
    int threads = a.has("--threads") ? num<int>(a.kv.at("--threads"), "--threads") : -1;
    if (threads < 0) {  // terrain_cli.cpp:66-76
        const char* env = std::getenv("TERRAIN_THREADS");
        threads = env ? num<int>(env, "TERRAIN_THREADS") : 1;
    }
    cfg.threads = threads;
    cfg.validate();
    return cfg;
}

struct DeviceMap {
    float* p = nullptr;
    DeviceMap(size_t n) {
        if (cudaMalloc(&p, n * sizeof(float)) != cudaSuccess) throw DeviceError("cudaMalloc failed");
    }
    ~DeviceMap() { cudaFree(p); }
};

std::string default_extension(const std::string& format) {  // terrain_cli.cpp:121-126
    if (format == "pgm16") return ".pgm";
    if (format == "png") return ".png";
    if (format == "csv") return ".csv";
    throw ValidationError("unknown format: " + format + " (expected pgm16, png, or csv)");
}

// "a/b.png" + "_grad" -> "a/b_grad.png" (terrain_cli.cpp:128-134)
std::string with_suffix(const std::string& path, const std::string& suffix) {
    const auto slash = path.find_last_of('/'), dot = path.find_last_of('.');
    if (dot == std::string::npos || (slash != std::string::npos && dot < slash)) return path + suffix;
    return path.substr(0, dot) + suffix + path.substr(dot);
}

std::string output_path(const Args& a, const std::string& def) {
    std::string out = a.get("--out", def);
    const auto dot = out.find_last_of('.'), slash = out.find_last_of('/');
    if (dot == std::string::npos || (slash != std::string::npos && dot < slash))
        out += default_extension(a.get("--format", "pgm16"));
    return out;
}

void write_csv(const std::string& path, const float* dev, int w, int h);

void write_map(const std::string& format, const std::string& path, const float* dev, int w, int h) {
    if (format == "pgm16") io::write_file(path, io::encode_pgm16(dev, w, h, w));
    else if (format == "png") io::write_file(path, io::encode_png16(dev, w, h, w));
    else if (format == "csv") write_csv(path, dev, w, h);
    else throw ValidationError("unknown format: " + format + " (expected pgm16, png, or csv)");
}

void write_csv(const std::string& path, const float* dev, int w, int h) {  // io.hpp:346-358
    std::vector<float> host(static_cast<size_t>(w) * h);
    if (cudaMemcpy(host.data(), dev, host.size() * sizeof(float), cudaMemcpyDeviceToHost) != cudaSuccess)
        throw DeviceError("copy failed");
    std::ofstream out(path);
    if (!out) throw IoError("cannot open for writing: " + path);
    for (int y = 0; y < h; ++y) {
        for (int x = 0; x < w; ++x) {
            if (x) out << ',';
            out << io::detail::format_double(static_cast<double>(host[static_cast<size_t>(y) * w + x]));
        }
        out << '\n';
    }
    if (!out) throw IoError("write_csv_matrix: stream write failed");
}

int run_generate(const Args& a) {  // terrain_cli.cpp:242-271
    const auto cfg = to_config(a);
    std::array<long long, 2> origin{0, 0};
    if (a.has("--origin")) {
        const auto o = list<long long>(a.kv.at("--origin"), "--origin");
        if (o.size() != 2) throw ValidationError("--origin expects x,y");
        origin = {o[0], o[1]};
    }
    const int extent = a.has("--extent") ? num<int>(a.kv.at("--extent"), "--extent") : cfg.resolution;
    const tg_fbm_config c = cfg.to_c();
    check(tg_fbm_validate_window(&c, origin[0], origin[1], extent, extent));
    DeviceMap d(static_cast<size_t>(extent) * extent);
    fbm::generate_device(cfg, origin, extent, extent, d.p, extent);
    if (cfg.normalize) {
        double lo, hi;
        check(tg_minmax_f32(d.p, static_cast<uint64_t>(extent) * extent, &lo, &hi, nullptr));
        if (hi > lo) check(tg_rescale_f32(d.p, static_cast<uint64_t>(extent) * extent, lo, hi, nullptr));
    }
    if (cudaDeviceSynchronize() != cudaSuccess) throw DeviceError("generation failed");
    for (const auto& w : fbm::detail::subpixel_warnings(cfg)) std::cerr << "warning: " << w << "\n";
    const std::string format = a.get("--format", "pgm16");
    const std::string out = output_path(a, "heightmap");
    write_map(format, out, d.p, extent, extent);
    std::cout << "wrote " << out << " (" << extent << "x" << extent << ", " << fbm::method_name(cfg.method)
              << ", " << cfg.octaves << " octaves)\n";
    if (a.flag("--gradient-maps")) {  // terrain_cli.cpp:261-264: first / second order norm images
        DeviceMap g(static_cast<size_t>(extent) * extent);
        for (const int hessian : {0, 1}) {
            check(tg_norm_map_f32(d.p, extent, extent, hessian, g.p, nullptr));
            if (cudaDeviceSynchronize() != cudaSuccess) throw DeviceError("norm map failed");
            const std::string p = with_suffix(out, hessian ? "_hess" : "_grad");
            write_map(format, p, g.p, extent, extent);
            std::cout << "wrote " << p << "\n";
        }
    }
    return 0;
}

int run_texture(const Args& a) {  // terrain_cli.cpp:282-298 (texture::render, texture.hpp:50-72)
    const auto cfg = to_config(a);
    const std::string k = a.get("--kind", "marble");
    const int kind = k == "marble" ? 0 : k == "wood" ? 1 : k == "cloud" ? 2 : -1;
    if (kind < 0) throw ValidationError("unknown texture kind: " + k);
    const double gain = num<double>(a.get("--gain", "1"), "--gain");
    const double pf = num<double>(a.get("--pattern-freq", "4"), "--pattern-freq");
    const int R = cfg.resolution;
    DeviceMap d(static_cast<size_t>(R) * R);
    const tg_fbm_config c = cfg.to_c();
    check(tg_texture_generate_f32(&c, kind, gain, pf, d.p, nullptr));
    if (cudaDeviceSynchronize() != cudaSuccess) throw DeviceError("texture failed");
    const std::string out = output_path(a, "texture");
    write_map(a.get("--format", "pgm16"), out, d.p, R, R);
    std::cout << "wrote " << out << " (" << R << "x" << R << ")\n";
    return 0;
}

void emit(const Args& a, const std::string& csv) {
    if (a.has("--out")) {
        std::ofstream f(a.kv.at("--out"));
        if (!f) throw IoError("cannot open for writing: " + a.kv.at("--out"));
        f << csv;
        std::cout << "wrote " << a.kv.at("--out") << "\n";
    } else {
        std::cout << csv;
    }
}

int run_analyze(const Args& a) {  // terrain_cli.cpp:327-377
    if (a.flag("--crest"))
        throw ValidationError("--crest: the crest quadrature is outside the B200 path (SURVEY §2)");
    std::vector<int> sizes = a.has("--box-sizes") ? list<int>(a.kv.at("--box-sizes"), "--box-sizes")
                                                  : analysis::default_box_sizes();
    if (a.flag("--sweep")) {  // dimension_vs_octaves (analysis.hpp:320-346), io.hpp:410-416
        const auto base = to_config(a);
        std::vector<double> ps = a.has("--persistences") ? list<double>(a.kv.at("--persistences"), "--persistences")
                                                         : std::vector<double>{0.3, 0.5, 0.7};
        const int n_min = num<int>(a.get("--n-min", "1"), "--n-min"), n_max = num<int>(a.get("--n-max", "8"), "--n-max");
        const auto rows = analysis::dimension_vs_octaves(base, n_min, n_max, ps, sizes);
        std::ostringstream csv;
        csv << "octaves,persistence,dimension,r2\n";
        for (const auto& r : rows)
            csv << r.octaves << ',' << io::detail::format_double(r.persistence) << ','
                << io::detail::format_double(r.d) << ',' << io::detail::format_double(r.r2) << '\n';
        emit(a, csv.str());
        std::printf("sweep: %zu rows (N=%d..%d, %zu persistence values)\n", rows.size(), n_min, n_max, ps.size());
        return 0;
    }
    std::optional<double> sea;
    if (a.has("--sea-level")) sea = num<double>(a.kv.at("--sea-level"), "--sea-level");
    int R = 0;
    std::unique_ptr<DeviceMap> d;
    analysis::BoxCountReport rep;
    if (a.has("--in")) {
        // An existing 16-bit PGM (read_pgm16_heightmap, io.hpp:170-178): its
        // heights hmin + s/65535 (hmax - hmin) are monotone in the sample s,
        // so the analysis runs exactly on the samples (integers, exact in
        // fp32) with the sea level mapped to the sample domain, and reports
        // heights — the same mask and counts as the reference's doubles.
        const auto img = io::read_pgm16(a.kv.at("--in"));
        if (img.width != img.height) throw IoError("read_pgm16_heightmap: heightmaps must be square");
        R = img.width;
        std::vector<float> h(img.samples.size());
        const bool mono = img.hmax > img.hmin;
        for (size_t i = 0; i < h.size(); ++i)
            h[i] = mono ? static_cast<float>(img.samples[i]) : static_cast<float>(img.height_of(img.samples[i]));
        d = std::make_unique<DeviceMap>(h.size());
        if (cudaMemcpy(d->p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
            throw DeviceError("upload failed");
        std::optional<double> s_sea;
        if (sea && mono) {  // smallest sample whose height reaches the sea level
            uint32_t lo = 0, hi = 65536;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) / 2;
                if (img.height_of(mid) >= *sea) hi = mid;
                else lo = mid + 1;
            }
            s_sea = static_cast<double>(lo);
        } else if (sea) {
            s_sea = sea;
        }
        rep = analysis::box_count_device(d->p, R, sizes, s_sea);
        if (mono) rep.sea_level = sea ? *sea : img.height_of(static_cast<uint32_t>(rep.sea_level));
    } else {
        const auto cfg = to_config(a);
        R = cfg.resolution;
        d = std::make_unique<DeviceMap>(static_cast<size_t>(R) * R);
        fbm::generate_device(cfg, {0, 0}, R, R, d->p, R);
        rep = analysis::box_count_device(d->p, R, sizes, sea);
    }
    std::ostringstream csv;  // io.hpp:402-408
    csv << "epsilon,count,length\n";
    for (size_t i = 0; i < rep.sizes.size(); ++i)
        csv << rep.sizes[i] << ',' << rep.counts[i] << ',' << io::detail::format_double(rep.lengths[i]) << '\n';
    emit(a, csv.str());
    std::printf("box-count: R=%d sea=%.6g land=%.3f coast_px=%lld  D=%.6f k=%.6g r2=%.6f\n", R, rep.sea_level,
                rep.land_fraction, rep.coast_pixels, rep.d, rep.k, rep.r2);
    return 0;
}

int run_bench(const Args& a) {  // terrain_cli.cpp:391-452, device-timed
    const auto methods = [&] {
        std::vector<std::string> m;
        std::stringstream ss(a.get("--methods", "zg,perlin3,generic"));
        std::string t;
        while (std::getline(ss, t, ',')) m.push_back(t);
        return m;
    }();
    const auto octaves = list<int>(a.get("--octaves", "1,2,4,8"), "--octaves");
    const auto sizes = list<int>(a.get("--sizes", "256"), "--sizes");
    const int reps = num<int>(a.get("--reps", "100"), "--reps");
    const int warmup = num<int>(a.get("--warmup", "1"), "--warmup");
    if (reps < 3) throw ValidationError("run_bench: need at least 3 repetitions");
    struct Run {
        fbm::Method m;
        int n, r, reps;
        double mean, median, min, sd;
    };
    std::vector<Run> runs;
    for (const auto& name : methods) {
        const auto m = fbm::parse_method(name);
        if (!m) throw ValidationError("unknown method: " + name);
        for (const int n : octaves)
            for (const int r : sizes) {
                fbm::FbmConfig cfg;
                cfg.method = *m;
                cfg.octaves = n;
                cfg.resolution = r;
                cfg.seed = num<unsigned long long>(a.get("--seed", "0"), "--seed");
                cfg.validate();
                DeviceMap d(static_cast<size_t>(r) * r);
                for (int i = 0; i < warmup; ++i) fbm::generate_device(cfg, {0, 0}, r, r, d.p, r);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                std::vector<double> sec(static_cast<size_t>(reps));
                for (int i = 0; i < reps; ++i) {
                    cudaEventRecord(e0);
                    fbm::generate_device(cfg, {0, 0}, r, r, d.p, r);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms = 0.f;
                    cudaEventElapsedTime(&ms, e0, e1);
                    sec[static_cast<size_t>(i)] = ms * 1e-3;
                }
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
                // bench.hpp:34-52: mean, median, min, sample standard deviation
                std::vector<double> sorted = sec;
                std::sort(sorted.begin(), sorted.end());
                double mean = 0;
                for (double v : sec) mean += v;
                mean /= reps;
                double var = 0;
                for (double v : sec) var += (v - mean) * (v - mean);
                const double med = reps % 2 ? sorted[reps / 2] : 0.5 * (sorted[reps / 2 - 1] + sorted[reps / 2]);
                runs.push_back({*m, n, r, reps, mean, med, sorted.front(), std::sqrt(var / (reps - 1))});
                std::printf("%-12s N=%d R=%-5d reps=%d  median=%.6fs mean=%.6fs sd=%.2g\n", fbm::method_name(*m), n,
                            r, reps, med, mean, runs.back().sd);
            }
    }
    if (a.has("--csv")) {  // bench.hpp:165-175
        std::ofstream f(a.kv.at("--csv"));
        if (!f) throw IoError("cannot open for writing: " + a.kv.at("--csv"));
        f << "method,octaves,resolution,repetitions,mean_seconds,median_seconds,min_seconds,stddev_seconds\n";
        char buf[192];
        for (const auto& r : runs) {
            std::snprintf(buf, sizeof(buf), "%s,%d,%d,%d,%.9g,%.9g,%.9g,%.9g\n", fbm::method_name(r.m), r.n, r.r,
                          r.reps, r.mean, r.median, r.min, r.sd);
            f << buf;
        }
    }
    // speedups vs zg_paper at the same (N, R) (bench.hpp:96-117, 177-185)
    std::map<std::pair<int, int>, double> base;
    for (const auto& r : runs)
        if (r.m == fbm::Method::zg_paper) base[{r.n, r.r}] = r.median;
    if (base.empty()) {
        std::cerr << "warning: no zg baseline run, speedups skipped\n";
    } else {
        std::ostringstream csv;
        csv << "method,octaves,resolution,median_seconds,baseline_seconds,speedup\n";
        for (const auto& r : runs) {
            const auto it = base.find({r.n, r.r});
            if (it == base.end()) continue;
            const double sp = r.median / it->second;
            std::printf("speedup %-12s N=%d R=%-5d  S=%.4f\n", fbm::method_name(r.m), r.n, r.r, sp);
            char buf[192];
            std::snprintf(buf, sizeof(buf), "%s,%d,%d,%.9g,%.9g,%.6g\n", fbm::method_name(r.m), r.n, r.r, r.median,
                          it->second, sp);
            csv << buf;
        }
        if (a.has("--speedup-csv")) {
            std::ofstream f(a.kv.at("--speedup-csv"));
            if (!f) throw IoError("cannot open for writing: " + a.kv.at("--speedup-csv"));
            f << csv.str();
        }
    }
    // cost model T = alpha N R^2 + beta 4^N per method (bench.hpp:119-163),
    // when the grid spans at least three runs of distinct shapes
    for (const auto& name : methods) {
        const auto m = *fbm::parse_method(name);
        double suu = 0, suv = 0, svv = 0, sut = 0, svt = 0, st = 0, stt = 0;
        int cnt = 0;
        for (const auto& r : runs) {
            if (r.m != m) continue;
            const double u = static_cast<double>(r.n) * r.r * r.r, v = std::pow(4.0, r.n), t = r.median;
            suu += u * u, suv += u * v, svv += v * v, sut += u * t, svt += v * t, st += t, stt += t * t;
            ++cnt;
        }
        const double det = suu * svv - suv * suv;
        if (cnt < 3 || det == 0.0 || std::abs(det) < 1e-12 * std::max(suu, svv) * std::max(suu, svv)) continue;
        const double alpha = (svv * sut - suv * svt) / det, beta = (suu * svt - suv * sut) / det;
        double ssr = 0;
        for (const auto& r : runs)
            if (r.m == m) {
                const double e = r.median - (alpha * r.n * r.r * r.r + beta * std::pow(4.0, r.n));
                ssr += e * e;
            }
        const double sst = stt - st * st / cnt;
        std::printf("cost model %-12s T = %.4g * N * R^2 + %.4g * 4^N  (r2=%.4f)\n", fbm::method_name(m), alpha, beta,
                    sst > 0 ? 1.0 - ssr / sst : 1.0);
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) {
            std::cerr << "usage: terrain_b200 {generate|texture|analyze|bench} [--flag value ...]\n";
            return 1;
        }
        Args a;
        a.cmd = argv[1];
        for (int i = 2; i < argc; ++i) {
            const std::string k = argv[i];
            if (k.rfind("--", 0) != 0) throw ValidationError("unexpected argument: " + k);
            if (k == "--normalize" || k == "--gradient-maps" || k == "--sweep" || k == "--crest") {
                a.flags.push_back(k);
                continue;
            }
            if (i + 1 >= argc) throw ValidationError("missing value for " + k);
            a.kv[k] = argv[++i];
        }
        if (a.cmd == "generate") return run_generate(a);
        if (a.cmd == "analyze") return run_analyze(a);
        if (a.cmd == "texture") return run_texture(a);
        if (a.cmd == "bench") return run_bench(a);
        throw ValidationError("unknown subcommand: " + a.cmd);
    } catch (const ValidationError& e) {  // terrain_cli.cpp:538-553
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const IoError& e) {
        std::cerr << "io error: " << e.what() << "\n";
        return 2;
    } catch (const NumericalError& e) {
        std::cerr << "numerical error: " << e.what() << "\n";
        return 3;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
