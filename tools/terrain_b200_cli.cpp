// terrain_b200 — GPU command-line front-end, mirroring the
// reference CLI's generate / analyze / bench subcommands and flags
// (/root/reference/proj/tools/terrain_cli.cpp:44-64, 242-271, 327-377,
// 391-452) and its exit codes (538-553: 0 ok, 1 validation, 2 io,
// 3 numerical).  Everything runs on the B200 through include/terrain_b200/.
//
//   terrain_b200 generate --size 4096 --octaves 12 --freq 8 --smoothstep 5 --out map --format png
//   terrain_b200 analyze  --size 1024 --octaves 8 [--sea-level v] [--box-sizes 2,4,8,16]
//   terrain_b200 bench    --methods zg,perlin3,generic --octaves 1,2,4,8 --sizes 1024 --reps 20
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
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
    std::string out = a.get("--out", "heightmap");
    const auto dot = out.find_last_of('.'), slash = out.find_last_of('/');
    const std::string ext = format == "pgm16" ? ".pgm" : format == "png" ? ".png" : format == "csv" ? ".csv" : "";
    if (ext.empty()) throw ValidationError("unknown format: " + format + " (expected pgm16, png, or csv)");
    if (dot == std::string::npos || (slash != std::string::npos && dot < slash)) out += ext;
    if (format == "pgm16") io::write_file(out, io::encode_pgm16(d.p, extent, extent, extent));
    else if (format == "png") io::write_file(out, io::encode_png16(d.p, extent, extent, extent));
    else write_csv(out, d.p, extent, extent);
    std::cout << "wrote " << out << " (" << extent << "x" << extent << ", " << fbm::method_name(cfg.method)
              << ", " << cfg.octaves << " octaves)\n";
    return 0;
}

int run_analyze(const Args& a) {  // terrain_cli.cpp:327-377 (map path)
    const auto cfg = to_config(a);
    const int R = cfg.resolution;
    std::vector<int> sizes = a.has("--box-sizes") ? list<int>(a.kv.at("--box-sizes"), "--box-sizes")
                                                  : analysis::default_box_sizes();
    std::optional<double> sea;
    if (a.has("--sea-level")) sea = num<double>(a.kv.at("--sea-level"), "--sea-level");
    DeviceMap d(static_cast<size_t>(R) * R);
    fbm::generate_device(cfg, {0, 0}, R, R, d.p, R);
    const auto rep = analysis::box_count_device(d.p, R, sizes, sea);
    std::ostringstream csv;  // io.hpp:402-408
    csv << "epsilon,count,length\n";
    for (size_t i = 0; i < rep.sizes.size(); ++i)
        csv << rep.sizes[i] << ',' << rep.counts[i] << ',' << io::detail::format_double(rep.lengths[i]) << '\n';
    if (a.has("--out")) {
        std::ofstream f(a.kv.at("--out"));
        if (!f) throw IoError("cannot open for writing: " + a.kv.at("--out"));
        f << csv.str();
    } else {
        std::cout << csv.str();
    }
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
    std::map<std::pair<int, int>, double> zg_median;
    std::vector<std::string> rows;
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
                std::vector<float> ms(static_cast<size_t>(reps));
                for (int i = 0; i < reps; ++i) {
                    cudaEventRecord(e0);
                    fbm::generate_device(cfg, {0, 0}, r, r, d.p, r);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    cudaEventElapsedTime(&ms[static_cast<size_t>(i)], e0, e1);
                }
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
                std::sort(ms.begin(), ms.end());
                const double med = ms[ms.size() / 2] * 1e-3;
                if (*m == fbm::Method::zg_paper) zg_median[{n, r}] = med;
                std::printf("%-12s N=%d R=%-5d reps=%d  median=%.6fs min=%.6fs\n", fbm::method_name(*m), n, r, reps,
                            med, ms.front() * 1e-3);
                std::ostringstream row;
                row << fbm::method_name(*m) << ',' << n << ',' << r << ',' << reps << ','
                    << io::detail::format_double(med);
                rows.push_back(row.str());
            }
    }
    for (const auto& row : rows) {  // speedups vs zg_paper (bench.hpp:96-117 semantics)
        std::stringstream ss(row);
        std::string meth, ns, rs, reps_s, med_s;
        std::getline(ss, meth, ',');
        std::getline(ss, ns, ',');
        std::getline(ss, rs, ',');
        std::getline(ss, reps_s, ',');
        std::getline(ss, med_s, ',');
        const auto it = zg_median.find({std::stoi(ns), std::stoi(rs)});
        if (it != zg_median.end())
            std::printf("speedup %-12s N=%s R=%-5s  S=%.4f\n", meth.c_str(), ns.c_str(), rs.c_str(),
                        std::stod(med_s) / it->second);
    }
    if (a.has("--csv")) {
        std::ofstream f(a.kv.at("--csv"));
        if (!f) throw IoError("cannot open for writing: " + a.kv.at("--csv"));
        f << "method,octaves,resolution,repetitions,median_s\n";
        for (const auto& row : rows) f << row << '\n';
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        if (argc < 2) {
            std::cerr << "usage: terrain_b200 {generate|analyze|bench} [--flag value ...]\n";
            return 1;
        }
        Args a;
        a.cmd = argv[1];
        for (int i = 2; i < argc; ++i) {
            const std::string k = argv[i];
            if (k.rfind("--", 0) != 0) throw ValidationError("unexpected argument: " + k);
            if (k == "--normalize") {
                a.flags.push_back(k);
                continue;
            }
            if (i + 1 >= argc) throw ValidationError("missing value for " + k);
            a.kv[k] = argv[++i];
        }
        if (a.cmd == "generate") return run_generate(a);
        if (a.cmd == "analyze") return run_analyze(a);
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
