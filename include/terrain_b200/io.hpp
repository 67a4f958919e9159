#pragma once

// terrain_b200/io.hpp — 16-bit PGM / PNG export of device heightmaps
// (SURVEY §8f row 1), byte-identical to the reference writers
// (/root/reference/proj/include/terrain/io.hpp:91-111 write_pgm16,
// 203-257 write_png16) on the same (fp32-widened) heights: the range and the
// quantize16 packing run on the device (tg_minmax_f32, tg_pack16_f32); the
// header, CRCs and zlib (level 9, io.hpp:245-247) stay on the host.
// Link with -lz.

#include <zlib.h>

#include <cstdint>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "fbm.hpp"

namespace terrain_b200::io {

namespace detail {
inline std::string format_double(double v) {  // io.hpp:30-34
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return buf;
}
inline void push_be32(std::vector<unsigned char>& out, std::uint32_t v) {
    out.push_back(static_cast<unsigned char>(v >> 24));
    out.push_back(static_cast<unsigned char>(v >> 16));
    out.push_back(static_cast<unsigned char>(v >> 8));
    out.push_back(static_cast<unsigned char>(v));
}
inline void chunk(std::vector<unsigned char>& file, const char type[5], const std::vector<unsigned char>& data) {
    std::vector<unsigned char> buf;
    push_be32(buf, static_cast<std::uint32_t>(data.size()));
    buf.insert(buf.end(), type, type + 4);
    buf.insert(buf.end(), data.begin(), data.end());
    const auto crc = ::crc32(0L, buf.data() + 4, static_cast<uInt>(buf.size() - 4));
    push_be32(buf, static_cast<std::uint32_t>(crc));
    file.insert(file.end(), buf.begin(), buf.end());
}
// range + device packing of a width x height window (pitch ld)
inline std::vector<unsigned char> pack(const float* dev_map, int width, int height, long long ld, bool png,
                                       double* lo, double* hi) {
    if (width < 1 || height < 1) throw ValidationError("write: empty grid");
    check(tg_minmax_f32(dev_map, static_cast<std::uint64_t>(ld) * (height - 1) + width, lo, hi, nullptr));
    if (ld != width) {  // range of the window only
        // the row pitch covers out-of-window samples: take the range per row
        double l = 0, h = 0;
        for (int y = 0; y < height; ++y) {
            double a, b;
            check(tg_minmax_f32(dev_map + static_cast<long long>(y) * ld, width, &a, &b, nullptr));
            l = y == 0 ? a : (a < l ? a : l);
            h = y == 0 ? b : (b > h ? b : h);
        }
        *lo = l;
        *hi = h;
    }
    const std::size_t bytes = static_cast<std::size_t>(height) * (2 * static_cast<std::size_t>(width) + (png ? 1 : 0));
    unsigned char* dev = nullptr;
    if (cudaMalloc(&dev, bytes) != cudaSuccess) throw DeviceError("write: cudaMalloc failed");
    std::vector<unsigned char> host(bytes);
    const int st = tg_pack16_f32(dev_map, width, height, ld, *lo, *hi, png ? 1 : 0, dev, nullptr);
    const cudaError_t e = st == TG_OK ? cudaMemcpy(host.data(), dev, bytes, cudaMemcpyDeviceToHost) : cudaSuccess;
    cudaFree(dev);
    check(st);
    if (e != cudaSuccess) throw DeviceError("write: copy failed");
    return host;
}
}  // namespace detail

// write_pgm16 (io.hpp:91-106) of a device map: whole file as bytes.
inline std::vector<unsigned char> encode_pgm16(const float* dev_map, int width, int height, long long ld) {
    double lo, hi;
    const auto body = detail::pack(dev_map, width, height, ld, false, &lo, &hi);
    const std::string head = "P5\n# hmin=" + detail::format_double(lo) + " hmax=" + detail::format_double(hi) +
                             "\n" + std::to_string(width) + " " + std::to_string(height) + "\n65535\n";
    std::vector<unsigned char> file(head.begin(), head.end());
    file.insert(file.end(), body.begin(), body.end());
    return file;
}

// write_png16 (io.hpp:203-250) of a device map: whole file as bytes.
inline std::vector<unsigned char> encode_png16(const float* dev_map, int width, int height, long long ld) {
    double lo, hi;
    const auto raw = detail::pack(dev_map, width, height, ld, true, &lo, &hi);
    static const unsigned char signature[8] = {137, 80, 78, 71, 13, 10, 26, 10};
    std::vector<unsigned char> file(signature, signature + 8);
    std::vector<unsigned char> ihdr;
    detail::push_be32(ihdr, static_cast<std::uint32_t>(width));
    detail::push_be32(ihdr, static_cast<std::uint32_t>(height));
    ihdr.insert(ihdr.end(), {16, 0, 0, 0, 0});
    detail::chunk(file, "IHDR", ihdr);
    const std::string note = "hmin=" + detail::format_double(lo) + " hmax=" + detail::format_double(hi);
    std::vector<unsigned char> text;
    const char* keyword = "Comment";
    text.insert(text.end(), keyword, keyword + 8);
    text.insert(text.end(), note.begin(), note.end());
    detail::chunk(file, "tEXt", text);
    uLongf n = ::compressBound(static_cast<uLong>(raw.size()));
    std::vector<unsigned char> z(n);
    if (::compress2(z.data(), &n, raw.data(), static_cast<uLong>(raw.size()), 9) != Z_OK)
        throw IoError("write_png16: zlib compression failed");
    z.resize(n);
    detail::chunk(file, "IDAT", z);
    detail::chunk(file, "IEND", {});
    return file;
}

inline void write_file(const std::string& path, const std::vector<unsigned char>& bytes) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot open for writing: " + path);
    out.write(reinterpret_cast<const char*>(bytes.data()), static_cast<std::streamsize>(bytes.size()));
    if (!out) throw IoError("write failed: " + path);
}

inline void write_pgm16(const std::string& path, const float* dev_map, int width, int height) {
    write_file(path, encode_pgm16(dev_map, width, height, width));
}
inline void write_png16(const std::string& path, const float* dev_map, int width, int height) {
    write_file(path, encode_png16(dev_map, width, height, width));
}

// 16-bit P5 PGM reader (the reference's read_pgm16, io.hpp:113-160): header
// tokens (width, height, maxval = 65535) with '#' comment lines anywhere, the
// "# hmin=... hmax=..." comment giving the height range (default [0, 1]),
// one whitespace byte, then big-endian samples.
struct Image16 {
    int width = 0, height = 0;
    double hmin = 0.0, hmax = 1.0;
    std::vector<std::uint16_t> samples;
    // sample -> height (io.hpp:162-168)
    double height_of(std::uint32_t s) const { return hmin + static_cast<double>(s) / 65535.0 * (hmax - hmin); }
};

inline Image16 read_pgm16(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot open for reading: " + path);
    std::string magic;
    in >> magic;
    if (magic != "P5") throw IoError("read_pgm16: not a P5 PGM stream");
    Image16 img;
    int field[3] = {0, 0, 0};
    for (int got = 0; got < 3;) {
        in >> std::ws;
        if (in.peek() == '#') {
            std::string line;
            std::getline(in, line);
            double lo, hi;
            if (std::sscanf(line.c_str(), "# hmin=%lf hmax=%lf", &lo, &hi) == 2) {
                img.hmin = lo;
                img.hmax = hi;
            }
            continue;
        }
        if (!(in >> field[got++])) throw IoError("read_pgm16: malformed header");
    }
    img.width = field[0];
    img.height = field[1];
    if (img.width < 1 || img.height < 1) throw IoError("read_pgm16: bad dimensions");
    if (field[2] != 65535) throw IoError("read_pgm16: expected 16-bit maxval 65535");
    in.get();
    const std::size_t n = static_cast<std::size_t>(img.width) * static_cast<std::size_t>(img.height);
    std::vector<unsigned char> raw(2 * n);
    in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
    if (in.gcount() != static_cast<std::streamsize>(raw.size())) throw IoError("read_pgm16: truncated pixel data");
    img.samples.resize(n);
    for (std::size_t i = 0; i < n; ++i) img.samples[i] = static_cast<std::uint16_t>(raw[2 * i] << 8 | raw[2 * i + 1]);
    return img;
}

}  // namespace terrain_b200::io
