// terrain.cpp — multi-GPU terrain statistics behind the C-ABI:
// row-band planning, the collective statistics driver, and its communicators
// (NCCL loaded at run time, or a caller-supplied host all-reduce).
//
// A terrain of width x height splits into contiguous row bands, one per rank;
// every sample is a function of (config, global pixel) (fbm.hpp:7-8), so the
// bands are generated independently (fbm::generate_region, fbm.hpp:658-685,
// per band) and only statistics cross GPUs:
//   * the upper-median sea level (analysis.hpp:244-250): a 3-pass radix select
//     whose per-rank digit histograms are summed (11 / 11 / 10-bit digits of
//     the order-preserving u32 key of the fp32 sample);
//   * the box counts (analysis.hpp:269-299): boxes anchored at band starts
//     that are multiples of every box size, so per-band counts add up, plus
//     the land and coast pixel counts;
//   * the variogram sums and pair counts (lookahead rows regenerated below
//     each band so vertical pairs across band edges are counted once).
// The fits (analysis.hpp:29-63) run on the reduced statistics on every rank.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/polyterrain_b200.h"
#include "select.h"

namespace tg {
int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* where);
int check_device();
}  // namespace tg

struct tg_comm {
    int kind = 0;  // 0 host hook, 1 NCCL
    int nranks = 1, rank = 0;
    tg_allreduce_fn fn = nullptr;
    void* ctx = nullptr;
    ncclComm_t nc = nullptr;
    int device = 0;
    cudaStream_t st = nullptr;
    void* dbuf = nullptr;  // device staging for NCCL reductions of host buffers
    size_t dbytes = 0;
};

namespace {

// ---- NCCL, loaded at run time (the library has no link-time dependency on it)
struct Nccl {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    bool ok = false;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        n.init_rank = reinterpret_cast<decltype(n.init_rank)>(dlsym(h, "ncclCommInitRank"));
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
        n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "ncclCommDestroy"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
        n.ok = n.get_unique_id && n.init_rank && n.all_reduce && n.destroy && n.error_string;
    });
    return n;
}

int nccl_fail(ncclResult_t r, const char* where) {
    const std::string m = std::string(where) + ": " + nccl().error_string(r);
    return tg::set_error(TG_EDEVICE, m.c_str());
}

// Upper-median radix select digits (shard.py / analysis.cu share them).
constexpr int kDigits[3][2] = {{21, 11}, {10, 11}, {0, 10}};

double float_from_key(uint32_t k) {
    const uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    float f;
    std::memcpy(&f, &b, 4);
    return static_cast<double>(f);
}

// OLS of analysis.hpp:29-63 on a handful of points.
bool linear_fit(const std::vector<double>& xs, const std::vector<double>& ys, double* slope, double* icept,
                double* r2) {
    const size_t n = xs.size();
    if (n < 2 || ys.size() != n) return false;
    double mx = 0, my = 0;
    for (size_t i = 0; i < n; ++i) {
        mx += xs[i];
        my += ys[i];
    }
    mx /= n;
    my /= n;
    double sxx = 0, sxy = 0, syy = 0;
    for (size_t i = 0; i < n; ++i) {
        sxx += (xs[i] - mx) * (xs[i] - mx);
        sxy += (xs[i] - mx) * (ys[i] - my);
        syy += (ys[i] - my) * (ys[i] - my);
    }
    if (sxx == 0.0) return false;
    *slope = sxy / sxx;
    *icept = my - *slope * mx;
    if (syy == 0.0) {
        *r2 = 1.0;
        return true;
    }
    double ssr = 0;
    for (size_t i = 0; i < n; ++i) {
        const double e = ys[i] - (*slope * xs[i] + *icept);
        ssr += e * e;
    }
    *r2 = 1.0 - ssr / syy;
    return true;
}

int allreduce(tg_comm* c, void* buf, uint64_t count, int dtype, int op) {
    // one rank: the reduction is the identity (the driver skips the six
    // host -> device -> NCCL -> host round trips of a one-band terrain;
    // tg_comm_allreduce itself still reduces on a 1-rank communicator)
    if (!c || count == 0 || c->nranks <= 1) return TG_OK;
    return tg_comm_allreduce(c, buf, count, dtype, op);
}

// ---- device band operations (the product path) -------------------------------
struct DeviceBand {
    const tg_fbm_config* cfg;
    const tg_terrain* t;
    const tg_band* b;
    float* buf = nullptr;  // gen rows x width, contiguous
    cudaStream_t st;
    tg::SelectCache sel;   // candidate keys kept by the first median pass
    float* ext = nullptr;  // caller's band buffer (tg_terrain_stats_band_buf)
    bool owned_ready = false;  // ... whose owned rows the caller already generated

    const float* owned() const { return buf + b->halo_top * t->width; }
    bool last() const { return b->y0 - t->y_origin + b->rows >= t->height; }
};

// One grow-only band buffer per device and host thread (bands are regenerated
// on every call; the allocation is not).
float* band_buffer(size_t bytes, int* err) {
    struct Cache {
        int dev = -1;
        void* p = nullptr;
        size_t n = 0;
    };
    thread_local Cache cache[16];
    int dev = 0;
    cudaGetDevice(&dev);
    Cache& c = cache[dev & 15];
    if (c.dev != dev || c.n < bytes) {
        if (c.p && c.dev == dev) cudaFree(c.p);
        c.p = nullptr;
        const cudaError_t e = cudaMalloc(&c.p, bytes);
        if (e != cudaSuccess) {
            *err = tg::set_cuda_error(e, "terrain band buffer");
            c.n = 0;
            return nullptr;
        }
        c.dev = dev;
        c.n = bytes;
    }
    return static_cast<float*>(c.p);
}

int dev_generate(void* ctx, const tg_band* b) {
    auto* d = static_cast<DeviceBand*>(ctx);
    const int64_t gen_rows = b->halo_top + b->rows + b->below;
    const int64_t W = d->t->width;
    if (d->ext && d->owned_ready) {  // regenerate only the halo row above and the lookahead rows below
        d->buf = d->ext;
        if (b->halo_top)
            if (int st = tg_fbm_generate_rect_f32(d->cfg, d->t->x0, b->y0 - b->halo_top, W, b->halo_top, d->buf, W,
                                                  d->st))
                return st;
        if (b->below)
            return tg_fbm_generate_rect_f32(d->cfg, d->t->x0, b->y0 + b->rows, W, b->below,
                                            d->buf + (b->halo_top + b->rows) * W, W, d->st);
        return TG_OK;
    }
    if (d->ext) {
        d->buf = d->ext;
        return tg_fbm_generate_rect_f32(d->cfg, d->t->x0, b->y0 - b->halo_top, W, gen_rows, d->buf, W, d->st);
    }
    int err = TG_OK;
    d->buf = band_buffer(static_cast<size_t>(gen_rows) * static_cast<size_t>(d->t->width) * sizeof(float), &err);
    if (!d->buf) return err;
    return tg_fbm_generate_rect_f32(d->cfg, d->t->x0, b->y0 - b->halo_top, d->t->width, gen_rows, d->buf,
                                    d->t->width, d->st);
}
int dev_histogram(void* ctx, uint32_t prefix, uint32_t mask, int32_t shift, int32_t bits, uint64_t* hist) {
    auto* d = static_cast<DeviceBand*>(ctx);
    if (bits < 1 || bits > 11 || shift < 0 || shift + bits > 32)
        return tg::set_error(TG_EVALIDATION, "histogram: bad arguments");
    return tg::select_hist(d->owned(), d->t->width, d->b->rows, d->t->width, prefix, mask, shift, bits, hist, &d->sel,
                           d->st);
}
int dev_boxcount(void* ctx, double sea, const int32_t* sizes, int32_t n, int64_t* counts, int64_t* coast,
                 int64_t* land) {
    auto* d = static_cast<DeviceBand*>(ctx);
    return tg_coastline_boxcount_band(d->owned(), d->t->width, d->b->rows, d->t->width,
                                      d->b->halo_top ? 1 : 0, d->last() ? 0 : 1, sea, sizes, n, counts, coast,
                                      land, d->st);
}
int dev_variogram(void* ctx, const int32_t* lags, int32_t n, double* ss, int64_t* pairs) {
    auto* d = static_cast<DeviceBand*>(ctx);
    return tg_variogram_band_f32(d->owned(), d->t->width, d->b->rows + d->b->below, d->t->width, d->b->rows, lags,
                                 n, ss, pairs, d->st);
}

}  // namespace

extern "C" {

int tg_comm_unique_id(uint8_t id_out[128]) {
    if (!id_out) return tg::set_error(TG_EVALIDATION, "comm: null id");
    const Nccl& n = nccl();
    if (!n.ok) return tg::set_error(TG_EDEVICE, "comm: libnccl.so.2 not found");
    ncclUniqueId id;
    const ncclResult_t r = n.get_unique_id(&id);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, sizeof(id.internal));
    return TG_OK;
}

int tg_comm_init_nccl(const uint8_t id[128], int32_t nranks, int32_t rank, tg_comm** out) {
    if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
        return tg::set_error(TG_EVALIDATION, "comm: bad nranks / rank");
    if (int st = tg::check_device()) return st;
    const Nccl& n = nccl();
    if (!n.ok) return tg::set_error(TG_EDEVICE, "comm: libnccl.so.2 not found");
    auto* c = new tg_comm;
    c->kind = 1;
    c->nranks = nranks;
    c->rank = rank;
    cudaGetDevice(&c->device);
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    ncclResult_t r = n.init_rank(&c->nc, nranks, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    cudaError_t e = cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking);
    if (e == cudaSuccess) {
        c->dbytes = 64 * 1024;
        e = cudaMalloc(&c->dbuf, c->dbytes);
    }
    if (e != cudaSuccess) {
        tg_comm_destroy(c);
        return tg::set_cuda_error(e, "comm setup");
    }
    *out = c;
    return TG_OK;
}

int tg_comm_init_host(tg_allreduce_fn fn, void* ctx, int32_t nranks, int32_t rank, tg_comm** out) {
    if (!out || nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !fn))
        return tg::set_error(TG_EVALIDATION, "comm: bad host communicator");
    auto* c = new tg_comm;
    c->kind = 0;
    c->fn = fn;
    c->ctx = ctx;
    c->nranks = nranks;
    c->rank = rank;
    *out = c;
    return TG_OK;
}

int tg_comm_allreduce(tg_comm* c, void* buf, uint64_t count, int32_t dtype, int32_t op) {
    if (!c || (!buf && count)) return tg::set_error(TG_EVALIDATION, "comm: null argument");
    if ((dtype != 0 && dtype != 1) || (op != 0 && op != 1)) return tg::set_error(TG_EVALIDATION, "comm: bad dtype / op");
    if (count == 0 || (c->kind == 0 && c->nranks <= 1)) return TG_OK;  // (a 1-rank NCCL comm still reduces)
    if (c->kind == 0) {
        const int r = c->fn(c->ctx, buf, count, dtype, op);
        return r == 0 ? TG_OK : tg::set_error(TG_EDEVICE, "comm: host all-reduce failed");
    }
    const size_t bytes = count * 8;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != c->device) cudaSetDevice(c->device);
    cudaError_t e = cudaSuccess;
    if (bytes > c->dbytes) {
        cudaFree(c->dbuf);
        c->dbuf = nullptr;
        e = cudaMalloc(&c->dbuf, bytes);
        c->dbytes = e == cudaSuccess ? bytes : 0;
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->dbuf, buf, bytes, cudaMemcpyHostToDevice, c->st);
    int status = TG_OK;
    if (e == cudaSuccess) {
        const ncclResult_t r = nccl().all_reduce(c->dbuf, c->dbuf, count, dtype == 0 ? ncclInt64 : ncclFloat64,
                                                 op == 0 ? ncclSum : ncclMax, c->nc, c->st);
        if (r != ncclSuccess) status = nccl_fail(r, "ncclAllReduce");
    }
    if (e == cudaSuccess && status == TG_OK) e = cudaMemcpyAsync(buf, c->dbuf, bytes, cudaMemcpyDeviceToHost, c->st);
    if (e == cudaSuccess && status == TG_OK) e = cudaStreamSynchronize(c->st);
    if (dev != c->device) cudaSetDevice(dev);
    if (status != TG_OK) return status;
    if (e != cudaSuccess) return tg::set_cuda_error(e, "comm all-reduce");
    return TG_OK;
}

int tg_comm_destroy(tg_comm* c) {
    if (!c) return TG_OK;
    if (c->kind == 1) {
        if (c->nc) nccl().destroy(c->nc);
        if (c->dbuf) cudaFree(c->dbuf);
        if (c->st) cudaStreamDestroy(c->st);
    }
    delete c;
    return TG_OK;
}

int tg_plan_band(const tg_terrain* t, int32_t world, int32_t rank, tg_band* out) {
    if (!t || !out) return tg::set_error(TG_EVALIDATION, "plan_band: null argument");
    if (world < 1 || rank < 0 || rank >= world) return tg::set_error(TG_EVALIDATION, "plan_band: bad rank/world");
    if (t->align < 1 || t->width < 1 || t->height < 1 || t->max_lag < 0)
        return tg::set_error(TG_EVALIDATION, "plan_band: bad terrain");
    if (t->height % t->align != 0)
        return tg::set_error(TG_EVALIDATION, "plan_band: height must be a multiple of the alignment");
    const int64_t units = t->height / t->align;
    if (units < world) return tg::set_error(TG_EVALIDATION, "plan_band: fewer aligned row blocks than ranks");
    const int64_t u0 = units * rank / world, u1 = units * (rank + 1) / world;
    const int64_t y0 = u0 * t->align, y1 = u1 * t->align;
    out->y0 = t->y_origin + y0;
    out->rows = y1 - y0;
    out->halo_top = y0 > 0 ? 1 : 0;
    out->below = std::min<int64_t>(std::max<int64_t>(1, t->max_lag), t->height - y1);
    return TG_OK;
}

int tg_terrain_stats_ops(const tg_terrain* t, const tg_band* b, const int32_t* sizes, int32_t n_sizes,
                         const int32_t* lags, int32_t n_lags, const double* sea_level, tg_comm* comm,
                         const tg_band_ops* ops, tg_terrain_stats* out) {
    if (!t || !b || !sizes || !lags || !ops || !out || !ops->generate || !ops->histogram || !ops->boxcount ||
        !ops->variogram)
        return tg::set_error(TG_EVALIDATION, "terrain_stats: null argument");
    if (n_sizes < 2 || n_sizes > TG_MAX_BOX_SIZES || n_lags < 1 || n_lags > TG_MAX_LAGS)
        return tg::set_error(TG_EVALIDATION, "terrain_stats: 2..16 box sizes and 1..32 lags");
    const int64_t local_y0 = b->y0 - t->y_origin;
    const bool last = local_y0 + b->rows >= t->height;
    for (int i = 0; i < n_sizes; ++i) {
        if (sizes[i] < 1) return tg::set_error(TG_EVALIDATION, "terrain_stats: box sizes must be >= 1");
        if (local_y0 % sizes[i] != 0 || (b->rows % sizes[i] != 0 && !last))
            return tg::set_error(TG_EVALIDATION, "terrain_stats: band starts/ends must be multiples of every box size");
    }
    int64_t hmax = 0;
    for (int i = 0; i < n_lags; ++i) {
        if (lags[i] < 1) return tg::set_error(TG_EVALIDATION, "terrain_stats: lags must be >= 1");
        hmax = std::max<int64_t>(hmax, lags[i]);
    }
    // vertical pairs need max(lags) rows below the band, or every row left in the terrain
    if (hmax > b->below && b->below < t->height - (local_y0 + b->rows))
        return tg::set_error(TG_EVALIDATION,
                             "terrain_stats: a variogram lag exceeds the band's regenerated lookahead (plan_band max_lag)");
    std::memset(out, 0, sizeof(*out));
    out->n_sizes = n_sizes;
    out->n_lags = n_lags;
    if (int st = ops->generate(ops->ctx, b)) return st;
    const int64_t total = t->width * t->height;
    // sea level: upper median (element total/2 of the sorted union)
    if (sea_level) {
        out->sea_level = *sea_level;
    } else {
        uint32_t prefix = 0, mask = 0;
        int64_t k = total / 2;
        std::vector<uint64_t> h;
        for (const auto& dg : kDigits) {
            const int shift = dg[0], bits = dg[1];
            h.assign(size_t(1) << bits, 0);
            if (int st = ops->histogram(ops->ctx, prefix, mask, shift, bits, h.data())) return st;
            if (int st = allreduce(comm, h.data(), h.size(), 0, 0)) return st;
            int64_t c = 0;
            size_t d = 0;
            for (; d < h.size(); ++d) {
                if (c + static_cast<int64_t>(h[d]) > k) break;
                c += static_cast<int64_t>(h[d]);
            }
            if (d == h.size()) return tg::set_error(TG_ENUMERICAL, "terrain_stats: median select out of range");
            k -= c;
            prefix |= static_cast<uint32_t>(d) << shift;
            mask |= ((1u << bits) - 1u) << shift;
        }
        out->sea_level = float_from_key(prefix);
    }
    // coastline + box counts
    int64_t red[TG_MAX_BOX_SIZES + 2] = {};
    if (int st = ops->boxcount(ops->ctx, out->sea_level, sizes, n_sizes, red, red + n_sizes, red + n_sizes + 1))
        return st;
    if (int st = allreduce(comm, red, n_sizes + 2, 0, 0)) return st;
    for (int i = 0; i < n_sizes; ++i) out->counts[i] = red[i];
    out->coast_pixels = red[n_sizes];
    out->land_pixels = red[n_sizes + 1];
    if (out->land_pixels == 0 || out->land_pixels == total)
        return tg::set_error(TG_EVALIDATION, "coastline_mask: map is entirely land or entirely water");
    out->land_fraction = static_cast<double>(out->land_pixels) / static_cast<double>(total);
    // variogram
    double ss[2 * TG_MAX_LAGS] = {};
    int64_t pr[2 * TG_MAX_LAGS] = {};
    if (int st = ops->variogram(ops->ctx, lags, n_lags, ss, pr)) return st;
    if (int st = allreduce(comm, ss, 2 * n_lags, 1, 0)) return st;
    if (int st = allreduce(comm, pr, 2 * n_lags, 0, 0)) return st;
    // fits (analysis.hpp:29-63, 299-305)
    std::vector<double> lx, ly;
    for (int i = 0; i < n_sizes; ++i) {
        if (out->counts[i] <= 0) return tg::set_error(TG_ENUMERICAL, "terrain_stats: empty box count");
        lx.push_back(std::log(static_cast<double>(sizes[i])));
        ly.push_back(std::log(static_cast<double>(out->counts[i])));
    }
    double slope, icept, r2;
    if (!linear_fit(lx, ly, &slope, &icept, &r2))
        return tg::set_error(TG_EVALIDATION, "linear_fit: x values are all equal");
    out->d_box = -slope;
    out->k_box = std::exp(icept);
    out->r2_box = r2;
    lx.clear();
    ly.clear();
    for (int i = 0; i < n_lags; ++i) {
        out->sum_sq[i][0] = ss[2 * i];
        out->sum_sq[i][1] = ss[2 * i + 1];
        out->pairs[i][0] = pr[2 * i];
        out->pairs[i][1] = pr[2 * i + 1];
        const int64_t p = pr[2 * i] + pr[2 * i + 1];
        out->gamma[i] = p > 0 ? (ss[2 * i] + ss[2 * i + 1]) / (2.0 * static_cast<double>(p)) : NAN;
        if (out->gamma[i] > 0) {
            lx.push_back(std::log(static_cast<double>(lags[i])));
            ly.push_back(std::log(out->gamma[i]));
        }
    }
    if (linear_fit(lx, ly, &slope, &icept, &r2)) {
        out->hurst = slope / 2.0;
        out->d_variogram = 3.0 - out->hurst;
    } else {
        out->hurst = out->d_variogram = NAN;
    }
    return TG_OK;
}

int tg_terrain_stats_band(const tg_fbm_config* cfg, const tg_terrain* t, const tg_band* b, const int32_t* sizes,
                          int32_t n_sizes, const int32_t* lags, int32_t n_lags, const double* sea_level,
                          tg_comm* comm, tg_terrain_stats* out, void* stream) {
    if (!cfg || !t || !b) return tg::set_error(TG_EVALIDATION, "terrain_stats: null argument");
    if (int st = tg::check_device()) return st;
    DeviceBand d{cfg, t, b, nullptr, static_cast<cudaStream_t>(stream)};
    // one band: the local median is the global one (narrow candidate window);
    // several: the global median's local rank is unknown (wide window)
    d.sel.delta = comm && comm->nranks > 1 ? 0.05 : 0.005;
    tg_band_ops ops{&d, dev_generate, dev_histogram, dev_boxcount, dev_variogram};
    const int st = tg_terrain_stats_ops(t, b, sizes, n_sizes, lags, n_lags, sea_level, comm, &ops, out);
    tg::select_cache_free(&d.sel, d.st);
    return st;
}

int tg_terrain_stats_band_buf(const tg_fbm_config* cfg, const tg_terrain* t, const tg_band* b, float* dev_band_buf,
                              int32_t owned_ready, const int32_t* sizes, int32_t n_sizes, const int32_t* lags,
                              int32_t n_lags, const double* sea_level, tg_comm* comm, tg_terrain_stats* out,
                              void* stream) {
    if (!cfg || !t || !b || !dev_band_buf) return tg::set_error(TG_EVALIDATION, "terrain_stats: null argument");
    if (int st = tg::check_device()) return st;
    DeviceBand d{cfg, t, b, nullptr, static_cast<cudaStream_t>(stream)};
    d.sel.delta = comm && comm->nranks > 1 ? 0.05 : 0.005;
    d.ext = dev_band_buf;
    d.owned_ready = owned_ready != 0;
    tg_band_ops ops{&d, dev_generate, dev_histogram, dev_boxcount, dev_variogram};
    const int st = tg_terrain_stats_ops(t, b, sizes, n_sizes, lags, n_lags, sea_level, comm, &ops, out);
    tg::select_cache_free(&d.sel, d.st);
    return st;
}

}  // extern "C"
