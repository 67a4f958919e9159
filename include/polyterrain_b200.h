/*
 * polyterrain_b200.h — C-ABI of the B200-native fBm heightmap path.
 *
 * This is the drop-in boundary for the reference's generator API
 * (/root/reference/proj/include/terrain/fbm.hpp:538-685) and the fractal
 * analysis pass after it (terrain/analysis.hpp:213-305).  Every entry point
 * takes plain pointers and sizes; device pointers are CUDA global memory and
 * `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 * Device entry points are asynchronous and stream-ordered unless stated.
 *
 * Status codes mirror terrain/errors.hpp:9-36:
 *   TG_OK          0  success
 *   TG_EVALIDATION 1  terrain::ValidationError   (bad argument / config)
 *   TG_EIO         2  terrain::IoError
 *   TG_ENUMERICAL  3  terrain::NumericalError
 *   TG_EDEVICE     4  CUDA / device failure (std::runtime_error in the C++ mirror)
 * tg_last_error() returns the thread-local message of the last failure.
 *
 * The library has no CPU fallback: every compute entry point launches CUDA
 * kernels built for sm_100a and fails with TG_EDEVICE when no device exists.
 */
#ifndef POLYTERRAIN_B200_H
#define POLYTERRAIN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_ABI_VERSION 1

enum tg_status {
    TG_OK = 0,
    TG_EVALIDATION = 1,
    TG_EIO = 2,
    TG_ENUMERICAL = 3,
    TG_EDEVICE = 4
};

/* terrain::fbm::Method, same order (fbm.hpp:27), plus the paper's third
 * comparison baseline that the reference does not implement:
 * OpenSimplex 2D (2014 geometry: stretch/squish skew, 3 + 1 vertex
 * contributions with (2 - d^2)^4 falloff, 8 gradients, /47) with gradients
 * chosen by the lattice hash instead of a permutation table.  New; parity
 * unpinned (restated oracle only). */
enum tg_method {
    TG_METHOD_ZG_PAPER = 0,
    TG_METHOD_ZG_SEPARABLE = 1,
    TG_METHOD_GENERIC = 2,
    TG_METHOD_PERLIN3 = 3,
    TG_METHOD_PERLIN5 = 4,
    TG_METHOD_OPENSIMPLEX = 5,
    /* Classic permutation-table Perlin gradient noise (BASELINE config 3; the
     * reference deliberately hashes gradient angles instead).
     * New, parity unpinned (restated oracle only).  Per seed: s = seed*K1;
     * P = the permutation of 0..255 sorting key_i = mix(s ^ i*TG_PERM_KI ^
     * TG_LANE_PERM) ascending (ties by i); per octave o an offset
     * t = mix((s + o*K2) ^ TG_LANE_PERM), (ox, oy) = (t & 255, (t >> 8) & 255);
     * corner (ix, iy) takes gradient k = P[(P[(ix + ox) & 255] + iy + oy) & 255]
     * & 7 of the 8 unit vectors at angles k*45 degrees; the cell is the
     * reference's Perlin cell (kernels2d.hpp:163-173) with the fade of
     * `smoothstep` (default S5, "improved noise"). */
    TG_METHOD_PERLIN_PERM = 6
};

/* Lifted caps: the reference caps resolution and extent at
 * 16384 (fbm.hpp:74,547); the B200 path accepts 32768^2 terrains and more. */
#define TG_MAX_RESOLUTION (1LL << 22)
#define TG_MAX_EXTENT (1LL << 17)
#define TG_MAX_OCTAVES 32

/* Lattice output lanes (lattice.hpp:53-54); lane 0 = corner height. */
#define TG_LANE_HEIGHT 0ULL
#define TG_LANE_ANGLE 0xA0761D6478BD642FULL
#define TG_LANE_MAGNITUDE 0xE7037ED1A0B428DBULL
/* OpenSimplex gradient-selection lane (new): index = mix(pack ^ lane) >> 61. */
#define TG_LANE_SIMPLEX 0x8EBC6AF09C88C6E3ULL
/* Permutation-table Perlin lanes (new): table keys and octave offsets. */
#define TG_LANE_PERM 0x5851F42D4C957F2DULL
#define TG_PERM_KI 0xD1B54A32D192ED03ULL
/* 3D key extension (new): pack3 = pack2 + (u64)iz * K5,
 * so iz = 0 reproduces the 2D lattice exactly. */
#define TG_PACK_K5 0xA24BAED4963EE407ULL

/*
 * Mirror of terrain::fbm::FbmConfig (fbm.hpp:49-89) plus the fields the
 * reference cannot express: an explicit smoothstep order and
 * the ZeroSource test hook (fbm.hpp:125-133).
 */
typedef struct tg_fbm_config {
    uint64_t seed;
    int32_t method;            /* enum tg_method */
    int32_t smoothstep;        /* 0 = reference default (S5 for perlin5, else S3); or 3 / 5 */
    int32_t octaves;           /* [1, 32] */
    int32_t threads;           /* validated [0, 256] like the reference, ignored on device */
    int64_t resolution;        /* [1, TG_MAX_RESOLUTION] */
    int64_t base_frequency;    /* cells across the map at octave 0, [1, TG_MAX_RESOLUTION] */
    double frequency_ratio;    /* > 1 */
    double persistence;        /* (0, 1] */
    double base_amplitude;     /* > 0 */
    double gradient_weight;    /* generic kernel only; read when has_gradient_weight != 0 */
    int32_t has_gradient_weight; /* 0 = std::nullopt -> base_amplitude / 100 (fbm.hpp:62-64) */
    int32_t normalize;         /* generate_heightmap/region rescale to [-1, 1] (fbm.hpp:668) */
    int32_t zero_lattice;      /* 1 = ZeroSource: every corner datum is 0 */
    int32_t reserved;
} tg_fbm_config;

/* terrain::fbm::detail::OctaveSpec (fbm.hpp:143-168). */
typedef struct tg_octave_spec {
    double freq;
    double amp;
    int32_t fast;    /* integer cell count dividing the resolution */
    int32_t ppc;     /* pixels per cell, valid when fast */
    int64_t cells;   /* valid when fast */
} tg_octave_spec;

/* terrain::lattice::LatticeKey (lattice.hpp:16-21); iz is the 3D extension. */
typedef struct tg_lattice_key {
    uint64_t seed;
    uint32_t octave;
    uint32_t pad;
    int64_t ix;
    int64_t iy;
} tg_lattice_key;

/* ---- library / host logic (no device needed) ---------------------------- */

int tg_abi_version(void);
const char* tg_last_error(void);
/* FbmConfig::validate (fbm.hpp:71-88) with the lifted caps. */
int tg_fbm_validate(const tg_fbm_config* cfg);
/* detail::octave_spec (fbm.hpp:151-168). */
int tg_fbm_octave_spec(const tg_fbm_config* cfg, int32_t octave, tg_octave_spec* out);
/* The window checks of generate_into_with_source (fbm.hpp:546-558). */
int tg_fbm_validate_window(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t width,
                           int64_t height);
/* Number of visible CUDA devices (0 when none); never launches a kernel. */
int tg_device_count(void);

/* ---- generation (replaces fbm::generate_into_with_source, fbm.hpp:541-628) */

/* Square window [ox, ox+extent) x [oy, oy+extent) into dev_out (n_out must
 * equal extent^2, row-major [y*extent + x], fp32).  Stream-ordered. */
int tg_fbm_generate_f32(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t extent,
                        float* dev_out, uint64_t n_out, void* stream);
/* Rectangular window with a row pitch (elements); used for row bands and
 * chunk grids.  Same per-pixel values as the square form (pure function of
 * the global pixel).  Unlike the square form (fbm.hpp:551-558) the origin
 * need not sit on an octave-0 cell boundary, so shards can regenerate halo
 * rows; |origin| <= 2^40 still applies. */
/* generate_region / generate_heightmap with cfg->normalize (fbm.hpp:638-685):
 * the extent^2 map normalised to [-1, 1] on the device in fp64 (min / max of
 * the samples, -1 + 2 (v - lo) / (hi - lo), fbm.hpp:653) and written to the
 * host doubles; a constant map is returned unchanged with *constant_source = 1.
 * out_min / out_max: the source range.  Synchronous. */
int tg_fbm_generate_normalized_f64_host(const tg_fbm_config* cfg, int64_t ox, int64_t oy,
                                        int32_t extent, double* host_out, uint64_t n_out,
                                        double* out_min, double* out_max, int32_t* constant_source);
/* Per-octave device seconds of a generation over the window (the drop-in's
 * octave_seconds, fbm.hpp:564,624-626): the increments T(k+1) - T(k) of
 * diagnostic launches of the octave prefixes (the fused kernel renders all
 * octaves in one pass).  seconds_out: cfg->octaves entries.  Synchronous. */
int tg_fbm_octave_times(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int32_t extent,
                        double* seconds_out, void* stream);
int tg_fbm_generate_rect_f32(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t width,
                             int64_t height, float* dev_out, int64_t ld, void* stream);
/* A batch of maps that differ only in seed: out[b] is the window for
 * seeds[b] (host array), contiguous maps of width*height.  One launch. */
int tg_fbm_generate_batch_f32(const tg_fbm_config* cfg, const uint64_t* seeds, int32_t n_seeds,
                              int64_t ox, int64_t oy, int64_t width, int64_t height,
                              float* dev_out, void* stream);
/* Drop-in for generate_into(cfg, origin, extent, std::span<double>): host
 * buffer of extent^2 doubles, synchronous.  Device work is fp32; the result
 * is widened on the device and copied back in pipelined row bands. */
int tg_fbm_generate_f64_host(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t extent,
                             double* host_out, uint64_t n_out);
/* Same, fp32 host buffer (pinned or pageable), synchronous. */
int tg_fbm_generate_f32_host(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t extent,
                             float* host_out, uint64_t n_out);

/* texture::render (texture.hpp:50-72) of the full R x R map: kind 0 marble,
 * 1 wood — sin(2*pi*f*phase + gain*noise) fused into the generation store —
 * 2 cloud (noise normalised to [-1, 1]).  Stream-ordered for marble/wood,
 * synchronous for cloud. */
int tg_texture_generate_f32(const tg_fbm_config* cfg, int32_t kind, double gain,
                            double pattern_frequency, float* dev_out, void* stream);

/* 3D fBm volume (new): separable zero-gradient cells
 * (method TG_METHOD_ZG_SEPARABLE only), layout [(z*ny + y)*nx + x]. */
int tg_fbm3d_generate_f32(const tg_fbm_config* cfg, int64_t ox, int64_t oy, int64_t oz,
                          int64_t nx, int64_t ny, int64_t nz, float* dev_out, void* stream);

/* ---- lattice (lattice.hpp:35-83) ------------------------------------------ */

/* out[i] = mix(pack(keys[i]) ^ lane), bit-exact u64.  keys/out are device. */
int tg_lattice_hash(const tg_lattice_key* dev_keys, uint64_t n, uint64_t lane,
                    uint64_t* dev_out, void* stream);
/* out[i] = float(corner_height(keys[i])) rounded to nearest. */
int tg_lattice_height_f32(const tg_lattice_key* dev_keys, uint64_t n, float* dev_out,
                          void* stream);
/* out[2i..2i+1] = corner_unit_gradient (fp32 cos/sin of the hashed angle). */
int tg_lattice_unit_gradient_f32(const tg_lattice_key* dev_keys, uint64_t n, float* dev_out,
                                 void* stream);

/* ---- normalization (fbm.hpp:638-656) -------------------------------------- */

/* Device min/max of n floats; results written to host doubles; synchronous. */
int tg_minmax_f32(const float* dev_map, uint64_t n, double* out_min, double* out_max,
                  void* stream);
/* In-place affine rescale to [-1, 1] with the given source range. */
int tg_rescale_f32(float* dev_map, uint64_t n, double lo, double hi, void* stream);

/* quantize16 (io.hpp:61-65) of a device map into the byte layout of a 16-bit
 * PGM body (big-endian samples) or, with png_rows != 0, of the PNG raw image
 * (filter byte 0 + big-endian samples per row, io.hpp:228-239); dev_out holds
 * height * (2*width [+1]) bytes.  lo/hi: the map's range (tg_minmax_f32).
 * Stream-ordered; the caller writes the header / zlib-compresses on the host. */
int tg_pack16_f32(const float* dev_map, int64_t width, int64_t height, int64_t ld, double lo,
                  double hi, int32_t png_rows, uint8_t* dev_out, void* stream);

/* Gradient-norm (hessian = 0) or Hessian-norm (1) map of a width x height
 * device map (terrain_cli.cpp:148-182: central differences, clamped borders,
 * fp64 arithmetic, fp32 result).  Stream-ordered. */
int tg_norm_map_f32(const float* dev_map, int64_t width, int64_t height, int32_t hessian,
                    float* dev_out, void* stream);

/* ---- fractal analysis (analysis.hpp:213-305; variogram new) --------------- */

/* Upper median (element n/2 of the sorted map, analysis.hpp:244-250) by
 * radix select on the device; synchronous, result to host. */
int tg_median_f32(const float* dev_map, uint64_t n, float* out_median, void* stream);
/* coastline_mask (analysis.hpp:213-240): dev_mask[i] = 1 for land pixels
 * (h >= sea) with a 4-neighbour water pixel; land count to host.
 * Synchronous. */
int tg_coastline_mask(const float* dev_map, int64_t resolution, double sea_level,
                      uint8_t* dev_mask, int64_t* out_land_count, void* stream);
/* Fused coastline + box count (analysis.hpp:213-240 + 269-299): occupied
 * box counts for each size (host arrays), plus coast pixel and land counts.
 * Synchronous. */
int tg_coastline_boxcount(const float* dev_map, int64_t resolution, double sea_level,
                          const int32_t* sizes, int32_t n_sizes, int64_t* out_counts,
                          int64_t* out_coast_pixels, int64_t* out_land_count, void* stream);
/* Row-band form for sharded terrains: `rows` rows of `width` (pitch ld)
 * starting at dev_rows; when has_top / has_bottom the rows just above / below
 * are present in memory (regenerated halos), otherwise the band touches the
 * map edge.  Boxes are anchored at the band's first row, so band starts must
 * be multiples of every box size for the per-band counts to sum to the
 * whole-map counts.  Counts only; the all-land/water checks are the caller's
 * (they are global properties).  Synchronous. */
int tg_coastline_boxcount_band(const float* dev_rows, int64_t width, int64_t rows, int64_t ld,
                               int32_t has_top, int32_t has_bottom, double sea_level,
                               const int32_t* sizes, int32_t n_sizes, int64_t* out_counts,
                               int64_t* out_coast_pixels, int64_t* out_land_count, void* stream);
/* Box counts of an explicit u8 mask (box_count on a CoastlineMask). */
int tg_boxcount_mask(const uint8_t* dev_mask, int64_t resolution, const int32_t* sizes,
                     int32_t n_sizes, int64_t* out_counts, void* stream);
/* Height-difference variogram: for each lag h in lags (host array) and axis
 * (0 = x, 1 = y): sum_sq[2*i+axis] = sum over in-window pairs of
 * (z(p + h e_axis) - z(p))^2 accumulated in fp64, pairs[2*i+axis] = pair
 * count.  Window is width x height with row pitch ld.  Synchronous. */
int tg_variogram_f32(const float* dev_map, int64_t width, int64_t height, int64_t ld,
                     const int32_t* lags, int32_t n_lags, double* out_sum_sq,
                     int64_t* out_pairs, void* stream);

/* Band form: only pairs whose first point lies in the first `pair_rows` rows
 * (the rows below are lookahead regenerated for a row-band shard), so the
 * per-shard sums add up to the whole-map variogram. */
int tg_variogram_band_f32(const float* dev_map, int64_t width, int64_t height, int64_t ld,
                          int64_t pair_rows, const int32_t* lags, int32_t n_lags,
                          double* out_sum_sq, int64_t* out_pairs, void* stream);
/* Local radix-select histogram (2^bits bins of key digit (shift, bits) among
 * keys with (key & mask) == prefix; key = order-preserving u32 of the fp32
 * value) over a strided window, to host.  The per-rank step of a distributed
 * upper median: ranks sum their histograms (NCCL all-reduce) and pick. */
int tg_histogram_f32(const float* dev_rows, int64_t width, int64_t rows, int64_t ld,
                     uint32_t prefix, uint32_t mask, int32_t shift, int32_t bits,
                     uint64_t* out_hist, void* stream);

/* ---- multi-GPU terrain ----------------------------------------- */
/* A large terrain splits into contiguous row bands, one per rank (one process
 * per GPU), generated with no exchange at all (every sample is a function of
 * (config, global pixel), fbm.hpp:7-8); the analysis regenerates a 1-row halo
 * and max_lag lookahead rows locally, and only statistics cross GPUs.
 * Replaces, for a sharded caller, fbm::generate_region (fbm.hpp:658-685) per
 * band + analysis::coastline_mask / box_count (analysis.hpp:213-305) on the
 * whole map; the reference's analogue of ranks are its row-band threads
 * (fbm.hpp:609-622). */

/* Communicator for the statistics all-reduces.  NCCL (over NVLink/NVSwitch on
 * a B200 node): rank 0 calls tg_comm_unique_id and hands the 128 bytes to
 * every rank over any host channel; libnccl.so.2 is loaded at run time.  Host
 * hook: the caller's own transport (MPI, TCP, torch.distributed/gloo) reduces
 * host buffers in place. */
typedef struct tg_comm tg_comm;
typedef int (*tg_allreduce_fn)(void* ctx, void* host_buf, uint64_t count,
                               int32_t dtype /* 0 int64, 1 float64 */,
                               int32_t op /* 0 sum, 1 max */);
int tg_comm_unique_id(uint8_t id_out[128]);
int tg_comm_init_nccl(const uint8_t id[128], int32_t nranks, int32_t rank, tg_comm** out);
int tg_comm_init_host(tg_allreduce_fn fn, void* ctx, int32_t nranks, int32_t rank, tg_comm** out);
int tg_comm_allreduce(tg_comm* comm, void* host_buf, uint64_t count, int32_t dtype, int32_t op);
int tg_comm_destroy(tg_comm* comm);

/* The terrain window and one rank's band of it (rows are global). */
typedef struct {
    int64_t x0, width;      /* columns */
    int64_t y_origin, height;  /* rows [y_origin, y_origin + height) */
    int32_t align;          /* band starts are multiples of align (box sizes, octave-0 cells) */
    int32_t max_lag;        /* largest vertical variogram lag: lookahead rows below a band */
} tg_terrain;
typedef struct {
    int64_t y0, rows;       /* owned rows [y0, y0 + rows), global */
    int64_t halo_top;       /* regenerated rows above (0 or 1) */
    int64_t below;          /* regenerated rows below: max(1, max_lag) clipped to the terrain */
} tg_band;
/* Host only: `world` contiguous bands whose starts are multiples of align,
 * sizes differing by at most align rows. */
int tg_plan_band(const tg_terrain* t, int32_t world, int32_t rank, tg_band* out);

#define TG_MAX_BOX_SIZES 16
#define TG_MAX_LAGS 32
typedef struct {
    double sea_level;       /* upper median of the whole terrain (analysis.hpp:244-250) or given */
    double land_fraction;
    int64_t land_pixels, coast_pixels;
    int32_t n_sizes, n_lags;
    int64_t counts[TG_MAX_BOX_SIZES];  /* box counts, whole terrain */
    double d_box, k_box, r2_box;       /* D = -slope of log N vs log eps (analysis.hpp:299-305) */
    double sum_sq[TG_MAX_LAGS][2];     /* variogram sums per lag, axis (0 x, 1 y) */
    int64_t pairs[TG_MAX_LAGS][2];
    double gamma[TG_MAX_LAGS];         /* both axes pooled: sum / (2 pairs) */
    double hurst, d_variogram;         /* slope / 2 of log gamma vs log h; D = 3 - H */
} tg_terrain_stats;

/* Product path: generate this rank's band (+ halo / lookahead) on the
 * current device, then the distributed statistics (sea level by a 3-pass
 * radix select over all-reduced histograms unless *sea_level is given).
 * Collective: every rank calls it with the same terrain, sizes and lags. */
int tg_terrain_stats_band(const tg_fbm_config* cfg, const tg_terrain* t, const tg_band* band,
                          const int32_t* sizes, int32_t n_sizes, const int32_t* lags,
                          int32_t n_lags, const double* sea_level, tg_comm* comm,
                          tg_terrain_stats* out, void* stream);

/* The same product path over a band buffer the caller owns: dev_band_buf
 * holds (halo_top + rows + below) rows of width floats (pitch = width), its
 * first row being global row y0 - halo_top.  owned_ready != 0: the caller has
 * already generated the owned rows into it (at row offset halo_top, e.g. with
 * tg_fbm_generate_rect_f32 — the terrain's own generation step), and only the
 * halo row above and the lookahead rows below are regenerated here (a single
 * band regenerates nothing).  owned_ready == 0: every row is generated here. */
int tg_terrain_stats_band_buf(const tg_fbm_config* cfg, const tg_terrain* t, const tg_band* band,
                              float* dev_band_buf, int32_t owned_ready, const int32_t* sizes,
                              int32_t n_sizes, const int32_t* lags, int32_t n_lags,
                              const double* sea_level, tg_comm* comm, tg_terrain_stats* out,
                              void* stream);

/* The same driver over caller-supplied band operations — the test hook of the
 * host logic (the reference's Source policy plays this role for generation,
 * fbm.hpp:110-133).  The product path above never uses it. */
typedef struct {
    void* ctx;
    int (*generate)(void* ctx, const tg_band* band);
    int (*histogram)(void* ctx, uint32_t prefix, uint32_t mask, int32_t shift, int32_t bits,
                     uint64_t* out_hist);
    int (*boxcount)(void* ctx, double sea_level, const int32_t* sizes, int32_t n_sizes,
                    int64_t* out_counts, int64_t* out_coast, int64_t* out_land);
    int (*variogram)(void* ctx, const int32_t* lags, int32_t n_lags, double* out_sum_sq,
                     int64_t* out_pairs);
} tg_band_ops;
int tg_terrain_stats_ops(const tg_terrain* t, const tg_band* band, const int32_t* sizes,
                         int32_t n_sizes, const int32_t* lags, int32_t n_lags,
                         const double* sea_level, tg_comm* comm, const tg_band_ops* ops,
                         tg_terrain_stats* out);

/* ---- measurement helpers ---------------------------------------------------- */

/* FP32 FFMA-chain peak on the current device (TFLOP/s), for the roofline
 * denominator; synchronous. */
int tg_measure_ffma_peak(double* out_tflops, double* out_ms);

#ifdef __cplusplus
}
#endif

#endif /* POLYTERRAIN_B200_H */
