/*
 * pf_b200.h — C ABI of the B200-native Online Patching hot path.
 *
 * Every entry point takes plain pointers, sizes and a cudaStream_t passed as
 * `void*` (NULL = legacy default stream).  No torch types cross this ABI, no
 * C++ exception crosses it, and it never allocates memory that it returns:
 * outputs are caller-allocated device (or host, where stated) buffers.
 * Errors are an int status (enum pf_status) plus a thread-local message from
 * pf_last_error().  All launches are asynchronous on the given stream; no
 * entry point synchronises the device unless its comment says so.
 *
 * The reference interface each entry point replaces is cited as
 * `pkg/<module>.py:<line>` = /root/reference/pkg/src/patchforge/<module>.py.
 */
#ifndef PF_B200_H
#define PF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_ABI_VERSION 3
#define PF_MAX_LEVELS 12
#define PF_MAX_MPPS 8
#define PF_MAX_CROPS 16

/* Status codes; the Python shim maps them onto the reference's exception
 * classes (pkg/store.py:46-67, pkg/foreground.py:33, pkg/sampler.py:26-31). */
enum pf_status {
    PF_OK = 0,
    PF_ERR_INVALID_ARG = 1,      /* ValueError */
    PF_ERR_OUT_OF_BOUNDS = 2,    /* store.OutOfBoundsError (pkg/store.py:66) */
    PF_ERR_INTEGRITY = 3,        /* store.IntegrityError (pkg/store.py:54) */
    PF_ERR_EXHAUSTED = 4,        /* sampler.ExhaustedAttemptsError (pkg/sampler.py:26) */
    PF_ERR_NO_SAMPLABLE = 5,     /* sampler.NoSamplableSlideError (pkg/sampler.py:30) */
    PF_ERR_CUDA = 6,             /* CUDA runtime failure */
    PF_ERR_EMPTY_FOREGROUND = 7, /* foreground.EmptyForegroundError (pkg/foreground.py:33) */
    PF_ERR_CAPACITY = 8,         /* caller buffer too small; required sizes were written */
    PF_ERR_INTERNAL = 9,
    PF_ERR_DECODE = 10           /* store.DecodeError (pkg/store.py:62) */
};

/* Output element types for the normalising epilogues. */
enum pf_dtype { PF_U8 = 0, PF_F32 = 1, PF_BF16 = 2 };

/* Output layouts for pf_read_regions.  OR with PF_SKIP_PASSTHROUGH to leave
 * the output of specs with side == out_size untouched (the multi-crop kernel
 * reads those straight from the pyramid). */
enum pf_layout { PF_HWC = 0, PF_NCHW = 1 };
#define PF_SKIP_PASSTHROUGH 256
/* OR with PF_SKIP_RESAMPLED to leave the output of specs with side != out_size
 * untouched: when every spec is a passthrough (the caller's target mpps all map
 * to side == out_size) a lean passthrough kernel serves the call. */
#define PF_SKIP_RESAMPLED 512

/* Tissue-mask rules for pf_mask. */
enum pf_mask_mode {
    PF_MASK_LUMINANCE = 0,  /* reference rule: Rec.709 luminance < thr (pkg/foreground.py:141-158) */
    PF_MASK_SATURATION = 1  /* BASELINE rule: HSV saturation (max-min)/max > thr */
};

/* ------------------------------------------------------------------------ */
/* Slide pyramid resident in HBM.                                            */
/*                                                                          */
/* Level l is stored padded and tile-major: tile (tx, ty) starts at          */
/*   level_ptr[l] + (ty * tiles_x[l] + tx) * tile_size * tile_size * 3       */
/* and pixel (u, v) of a tile at byte (v * tile_size + u) * 3 (RGB, HWC).    */
/* Edge tiles keep the full tile_size^2 footprint; the bytes beyond          */
/* width/height are never read.  The tile grid is the reference's           */
/* SlideRecord.tile_grid / tile_dims (pkg/store.py:140-149).                */
/*                                                                          */
/* Residency (replaces TileCache/fetch_chunk, pkg/store.py:270-319,          */
/* 611-649): when tile_map[l] != 0 the level is compacted -- level_ptr[l]    */
/* holds resident tiles only, as slots of tile_size^2*3 bytes, and           */
/* tile_map[l] is a device int32[tiles_y*tiles_x] giving tile (tx, ty)'s     */
/* slot; slot 0 is an all-zero hole that every non-resident tile maps to.    */
/* ------------------------------------------------------------------------ */
typedef struct pf_slide_desc {
    uint64_t level_ptr[PF_MAX_LEVELS]; /* device addresses */
    uint64_t tile_map[PF_MAX_LEVELS];  /* 0: dense level; else device int32 slot map */
    double mpp[PF_MAX_LEVELS];
    int32_t width[PF_MAX_LEVELS];
    int32_t height[PF_MAX_LEVELS];
    int32_t tiles_x[PF_MAX_LEVELS];
    int32_t tiles_y[PF_MAX_LEVELS];
    int32_t downsample[PF_MAX_LEVELS];
    int32_t n_levels;
    int32_t tile_size;
    double base_mpp;
    /* 0, or the device address of an int32 fault word: a read that resolves
     * to the zero hole (slot 0) of a compacted level stores
     * PF_ERR_OUT_OF_BOUNDS there (pf_slide_status reads and clears it). */
    uint64_t status_word;
} pf_slide_desc;

/* One patch to extract: the reference's PatchSpec (pkg/sampler.py:61-103)
 * plus the read plan of Slide.read_region (pkg/store.py:677-681). */
typedef struct pf_patch_spec {
    int64_t seq;
    double target_mpp;
    int32_t slide;     /* index into the slide array of the call */
    int32_t x, y, width, height;
    int32_t out_size;
    int32_t mpp_idx;   /* index into SamplerConfig.target_mpps, -1 if n/a */
    int32_t level;     /* select_level(record, target_mpp)      store.py:568-581 */
    int32_t side;      /* max(1, rha(out_size*target_mpp/mpp_L)) store.py:679 */
    int32_t sx, sy;    /* rha(x/ds_L), rha(y/ds_L) — filled on device */
    int32_t flags;
} pf_patch_spec;

/* ------------------------------------------------------------------------ */
/* Library-owned slide handles (ownership row of SURVEY §8(b)): the pyramid   */
/* lives in HBM allocated by the library; callers without torch create a      */
/* slide, upload level-0 pixels (then the pyramid is box-filtered on device)  */
/* or store tiles, and pass pf_slide_get_desc's descriptor (copied into a     */
/* device array) to the batched entry points.  Replaces open_slide /          */
/* SlideRecord + TileCache-backed reads (pkg/store.py:123-237, 270-319,       */
/* 727-751) for a resident pyramid.                                          */
/* ------------------------------------------------------------------------ */
typedef struct pf_slide pf_slide;
/* Level dims as ingest_image (pkg/store.py:496-498): ceil-divide by the
 * factor until max(dim) <= tile_size; mpp_l = base_mpp * factor^l. */
int pf_slide_create(int32_t width, int32_t height, double base_mpp, int32_t tile_size,
                    int32_t downsample_factor, pf_slide** out);
int pf_slide_destroy(pf_slide* slide); /* synchronises the device */
int pf_slide_get_desc(const pf_slide* slide, pf_slide_desc* out_host);
/* Level-0 RGB rows (row_stride bytes apart, 0 = 3 * width), host or device
 * memory, tiled into level 0; levels 1.. then built with pf_build_level.
 * Host uploads synchronise the stream per 256-row chunk. */
int pf_slide_upload_level0(pf_slide* slide, const uint8_t* hwc, int64_t row_stride, int32_t on_host,
                           void* stream);
/* One decoded store tile (tile_dims-cropped, pkg/store.py:140-149) from host
 * memory into its slot; then pf_slide_build_pyramid if upper levels are not
 * uploaded too. */
int pf_slide_upload_tile(pf_slide* slide, int32_t level, int32_t tx, int32_t ty, const uint8_t* tile_hwc_host,
                         int32_t tw, int32_t th, void* stream);
int pf_slide_build_pyramid(pf_slide* slide, void* stream);
/* Synchronise `stream` and read the descriptor's fault word: PF_ERR_OUT_OF_BOUNDS
 * (store.OutOfBoundsError, pkg/store.py:66) if a read since the last clear hit
 * the zero hole of a compacted level, else PF_OK.  clear != 0 resets it. */
int pf_slide_status(const pf_slide_desc* desc_host, int32_t clear, void* stream);

/* ------------------------------------------------------------------------ */
/* Host-backed tile tier (replaces TileCache/fetch_chunk,  */
/* pkg/store.py:270-319, 611-649, for slide sets whose reachable tiles exceed */
/* HBM).  A compacted level (tile_map != 0) gets a pool of n_slots HBM slots  */
/* smaller than its reachable set, backed by a pinned device-mapped host copy */
/* of every reachable tile.  All device addresses; one record per slide of    */
/* the call (slot_owner == 0: the slide has no tier).                         */
/* ------------------------------------------------------------------------ */
typedef struct pf_tile_tier {
    uint64_t host_tiles;    /* device address of the mapped host store (tile-major, T*T*3 per tile) */
    uint64_t host_index;    /* int64[tiles_y * tiles_x]: tile -> index in the host store, -1 if absent */
    uint64_t slot_owner;    /* int32[n_slots + 1]: tile held by each slot, -1 none */
    uint64_t slot_last_use; /* int32[n_slots + 1]: last batch id that read the slot */
    uint64_t requested;     /* int32[tiles]: request flags (all 0 between calls) */
    uint64_t miss_list;     /* int32[max_miss] */
    uint64_t victims;       /* int32[max_miss] */
    uint64_t counters;      /* int32[8]: [0] misses, [1] filled (this batch), [2] clock hand, [4..5] u64 filled total */
    int32_t level, n_slots, max_miss, _pad;
} pf_tile_tier;

/* Pinned host memory mapped into the device address space (the tier's host store). */
int pf_host_alloc_mapped(int64_t bytes, void** host_ptr, void** dev_ptr);
int pf_host_free(void* host_ptr);

/* Make every tile the windows of specs_dev (planned: level/side/sx/sy) touch resident for
 * batch id `batch` (>= 2, increasing per call): mark hits, claim victim slots no batch >=
 * batch - 1 uses (clock hand), copy the missing tiles from the host store (zero-copy), update
 * tile_map.  Stream-ordered, no host sync; the caller orders this call after the crops of
 * batch - 2.  max_fill: the largest max_miss of the tiers; max_tiles_per_spec: tiles a window
 * can touch (e.g. (ceil(side/T) + 1)^2).  A batch needing more tiles than a pool holds sets
 * the slide's fault word to PF_ERR_CAPACITY (pf_slide_status). */
int pf_tier_prefetch(const pf_slide_desc* slides_dev, const pf_tile_tier* tiers_dev, int32_t n_slides,
                     const pf_patch_spec* specs_dev, int32_t n, int32_t batch, int32_t max_fill,
                     int32_t max_tiles_per_spec, void* stream);

/* ------------------------------------------------------------------------ */
/* Library                                                                   */
/* ------------------------------------------------------------------------ */
int pf_abi_version(void);
const char* pf_last_error(void);
/* Number of CUDA kernels this library has launched in this process. */
uint64_t pf_launch_count(void);

/* ------------------------------------------------------------------------ */
/* Store (pkg/store.py)                                                      */
/* ------------------------------------------------------------------------ */

/* Box-downsample level `level-1` of `slide` by `factor` into level `level`
 * (both described by `slide`).  Replaces the pyramid loop of ingest_image
 * (pkg/store.py:496-498) over _box_downsample (pkg/store.py:429-441):
 * out = floor(sum/count + 0.5) with edge blocks averaging only the pixels they
 * contain.  Bit-exact. */
int pf_build_level(const pf_slide_desc* slide, int32_t level, int32_t factor, void* stream);

/* _box_downsample(level_src, factor) into a dense (ceil(H/f), ceil(W/f), 3)
 * uint8 HWC device buffer: the 1/32 thumbnail of BASELINE config 1 and
 * Slide.thumbnail (pkg/store.py:604-609) when factor == 1 on the coarsest
 * level.  Bit-exact. */
int pf_thumbnail(const pf_slide_desc* slide, int32_t src_level, int32_t factor,
                 uint8_t* out_hwc, void* stream);

/* Fill sx/sy of device specs from x/y and the slide's level downsample:
 * sx = round_half_away(x / ds) (pkg/store.py:70-72, 680-681). `slides_dev`
 * is a device array of pf_slide_desc. */
int pf_plan_regions(const pf_slide_desc* slides_dev, pf_patch_spec* specs_dev, int32_t n,
                    void* stream);

/* Batched Slide.read_region (pkg/store.py:651-688 + _read_window 690-724):
 * window of `side` px at (sx, sy) of `level`, clamped with edge replication,
 * passthrough when side == out_size else PIL BILINEAR (Resample.c semantics,
 * 22-bit fixed point, bit-exact).  All specs must share out_size.
 * dtype PF_U8: raw pixels; PF_F32/PF_BF16: (v/255 - mean[c]) / std[c] in FP32
 * (normalize_patch, pkg/pipeline.py:152-155, when mean = std = 0.5).
 * layout PF_HWC: [n, S, S, 3]; PF_NCHW: [n, 3, S, S]. */
int pf_read_regions(const pf_slide_desc* slides_dev, const pf_patch_spec* specs_dev, int32_t n,
                    int32_t out_size, int32_t dtype, int32_t layout, const float* mean3,
                    const float* std3, void* out, void* stream);

/* Whether pf_read_regions' fused kernel takes a window of `side` px resampled
 * to out_size (its shared-memory plan holds a band of >= 4 source rows and
 * <= 32 taps: down-ratios up to ~15 at out_size <= 512).  Other requests go
 * through pf_read_region_generic. */
int pf_read_region_fits(int32_t side, int32_t out_size, int32_t dtype, int32_t* fits);

/* Slide.read_region (pkg/store.py:651-688) for ONE spec of any size: PIL's
 * two BILINEAR passes (22-bit taps, bit-exact) through a global uint8
 * intermediate in `scratch_dev` (pf_read_region_generic_scratch_bytes), or
 * the clamped window itself when side == out_size.  `spec` is a HOST record
 * with level/side/sx/sy filled; `slides_dev` the device descriptor array.
 * Output as pf_read_regions for one patch ([S, S, 3] or [3, S, S]). */
int pf_read_region_generic_scratch_bytes(int32_t side, int32_t out_size, int64_t* bytes);
int pf_read_region_generic(const pf_slide_desc* slides_dev, const pf_patch_spec* spec, int32_t out_size,
                           int32_t dtype, int32_t layout, const float* mean3, const float* std3,
                           void* scratch_dev, int64_t scratch_bytes, void* out, void* stream);

/* normalize_patch (pkg/pipeline.py:152-155) on an HWC uint8 device buffer of
 * n_pixels RGB pixels: out = (v/255 - mean[c]) / std[c] in FP32 (same layout),
 * dtype PF_F32 or PF_BF16. */
int pf_normalize(const uint8_t* in_hwc, int64_t n_pixels, int32_t dtype, const float* mean3,
                 const float* std3, void* out, void* stream);

/* ------------------------------------------------------------------------ */
/* Foreground (pkg/foreground.py)                                            */
/* ------------------------------------------------------------------------ */

/* mask_from_rgb (pkg/foreground.py:141-158) and the BASELINE saturation rule.
 * in: dense (h, w, 3) uint8 device image; out: (h, w) uint8 {0,1}.
 * morph_radius > 0 (saturation mode only) applies binary opening then closing
 * with a (2r+1)^2 square, zero border (scipy.ndimage semantics); `scratch`
 * must then hold 2*h*w bytes. */
int pf_mask(const uint8_t* img_hwc, int32_t h, int32_t w, int32_t mode, double threshold,
            int32_t morph_radius, uint8_t* out, uint8_t* scratch, void* stream);

/* polygon_from_mask (pkg/foreground.py:169-220), host-side: marching squares
 * at iso 0.5 on the 1-px zero-padded mask (low-connected saddles), ring
 * assembly in creation order, (row,col)->(x,y)-1, drop rings with <3 points or
 * |area| < min_region_px, orient by nesting depth, divide by scale.
 * HOST buffers.  xy receives n_points (x, y) pairs; ring_off n_rings+1 offsets.
 * Returns PF_ERR_CAPACITY (with *n_points / *n_rings set) if caps are small,
 * PF_ERR_EMPTY_FOREGROUND if nothing survives. */
int pf_polygon_trace(const uint8_t* mask, int32_t h, int32_t w, double scale, double min_region_px,
                     double* xy, int64_t xy_cap_points, int64_t* ring_off, int32_t ring_cap,
                     int64_t* n_points, int32_t* n_rings);

/* polygon_from_mask on the GPU: the same rings as
 * pf_polygon_trace, ring for ring and vertex for vertex, from a DEVICE mask
 * (h, w) uint8 (e.g. pf_mask's output) into DEVICE outputs (xy: n_points
 * (x, y) float64 pairs, ring_off: n_rings + 1 int64 offsets).  Segments are
 * assembled into rings by pointer jumping (cycle first/last segment, list
 * ranking) instead of find_contours' sequential joining.  `scratch` of
 * pf_polygon_trace_device_scratch_bytes.  Synchronises `stream` (the ring and
 * point counts size the outputs); PF_ERR_CAPACITY with *n_points/*n_rings set
 * when the outputs are too small, PF_ERR_EMPTY_FOREGROUND as the reference. */
int pf_polygon_trace_device_scratch_bytes(int32_t h, int32_t w, int64_t* bytes);
int pf_polygon_trace_device(const uint8_t* mask_dev, int32_t h, int32_t w, double scale, double min_region_px,
                            void* scratch, int64_t scratch_bytes, double* xy_dev, int64_t xy_cap_points,
                            int64_t* ring_off_dev, int32_t ring_cap, int64_t* n_points, int32_t* n_rings,
                            void* stream);

/* Slab index of a ForegroundPolygon for the device even-odd test.  HOST
 * buffers: rings as concatenated (x, y) float64 with ring_off[n_rings+1].
 * _size reports the blob size; _build fills it (copy it to the device as is). */
int pf_polygon_index_size(const double* xy, const int64_t* ring_off, int32_t n_rings,
                          int64_t* bytes);
int pf_polygon_index_build(const double* xy, const int64_t* ring_off, int32_t n_rings, void* blob,
                           int64_t bytes);

/* Coarse classification raster of a polygon for the sampler's acceptance test
 * (no reference counterpart: a precomputed filter in front of overlap_fraction,
 * pkg/foreground.py:246-286).  Two levels of square cells, `cell` px (a power of
 * two, 8..16384) and 4 `cell` px, each covering the bounding box plus one cell;
 * each cell is 2 bits: 01 every point
 * of the cell (closed, grown by 1 px) is inside, 00 every point outside, 1x an
 * edge comes within 1 px of it.  A window whose cells are all 01 (all 00) has
 * overlap_fraction 1.0 (0.0) exactly, since the even-odd parity is constant over
 * an edge-free region.  DEVICE blob and output; _bytes sizes the output from
 * the polygon's bbox (ForegroundPolygon.bounding_box()). */
int pf_polygon_raster_bytes(const double* bbox, double cell, int64_t* bytes);
int pf_polygon_raster_build(const void* poly_blob_dev, const double* bbox, double cell, void* raster_dev,
                            int64_t raster_bytes, void* stream);

/* Batched overlap_fraction (pkg/foreground.py:246-286, points_in_polygon
 * 223-243): rects_dev is n x (x, y, w, h) float64; bit-exact FP64 even-odd
 * test on the (grid+1)^2 corners + grid^2 centres.  32 <= grid <= 256. */
int pf_overlap_fraction(const void* poly_blob_dev, const double* rects_dev, int32_t n, int32_t grid,
                        double* out_dev, void* stream);

/* ------------------------------------------------------------------------ */
/* Sampler (pkg/sampler.py, pkg/rng.py)                                      */
/* ------------------------------------------------------------------------ */
typedef struct pf_sampler_config {
    uint64_t seed;
    uint64_t key_slide, key_coords, key_mpp; /* mix64(seed ^ fnv1a(purpose)), rng.py:49 */
    double min_foreground;
    double mpp[PF_MAX_MPPS];
    double mpp_weight[PF_MAX_MPPS];
    int32_t n_mpps;
    int32_t patch_size;
    int32_t max_attempts;
    int32_t strategy; /* 0 uniform, 1 weighted (sampler.py:130-137) */
    int32_t n_slides;
    int32_t grid;     /* OVERLAP_GRID (foreground.py:30) */
} pf_sampler_config;

typedef struct pf_sampler_slide {
    uint64_t poly_blob; /* device address of the polygon slab index */
    double bbox[4];     /* ForegroundPolygon.bounding_box() */
    double weight;      /* slide_weights[slide_id] (weighted strategy) */
    int32_t width, height;
    int32_t fp[PF_MAX_MPPS];    /* footprint_px(patch, mpp_i, base_mpp) sampler.py:125 */
    int32_t x_lo[PF_MAX_MPPS], x_hi[PF_MAX_MPPS];
    int32_t y_lo[PF_MAX_MPPS], y_hi[PF_MAX_MPPS];
    int32_t level[PF_MAX_MPPS]; /* read plan per mpp: select_level */
    int32_t side[PF_MAX_MPPS];
    int32_t _pad;
    uint64_t raster;    /* device address of a pf_polygon_raster_build raster of poly_blob, or 0
                           (ABI 3; candidates it classifies skip the lattice test) */
} pf_sampler_slide;

/* Device-resident stream state: the reference's StreamSet counters plus the
 * epoch_stream loop variables (sampler.py:206-227). */
typedef struct pf_sampler_state {
    uint64_t c_slide, c_coords, c_mpp;
    int64_t seq;
    int64_t consecutive_failures;
    int64_t attempts;         /* statistics */
    int64_t slow_evals;       /* candidates evaluated on the sequential path */
    int32_t status;           /* pf_status of the last call */
    int32_t emitted;          /* specs emitted by the last call */
    int32_t cur_slide;        /* slide of an unfinished sample_patch call, -1 if none */
    int32_t cur_used;         /* attempts it has consumed */
    int64_t _reserved;
} pf_sampler_state;

/* On-GPU PNG tile decode (replaces decode_tile's Pillow path for the store's
 * default codec, pkg/store.py:397-416, 470).  pf_png_inflate: one thread per
 * tile inflates the zlib stream zdata[zoff[t] .. zoff[t+1]) (concatenated IDAT
 * payloads of an 8-bit RGB non-interlaced PNG) into raw[roff[t] .. +rlen[t]),
 * rlen = th * (1 + 3 * tw) filtered scanline bytes; status_dev[t] = 0 or a
 * negative parse error.  pf_png_unfilter: undoes the row filters of tiles
 * whose status is 0 into dst_dev[t] (a tile slot, row pitch tile_size * 3). */
int pf_png_inflate(const uint8_t* zdata_dev, const int64_t* zoff_dev, int32_t n, uint8_t* raw_dev,
                   const int64_t* roff_dev, const int64_t* rlen_dev, int32_t* status_dev, void* stream);
int pf_png_unfilter(const uint8_t* raw_dev, const int64_t* roff_dev, const int32_t* tile_w_dev,
                    const int32_t* tile_h_dev, uint8_t* const* dst_dev, int32_t tile_size, int32_t n,
                    int32_t* status_dev, void* stream);

/* On-GPU baseline JPEG tile decode (decode_tile's Pillow path for JPEG stores,
 * pkg/store.py:397-426), bit-exact with libjpeg-turbo's default decompression
 * (accurate integer IDCT, fancy 2x2 chroma upsampling).  tiles_dev: n packed
 * tile records (layout in csrc/pf_jpeg.cu, sizes via pf_jpeg_struct_sizes);
 * data_dev: unstuffed entropy-coded segments; huff_dev / quant_dev: table
 * pools; coef_dev / planes_dev: scratch; blk_*: the (tile, component, block)
 * list for the IDCT; px_off_dev: exclusive prefix of tile pixel counts.
 * status_dev[t] = 0 or a negative entropy-decode error. */
int pf_jpeg_decode(const void* tiles_dev, int32_t n, const uint8_t* data_dev, const void* huff_dev,
                   const uint16_t* quant_dev, int16_t* coef_dev, uint8_t* planes_dev, const int32_t* blk_tile_dev,
                   const int32_t* blk_comp_dev, const int32_t* blk_index_dev, int32_t nblk,
                   const int64_t* px_off_dev, int64_t total_px, int32_t tile_size, int32_t* status_dev,
                   void* stream);
int pf_jpeg_struct_sizes(int32_t* huff, int32_t* tile);

/* Host preparation for pf_jpeg_decode: parse n JPEG files bytes[off[t] .. off[t+1])
 * of expected size tw[t] x th[t] into tile records (destination slot dst[t]),
 * de-duplicated Huffman / quant pools, unstuffed entropy segments and the IDCT
 * block list (buffer bounds in csrc/pf_jpeg_host.cpp).  ok_out[t] = 1 marks a
 * tile the GPU path does not take (progressive, restart markers, other chroma
 * sampling) for the host decoder; malformed tiles fail with PF_ERR_DECODE. */
int pf_jpeg_prepare(const uint8_t* bytes, const int64_t* off, const int32_t* tw, const int32_t* th,
                    const uint64_t* dst, int32_t n, void* tiles_out, int32_t* ok_out, uint8_t* data_out,
                    void* huff_out, uint16_t* quant_out, int32_t* blk_tile_out, int32_t* blk_comp_out,
                    int32_t* blk_index_out, int64_t* px_off_out, int64_t* counts_out);

/* Capped replay draws (replaces CappedCache.draw inside capped_stream,
 * pkg/sampler.py:230-281): out[i] = stored[randrange(n_stored)] with the
 * "cache" RandomStream (key = stream key of (seed, "cache")); *counter_dev is
 * the stream's draw counter, advanced on device (rejections included). */
int pf_capped_draw(uint64_t key, uint64_t* counter_dev, const pf_patch_spec* stored_dev, int32_t n_stored,
                   int32_t n, pf_patch_spec* out_dev, void* stream);

/* Bytes of device workspace pf_sample needs for a speculation window. */
int pf_sample_workspace_bytes(const pf_sampler_config* cfg, int32_t window, int64_t* bytes);

/* Next n specs of epoch_stream (pkg/sampler.py:196-227) — bit-exact coords,
 * mpp and slide choice — written to specs_dev with the read plan (level,
 * side, sx, sy) filled.  Speculates `window` attempts per slide per round for
 * up to `rounds` rounds, then finishes on the sequential exact path.  Status
 * lands in state_dev->status (PF_ERR_NO_SAMPLABLE on stream failure).
 * all_fit != 0 asserts every (slide, mpp) footprint fits its bbox range
 * (enables speculation); 0 forces the sequential path. */
int pf_sample(const pf_sampler_config* cfg, const pf_sampler_slide* slides_dev,
              const pf_slide_desc* slide_descs_dev, pf_sampler_state* state_dev, int32_t n,
              pf_patch_spec* out_dev, void* workspace, int64_t workspace_bytes, int32_t window,
              int32_t rounds, int32_t all_fit, void* stream);

/* ------------------------------------------------------------------------ */
/* Multi-crop augmentation (BASELINE config 2; absent from the reference)    */
/* ------------------------------------------------------------------------ */
typedef struct pf_multicrop_config {
    uint64_t rrc_table_global;        /* device pf_rrc_table for global_size (0: computed per crop) */
    uint64_t rrc_table_local;         /* device pf_rrc_table for local_size  (0: computed per crop) */
    int32_t n_global, n_local;
    int32_t global_size, local_size;
    int32_t src_size;                 /* source patch side (224) */
    int32_t blur_kernel;              /* 9 */
    float global_scale[2], local_scale[2];
    float ratio[2];                   /* (3/4, 4/3) */
    float p_flip, p_jitter, p_gray;
    float brightness, contrast, saturation, hue;
    float sigma_min, sigma_max;
    float solarize_threshold;
    float p_blur[PF_MAX_CROPS];       /* per crop index (globals first) */
    float p_solarize[PF_MAX_CROPS];
} pf_multicrop_config;

/* Per-crop augmentation parameters (explicit; shared with the oracle). */
typedef struct pf_crop_param {
    int32_t top, left, height, width; /* RandomResizedCrop box in the source */
    int32_t out_size;
    int32_t flags;                    /* PF_AUG_* bits */
    uint8_t order[4];                 /* ColorJitter op order: 0 b, 1 c, 2 s, 3 h */
    float brightness, contrast, saturation, hue;
    float sigma;
    float solarize_threshold;
    int32_t patch, crop;
    int32_t _pad;
} pf_crop_param;

#define PF_AUG_FLIP 1
#define PF_AUG_JITTER 2
#define PF_AUG_GRAY 4
#define PF_AUG_BLUR 8
#define PF_AUG_SOLARIZE 16

/* Philox4x32-10 keyed by (seed, rank), counter (step, patch, crop, draw):
 * n_patches * (n_global + n_local) records, patch-major. */
int pf_crop_params(uint64_t seed, int32_t rank, uint64_t step, int32_t n_patches,
                   const pf_multicrop_config* cfg, pf_crop_param* out_dev, void* stream);

/* RandomResizedCrop resample taps for every crop extent 1..src_size to
 * out_size: torch uint8 antialiased bilinear (int16 weights, per-extent
 * precision), as used by torchvision resized_crop.  Built once on device;
 * pass its address in pf_multicrop_config.rrc_table_*. */
int pf_rrc_table_bytes(int32_t src_size, int32_t out_size, int64_t* bytes);
int pf_rrc_table_build(int32_t src_size, int32_t out_size, void* table_dev, void* stream);

/* One Philox4x32-10 block (Random123 semantics): out = philox(ctr, key). */
void pf_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Fused gather + RandomResizedCrop (torch uint8 antialiased bilinear) + flip
 * + ColorJitter (per-op uint8 quantisation, per-crop order) + grayscale +
 * gaussian blur (reflect) + solarize + (v/255 - mean)/std, written as
 * [crop][patch][3][S][S] (DINOv2 collate order) in `dtype`.
 * Source of patch i: if specs_dev[i].side == src_size the slide tiles are read
 * directly; otherwise src_hwc[i] (a [n, src, src, 3] uint8 buffer produced by
 * pf_read_regions) is used. */
int pf_multicrop(const pf_slide_desc* slides_dev, const pf_patch_spec* specs_dev,
                 const uint8_t* src_hwc, int32_t n_patches, const pf_crop_param* params_dev,
                 const pf_multicrop_config* cfg, int32_t dtype, const float* mean3,
                 const float* std3, void* out_global, void* out_local, void* stream);

/* ------------------------------------------------------------------------ */
/* Synthetic slides (BASELINE configs; stands in for TCGA WSIs)              */
/* ------------------------------------------------------------------------ */
/* Fill level 0 of `slide` from a smooth low-resolution field (device, float,
 * field_h x field_w, cell = field_cell level-0 px): tissue where field > thr,
 * H&E-like colours, near-white background + N(0, 4) noise, seeded. */
int pf_synth_level0(const pf_slide_desc* slide, const float* field, int32_t field_h,
                    int32_t field_w, int32_t field_cell, float threshold, uint64_t seed,
                    void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PF_B200_H */
