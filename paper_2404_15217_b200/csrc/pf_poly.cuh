// Device even-odd overlap test over the slab index (pf_poly.h).
//
// Restates overlap_fraction (pkg/foreground.py:246-286) on top of
// points_in_polygon (223-243) bit-exactly: the same FP64 lattice
//   edges_x = x + k * (w / grid), centres (e_k + e_{k+1}) / 2
// and the same crossing expression
//   crosses = (y1 > py) != (y2 > py);  x_at = x1 + (py - y1) * (x2 - x1) / (y2 - y1)
// evaluated with one IEEE rounding per op.  Parity over all rings is the XOR
// of the per-ring parities, i.e. the parity of the total crossing count, so
// rings are merged.  For a row py only the slab containing py can cross it;
// edges provably left of every point of the row never count, edges provably
// right always count, and only the few in between get x_at evaluated.
#pragma once

#include "pf_common.cuh"
#include "pf_poly.h"

namespace pf {

#ifdef PF_EVAL_TIMING  // phase stamps of the calling warp (tools/eval_timing.py)
__device__ unsigned long long g_tmarks[8192][2];
#define PF_TMARK(i)                                                                                   \
    do {                                                                                              \
        if ((threadIdx.x & 31) == 0) {                                                                \
            unsigned long long t_;                                                                    \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                    \
            g_tmarks[((blockIdx.x * blockDim.x + threadIdx.x) >> 5) & 8191][i] = t_;                 \
        }                                                                                             \
    } while (0)
#else
#define PF_TMARK(i) do {} while (0)
#endif

struct PolyView {
    const double* edges;
    const double* Y;
    const int32_t* slab_off;
    const int32_t* slab_edge;
    const double* lo;
    const double* hi;
    const int32_t* lut;
    int32_t n_y, lut_len, lut_base;
    double bx0, by0, bx1, by1;
};

__device__ __forceinline__ PolyView poly_view(const void* blob) {
    const PolyHeader* h = reinterpret_cast<const PolyHeader*>(blob);
    const uint8_t* b = reinterpret_cast<const uint8_t*>(blob);
    PolyView v;
    v.edges = reinterpret_cast<const double*>(b + h->off_edges);
    v.Y = reinterpret_cast<const double*>(b + h->off_y);
    v.slab_off = reinterpret_cast<const int32_t*>(b + h->off_slab_off);
    v.slab_edge = reinterpret_cast<const int32_t*>(b + h->off_slab_edge);
    v.lo = reinterpret_cast<const double*>(b + h->off_slab_lo);
    v.hi = reinterpret_cast<const double*>(b + h->off_slab_hi);
    v.lut = reinterpret_cast<const int32_t*>(b + h->off_lut);
    v.n_y = h->n_y;
    v.lut_len = h->lut_len;
    v.lut_base = h->lut_base;
    v.bx0 = h->bbox[0];
    v.by0 = h->bbox[1];
    v.bx1 = h->bbox[2];
    v.by1 = h->bbox[3];
    return v;
}

// Slab k with Y[k] <= py < Y[k+1], or -1.
__device__ __forceinline__ int slab_of(const PolyView& P, double py) {
    if (P.n_y < 2 || !(py >= __ldg(P.Y)) || !(py < __ldg(P.Y + P.n_y - 1))) return -1;
    int k;
    if (P.lut_len > 0) {
        const int idx = (int)floor(py) - P.lut_base;
        k = __ldg(P.lut + min(max(idx, 0), P.lut_len - 1));
        if (k < 0) k = 0;
    } else {
        int a = 0, b = P.n_y - 1;  // invariant Y[a] <= py < Y[b]
        while (b - a > 1) {
            const int m = (a + b) >> 1;
            if (__ldg(P.Y + m) <= py) a = m;
            else b = m;
        }
        k = a;
    }
    while (k + 1 < P.n_y && __ldg(P.Y + k + 1) <= py) ++k;
    return k;
}

__device__ __forceinline__ double x_at(double x1, double y1, double x2, double y2, double py) {
    return __dadd_rn(x1, __ddiv_rn(__dmul_rn(__dsub_rn(py, y1), __dsub_rn(x2, x1)), __dsub_rn(y2, y1)));
}

__device__ __forceinline__ double edge_x_at(const PolyView& P, int e, double py) {
    return x_at(__ldg(P.edges + 4 * e), __ldg(P.edges + 4 * e + 1), __ldg(P.edges + 4 * e + 2),
                __ldg(P.edges + 4 * e + 3), py);
}

// Lattice coordinate k of a row: corner rows use edges e_k = x0 + k*step,
// centre rows (e_k + e_{k+1}) / 2.
__device__ __forceinline__ double lattice(double x0, double step, int k, bool centre) {
    const double ek = __dadd_rn(x0, __dmul_rn((double)k, step));
    if (!centre) return ek;
    const double ek1 = __dadd_rn(x0, __dmul_rn((double)(k + 1), step));
    return __dmul_rn(__dadd_rn(ek, ek1), 0.5);  // == / 2.0 exactly (no subnormals here)
}

// Row mask from the slab's search results: edges [i_lo, i_hi) may cross inside the row's
// x-range, edges [i_hi, e1) cross right of it (each flips every point), earlier ones left.
// xs(i, py): crossing x of slab entry i.
template <class XAt>
__device__ inline void row_crossings_by(XAt xs, double py, double x0, double step, bool centre, int n_pts, int nw,
                                        uint32_t* words, int i_lo, int i_hi, int e1) {
    if ((e1 - i_hi) & 1) {
        for (int j = 0; j < nw; ++j) {
            const int rem = n_pts - 32 * j;
            words[j] = rem >= 32 ? 0xffffffffu : (rem > 0 ? ((1u << rem) - 1u) : 0u);
        }
    }
    const double inv = 1.0 / step;  // estimate only: the walk below is exact
    for (int i = i_lo; i < i_hi; ++i) {
        const double X = xs(i, py);
        // c = number of points with px < X (points ascend in k): start from the nearest lattice
        // index and step until lattice(m) < X <= lattice(m + 1)
        const double est = floor((X - x0) * inv - (centre ? 0.5 : 0.0));
        int m = est < -1.0 ? -1 : (est > (double)(n_pts - 1) ? n_pts - 1 : (int)est);
        while (m >= 0 && !(lattice(x0, step, m, centre) < X)) --m;
        while (m + 1 < n_pts && lattice(x0, step, m + 1, centre) < X) ++m;
        const int c = m + 1;
        for (int j = 0; j < nw; ++j) {
            const int rem = c - 32 * j;
            words[j] ^= rem >= 32 ? 0xffffffffu : (rem > 0 ? ((1u << rem) - 1u) : 0u);
        }
    }
}

__device__ inline void row_crossings(const PolyView& P, double py, double x0, double step, bool centre, int n_pts,
                                     int nw, uint32_t* words, int i_lo, int i_hi, int e1) {
    row_crossings_by([&P](int i, double y) { return edge_x_at(P, __ldg(P.slab_edge + i), y); }, py, x0, step, centre,
                     n_pts, nw, words, i_lo, i_hi, e1);
}

// Inside-mask of one lattice row into `words` (nw 32-bit words, bit k =
// point k).  n_pts points, first coordinate x0, spacing step.
__device__ inline void row_mask(const PolyView& P, double py, double x0, double step, bool centre,
                                int n_pts, int nw, uint32_t* words) {
    for (int j = 0; j < nw; ++j) words[j] = 0u;
    const int k = slab_of(P, py);
    if (k < 0) return;
    const int e0 = __ldg(P.slab_off + k), e1 = __ldg(P.slab_off + k + 1);
    if (e0 == e1) return;
    const double xmin = lattice(x0, step, 0, centre);
    const double xmax = lattice(x0, step, n_pts - 1, centre);
    // i_lo: first edge not provably left (hi >= xmin); hi is prefix-max sorted
    int a = e0, b = e1;
    while (a < b) {
        const int m = (a + b) >> 1;
        if (__ldg(P.hi + m) < xmin) a = m + 1;
        else b = m;
    }
    const int i_lo = a;
    // i_hi: first edge provably right (lo > xmax); lo is suffix-min sorted
    a = i_lo;
    b = e1;
    while (a < b) {
        const int m = (a + b) >> 1;
        if (__ldg(P.lo + m) > xmax) b = m;
        else a = m + 1;
    }
    row_crossings(P, py, x0, step, centre, n_pts, nw, words, i_lo, a, e1);
}

constexpr int kMaxGrid = 256;
constexpr int kMaxWords = (kMaxGrid + 1 + 31) / 32;  // 9

// Per-warp cache of the slabs a window's rows fall in (its first kSlabCache slabs [ka, kb]):
// the two edge-range searches of row_mask depend only on the slab and on the row type's
// x-range, which every row of the window shares, so they are done once per slab instead of
// once per row (a slab holds ~9 rows of a 224 px window at grid 128).
// The edges the rows can cross (entries [i_lo, i_hi) of either row type) are copied too when
// they fit, so a row's crossings read shared memory only.
constexpr int kSlabCache = 48;
constexpr int kEdgeCache = 48;
struct CachedEdge {
    double x1, y1, x2, y2;
};
struct SlabCache {
    int4 range[kSlabCache];          // corner i_lo, i_hi, centre i_lo, i_hi
    double Y[kSlabCache + 1];        // slab boundaries Y[ka .. kb+1]
    int32_t e1[kSlabCache];          // slab_off[k + 1]
    int32_t ebase[kSlabCache];       // edges[i + ebase[j]] is slab entry i of slab j
    int32_t n_edges;                 // cached edges, or -1 when they did not fit
    int32_t _pad[3];
    CachedEdge edges[kEdgeCache];
};
constexpr int kSlabCacheBytes = (int)((sizeof(SlabCache) + 15) / 16 * 16);

// Cell rows per step of a count with a stop: 15 cell rows are 31 lattice rows, one per lane,
// so every step costs one row latency and the stop test runs after each.
constexpr int kStopChunk = 15;

__host__ __device__ constexpr int overlap_words(int grid) { return (grid + 1 + 31) / 32; }
__host__ __device__ constexpr int overlap_mask_bytes(int rows, int grid) {
    return ((2 * rows + 1) * overlap_words(grid) * 4 + 15) / 16 * 16;
}
// shared bytes one warp needs for a grid (16-byte multiple: per-warp areas stay aligned)
__host__ __device__ constexpr int overlap_smem_bytes(int grid) {
    return kSlabCacheBytes + overlap_mask_bytes(grid, grid);
}
// ... when it only counts with a stop (rows traced in chunks of kStopChunk: warp_overlap_accept)
__host__ __device__ constexpr int overlap_smem_bytes_chunked(int grid) {
    return kSlabCacheBytes + overlap_mask_bytes(grid < kStopChunk ? grid : kStopChunk, grid);
}

// row_mask for a row of a window whose slabs are cached (nslab of them).
__device__ inline void row_mask_cached(const PolyView& P, const SlabCache& c, int nslab, double py, double x0,
                                       double step, bool centre, int n_pts, int nw, uint32_t* words) {
    for (int j = 0; j < nw; ++j) words[j] = 0u;
    if (!(py >= c.Y[0]) || !(py < c.Y[nslab])) return;  // slab_of == -1 (outside [Y0, Ylast))
    int a = 0, b = nslab;  // invariant Y[a] <= py < Y[b]: slab_of's largest k with Y[k] <= py
    while (b - a > 1) {
        const int m = (a + b) >> 1;
        if (c.Y[m] <= py) a = m;
        else b = m;
    }
    const int4 r = c.range[a];
    const int i_lo = centre ? r.z : r.x, i_hi = centre ? r.w : r.y;
    if (c.n_edges >= 0) {
        PF_CHECK(a < nslab && nslab <= kSlabCache && (i_lo >= i_hi || (i_lo + c.ebase[a] >= 0 && i_hi + c.ebase[a] <= c.n_edges)));
        const CachedEdge* ed = c.edges + c.ebase[a];
        row_crossings_by([ed](int i, double y) { const CachedEdge& e = ed[i]; return x_at(e.x1, e.y1, e.x2, e.y2, y); },
                         py, x0, step, centre, n_pts, nw, words, i_lo, i_hi, c.e1[a]);
    } else {
        row_crossings(P, py, x0, step, centre, n_pts, nw, words, i_lo, i_hi, c.e1[a]);
    }
}

// Fill the cache for slabs [ka, ka + nslab) of a window with corner x-range [x, xlast] and
// centre x-range [xc0, xc1] (the searches of row_mask, one lane per slab).
__device__ inline void fill_slab_cache(const PolyView& P, SlabCache& c, int ka, int nslab, double x, double xlast,
                                       double xc0, double xc1) {
    const int lane = threadIdx.x & 31;
    for (int j = lane; j < nslab; j += 32) {
        const int k = ka + j;
        const int e0 = __ldg(P.slab_off + k), e1 = __ldg(P.slab_off + k + 1);
        int lo_c = e0, hi_c = e0, lo_m = e0, hi_m = e0;
        {
            int a = e0, b = e1;
            while (a < b) { const int m = (a + b) >> 1; if (__ldg(P.hi + m) < x) a = m + 1; else b = m; }
            lo_c = a;
            b = e1;
            while (a < b) { const int m = (a + b) >> 1; if (__ldg(P.lo + m) > xlast) b = m; else a = m + 1; }
            hi_c = a;
        }
        {
            int a = e0, b = e1;
            while (a < b) { const int m = (a + b) >> 1; if (__ldg(P.hi + m) < xc0) a = m + 1; else b = m; }
            lo_m = a;
            b = e1;
            while (a < b) { const int m = (a + b) >> 1; if (__ldg(P.lo + m) > xc1) b = m; else a = m + 1; }
            hi_m = a;
        }
        c.range[j] = make_int4(lo_c, hi_c, lo_m, hi_m);
        c.e1[j] = e1;
        c.Y[j] = __ldg(P.Y + k);
        if (j == nslab - 1) c.Y[nslab] = __ldg(P.Y + k + 1);
    }
    // edges: slab j's entries [u0, u1) = the union of its two ranges, packed in slab order
    int base = 0;
    for (int j0 = 0; j0 < nslab; j0 += 32) {
        const int j = j0 + lane;
        int u0 = 0, cnt = 0;
        if (j < nslab) {
            const int4 r = c.range[j];
            u0 = min(r.x, r.z);
            cnt = max(r.y, r.w) - u0;
            cnt = max(cnt, 0);
        }
        int incl = cnt;  // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int off = base + incl - cnt;
        if (j < nslab) c.ebase[j] = off - u0;
        if (j < nslab && off + cnt <= kEdgeCache)
            for (int t = 0; t < cnt; ++t) {
                PF_CHECK(off + t < kEdgeCache);
                const int e = __ldg(P.slab_edge + u0 + t);
                c.edges[off + t] = CachedEdge{__ldg(P.edges + 4 * e), __ldg(P.edges + 4 * e + 1),
                                              __ldg(P.edges + 4 * e + 2), __ldg(P.edges + 4 * e + 3)};
            }
        base += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) c.n_edges = base <= kEdgeCache ? base : -1;
    __syncwarp();
}

// Covered cells of lattice cell rows [r_lo, r_hi): corner rows r_lo..r_hi and centre rows
// r_lo..r_hi-1 are traced into `smem`, then counted.  With stop >= 0 the rows are taken in
// chunks of kStopChunk and the count returns early once it reaches `stop` or can no longer reach it
// (the returned value is then only compared against `stop`).
// `cache` (nslab slabs) replaces each row's slab and edge-range searches when non-null.
// `chunked` takes kStopChunk rows at a time without a stop (smem of overlap_smem_bytes_chunked).
__device__ inline int warp_overlap_rows(const PolyView& P, double x, double y, double sx, double sy, int grid,
                                        uint32_t* smem, int r_lo, int r_hi, int stop,
                                        const SlabCache* cache = nullptr, int nslab = 0, bool chunked = false) {
    const int lane = threadIdx.x & 31;
    const int nw = overlap_words(grid);
    const int chunk = stop >= 0 || chunked ? kStopChunk : grid;
    uint32_t* corner = smem + kSlabCacheBytes / 4;  // chunk + 1 rows
    uint32_t* centre = corner + (chunk + 1) * nw;    // chunk rows
    uint32_t words[kMaxWords];
    int total = 0;
    for (int c0 = r_lo; c0 < r_hi; c0 += chunk) {
        const int nrow = min(chunk, r_hi - c0);
        const int n_rows = 2 * nrow + 1;
        for (int ri = lane; ri < n_rows; ri += 32) {
            const bool is_centre = ri > nrow;
            const int r = is_centre ? ri - nrow - 1 : ri;
            const double py = lattice(y, sy, c0 + r, is_centre);
            if (cache) row_mask_cached(P, *cache, nslab, py, x, sx, is_centre, is_centre ? grid : grid + 1, nw, words);
            else row_mask(P, py, x, sx, is_centre, is_centre ? grid : grid + 1, nw, words);
            uint32_t* dst = (is_centre ? centre + r * nw : corner + r * nw);
            for (int j = 0; j < nw; ++j) dst[j] = words[j];
        }
        __syncwarp();
        int count = 0;
        for (int r = lane; r < nrow; r += 32) {
            const uint32_t* cr0 = corner + r * nw;
            const uint32_t* cr1 = corner + (r + 1) * nw;
            const uint32_t* m = centre + r * nw;
            for (int j = 0; j * 32 < grid; ++j) {
                const uint32_t a = cr0[j], b = cr1[j];
                const uint32_t a_next = (j + 1 < nw) ? cr0[j + 1] : 0u;
                const uint32_t b_next = (j + 1 < nw) ? cr1[j + 1] : 0u;
                const uint32_t a1 = (a >> 1) | (a_next << 31);
                const uint32_t b1 = (b >> 1) | (b_next << 31);
                const int rem = grid - 32 * j;
                const uint32_t valid = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
                count += __popc(a & a1 & b & b1 & m[j] & valid);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
        __syncwarp();
        total += count;
        if (stop >= 0 && (total >= stop || total + (r_hi - c0 - nrow) * grid < stop)) break;
    }
    return total;
}

// Warp-cooperative overlap_fraction numerator: number of covered cells, or
// -1 when the bounding-box early-out returns 0.0.  All lanes return the same
// value.  `smem` holds overlap_smem_bytes(grid) for this warp.
__device__ inline int warp_overlap_count_upto(const PolyView& P, double x, double y, double w, double h,
                                              int grid, uint32_t* smem, int stop) {
    if (x >= P.bx1 || y >= P.by1 || __dadd_rn(x, w) <= P.bx0 || __dadd_rn(y, h) <= P.by0) return -1;
    const int lane = threadIdx.x & 31;
    const int nw = overlap_words(grid);
    const double sx = __ddiv_rn(w, (double)grid), sy = __ddiv_rn(h, (double)grid);
    // Exact shortcut for windows no edge comes near: every lattice row lies in one of the slabs
    // ka..kb and every lattice point in [x, x_last].  If no slab has an edge whose x-bounds
    // overlap [x, x_last] (row_mask would evaluate no x_at), each row's mask is all-ones or
    // all-zeros by its slab's parity (e1 - i_hi) & 1 -- row_mask's own i_lo/i_hi collapse to the
    // window's -- so when every parity agrees the count is grid^2 or 0.
    if (P.n_y >= 2) {
        const double ylast = lattice(y, sy, grid, false), xlast = lattice(x, sx, grid, false);
        const double Yfirst = __ldg(P.Y), Ylast = __ldg(P.Y + P.n_y - 1);
        const bool rows_outside = !(y >= Yfirst) || !(ylast < Ylast);  // some rows get an empty mask
        // the two slab lookups are dependent load chains: odd lanes walk the last row's, in step
        // with the even lanes' first-row lookup (same code path, per-lane argument)
        const bool odd = lane & 1;
        const int kq0 = slab_of(P, odd ? ylast : y);
        const int kq = odd ? (ylast < Ylast ? kq0 : P.n_y - 2) : (y >= Yfirst ? kq0 : 0);
        const int ka = __shfl_sync(0xffffffffu, kq, 0), kb = __shfl_sync(0xffffffffu, kq, 1);
        bool amb = ka < 0;
        int par_or = 0, par_and = 1;
        for (int k = ka + lane; !amb && k <= kb; k += 32) {
            const int e0 = __ldg(P.slab_off + k), e1 = __ldg(P.slab_off + k + 1);
            int a = e0, b = e1;
            while (a < b) {
                const int m = (a + b) >> 1;
                if (__ldg(P.hi + m) < x) a = m + 1;
                else b = m;
            }
            // lo is suffix-min sorted: no edge of [i_lo, e1) starts left of x_last iff lo[i_lo] does
            // not, and then i_hi == i_lo
            amb |= a < e1 && !(__ldg(P.lo + a) > xlast);
            const int par = (e1 - a) & 1;
            par_or |= par;
            par_and &= par;
        }
        amb = __any_sync(0xffffffffu, amb);
        par_or = __any_sync(0xffffffffu, par_or);
        par_and = __all_sync(0xffffffffu, par_and);
        if (!amb && (par_or == 0 || (par_and && !rows_outside))) return par_or ? grid * grid : 0;
        PF_TMARK(0);
        const int nslab = kb - ka + 1;
        if (ka >= 0 && nslab >= 1 && nslab <= kSlabCache) {
            SlabCache* cache = reinterpret_cast<SlabCache*>(smem);
            fill_slab_cache(P, *cache, ka, nslab, x, xlast, lattice(x, sx, 0, true), lattice(x, sx, grid - 1, true));
            PF_TMARK(1);
            return warp_overlap_rows(P, x, y, sx, sy, grid, smem, 0, grid, stop, cache, nslab);
        }
    }
    return warp_overlap_rows(P, x, y, sx, sy, grid, smem, 0, grid, stop);
}

// Covered cells of the lattice cell rows [r_lo, r_hi) of a w x w window (a share of
// overlap_fraction's numerator; the shares of a partition of [0, grid) add up to it).  No
// shortcut: the sampler only sends windows its raster bounds could not settle.  `smem` of
// overlap_smem_bytes_chunked(grid); all lanes return the same value.
__device__ inline int warp_overlap_count_rows(const PolyView& P, double x, double y, double w, int grid,
                                              uint32_t* smem, int r_lo, int r_hi) {
    if (x >= P.bx1 || y >= P.by1 || __dadd_rn(x, w) <= P.bx0 || __dadd_rn(y, w) <= P.by0) return 0;
    const int lane = threadIdx.x & 31;
    const double sx = __ddiv_rn(w, (double)grid), sy = sx;
    if (P.n_y >= 2) {
        const double y0 = lattice(y, sy, r_lo, false), y1 = lattice(y, sy, r_hi, false);  // first, last row
        const double Yfirst = __ldg(P.Y), Ylast = __ldg(P.Y + P.n_y - 1);
        const bool odd = lane & 1;  // the two slab lookups in step on even / odd lanes
        const int kq0 = slab_of(P, odd ? y1 : y0);
        const int kq = odd ? (y1 < Ylast ? kq0 : P.n_y - 2) : (y0 >= Yfirst ? kq0 : 0);
        const int ka = __shfl_sync(0xffffffffu, kq, 0), kb = __shfl_sync(0xffffffffu, kq, 1);
        const int nslab = kb - ka + 1;
        if (ka >= 0 && nslab >= 1 && nslab <= kSlabCache) {
            SlabCache* cache = reinterpret_cast<SlabCache*>(smem);
            fill_slab_cache(P, *cache, ka, nslab, x, lattice(x, sx, grid, false), lattice(x, sx, 0, true),
                            lattice(x, sx, grid - 1, true));
            return warp_overlap_rows(P, x, y, sx, sy, grid, smem, r_lo, r_hi, -1, cache, nslab, true);
        }
    }
    return warp_overlap_rows(P, x, y, sx, sy, grid, smem, r_lo, r_hi, -1, nullptr, 0, true);
}

__device__ inline int warp_overlap_count(const PolyView& P, double x, double y, double w, double h, int grid,
                                         uint32_t* smem) {
    return warp_overlap_count_upto(P, x, y, w, h, grid, smem, -1);
}

// Raster decision for a window whose lattice points lie in [x, x1] x [y, y1]: 1 if every
// point is inside (overlap count grid^2), 0 if every point is outside (count 0; the bbox
// early-out's 0.0 compares the same), -1 undecided.  All lanes return the same value.
// Points within the last cell's 1 px growth share its parity, so x1 = x + w suffices for
// lattice points that round a hair past it.
__device__ inline int raster_decide(const RasterHeader* R, double x, double y, double x1, double y1) {
    const int lane = threadIdx.x & 31;
    const double ox = __ldg(&R->ox), oy = __ldg(&R->oy), ic = __ldg(&R->inv_cell);
    const int nx = __ldg(&R->nx), ny = __ldg(&R->ny), pitch = __ldg(&R->pitch);
    const uint32_t* words = reinterpret_cast<const uint32_t*>(R + 1);
    // cells outside the raster are more than a cell from every edge, and outside
    const double fx0 = floor(__dmul_rn(__dsub_rn(x, ox), ic)), fx1 = floor(__dmul_rn(__dsub_rn(x1, ox), ic));
    const double fy0 = floor(__dmul_rn(__dsub_rn(y, oy), ic)), fy1 = floor(__dmul_rn(__dsub_rn(y1, oy), ic));
    const bool partial = fx0 < 0.0 || fy0 < 0.0 || fx1 >= (double)nx || fy1 >= (double)ny;
    const int a0 = (int)fmax(fx0, 0.0), a1 = (int)fmin(fx1, (double)(nx - 1));
    const int b0 = (int)fmax(fy0, 0.0), b1 = (int)fmin(fy1, (double)(ny - 1));
    int in_ok = !partial && a0 <= a1 && b0 <= b1, out_ok = 1;
    if (a0 <= a1) {
        for (int r = b0 + lane; r <= b1; r += 32) {
            const uint32_t* row = words + (size_t)r * pitch;
            for (int w = a0 >> 4; w <= (a1 >> 4); ++w) {
                const uint32_t v = __ldg(row + w);
                const int lo = max(a0 - 16 * w, 0), hi = min(a1 - 16 * w, 15);
                const uint32_t m = (hi == 15 ? 0xffffffffu : ((1u << (2 * hi + 2)) - 1u)) & ~((1u << (2 * lo)) - 1u);
                in_ok &= (v & m) == (kRasterInside & m);
                out_ok &= (v & m) == 0u;
            }
        }
    }
    in_ok = __all_sync(0xffffffffu, in_ok);
    out_ok = __all_sync(0xffffffffu, out_ok);
    return in_ok ? 1 : (out_ok ? 0 : -1);
}

// raster_decide for one thread (the sampler's classification pass: a thread per candidate).
__device__ inline int raster_decide_thread(const RasterHeader* R, double x, double y, double x1, double y1) {
    const double ox = __ldg(&R->ox), oy = __ldg(&R->oy), ic = __ldg(&R->inv_cell);
    const int nx = __ldg(&R->nx), ny = __ldg(&R->ny), pitch = __ldg(&R->pitch);
    const uint32_t* words = reinterpret_cast<const uint32_t*>(R + 1);
    const double fx0 = floor(__dmul_rn(__dsub_rn(x, ox), ic)), fx1 = floor(__dmul_rn(__dsub_rn(x1, ox), ic));
    const double fy0 = floor(__dmul_rn(__dsub_rn(y, oy), ic)), fy1 = floor(__dmul_rn(__dsub_rn(y1, oy), ic));
    const bool partial = fx0 < 0.0 || fy0 < 0.0 || fx1 >= (double)nx || fy1 >= (double)ny;
    const int a0 = (int)fmax(fx0, 0.0), a1 = (int)fmin(fx1, (double)(nx - 1));
    const int b0 = (int)fmax(fy0, 0.0), b1 = (int)fmin(fy1, (double)(ny - 1));
    bool in_ok = !partial && a0 <= a1 && b0 <= b1, out_ok = true;
    if (a0 <= a1) {
        for (int r = b0; r <= b1 && (in_ok || out_ok); ++r) {
            const uint32_t* row = words + (size_t)r * pitch;
            for (int w = a0 >> 4; w <= (a1 >> 4); ++w) {
                const uint32_t v = __ldg(row + w);
                const int lo = max(a0 - 16 * w, 0), hi = min(a1 - 16 * w, 15);
                const uint32_t m = (hi == 15 ? 0xffffffffu : ((1u << (2 * hi + 2)) - 1u)) & ~((1u << (2 * lo)) - 1u);
                in_ok &= (v & m) == (kRasterInside & m);
                out_ok &= (v & m) == 0u;
            }
        }
    }
    return in_ok ? 1 : (out_ok ? 0 : -1);
}

// Bounds on the covered lattice cells of window (x, y, w, w) at `grid` from the raster (one
// thread): a lattice cell lying inside a clean-inside raster cell is covered, one inside a
// clean-outside raster cell (or outside the raster) is not; cells straddling a raster cell
// border or lying in a dirty cell are unknown.  lo <= count <= hi.  The lattice spacing of
// the counts is computed in plain FP64: a lattice line can only be misplaced when it lies
// within rounding of a raster cell border, and the 1 px growth of a clean cell covers it.
__device__ inline void raster_bounds_thread(const RasterHeader* R, double x, double y, double w, int grid, int& lo,
                                            int& hi) {
    {  // a window 16 or more cells wide takes the coarse level (the common path reads <= 16 columns)
        const double ic0 = __ldg(&R->inv_cell), ox0 = __ldg(&R->ox);
        const int64_t coarse = __ldg(&R->coarse);
        if (coarse && (int)floor((x + w - ox0) * ic0) - (int)floor((x - ox0) * ic0) >= 16)
            R = reinterpret_cast<const RasterHeader*>(reinterpret_cast<const uint8_t*>(R) + coarse);
    }
    const double ox = __ldg(&R->ox), oy = __ldg(&R->oy), C = __ldg(&R->cell), ic = __ldg(&R->inv_cell);
    const int nx = __ldg(&R->nx), ny = __ldg(&R->ny), pitch = __ldg(&R->pitch);
    const uint32_t* words = reinterpret_cast<const uint32_t*>(R + 1);
    const double step = w / grid, inv = grid / w;
    // lattice intervals [k, k+1) of one axis lying in raster cell c: k from ceil((c0 - x)/step)
    // to floor((c0 + C - x)/step) - 1
    auto span = [&](double origin, double p0, int c) {
        const double c0 = origin + c * C;
        const int k0 = max(0, (int)ceil((c0 - p0) * inv));
        const int k1 = min(grid - 1, (int)floor((c0 + C - p0) * inv) - 1);
        return max(0, k1 - k0 + 1);
    };
    const int a0 = (int)floor((x - ox) * ic), a1 = (int)floor((x + w - ox) * ic);
    const int b0 = (int)floor((y - oy) * ic), b1 = (int)floor((y + w - oy) * ic);
    int in_sum = 0, out_sum = 0;
    if (a1 - a0 < 16 && a0 >= 0 && a1 < nx && b0 >= 0 && b1 < ny) {
        // common case: <= 16 columns inside the raster, their spans in registers, each row's
        // codes from one 64-bit window of its two words
        int aw[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) aw[j] = a0 + j <= a1 ? span(ox, x, a0 + j) : 0;
        const int w0 = a0 >> 4, sh = 2 * (a0 & 15);
        for (int r = b0; r <= b1; ++r) {
            const int bh = span(oy, y, r);
            const uint32_t* row = words + (size_t)r * pitch;
            const uint64_t v = (uint64_t)__ldg(row + w0) | (w0 + 1 < pitch ? (uint64_t)__ldg(row + w0 + 1) << 32 : 0ull);
            const uint32_t codes = (uint32_t)(v >> sh);
            int in_w = 0, out_w = 0;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t cd = (codes >> (2 * j)) & 3u;
                in_w += cd == 1u ? aw[j] : 0;
                out_w += cd == 0u ? aw[j] : 0;
            }
            in_sum += bh * in_w;
            out_sum += bh * out_w;
        }
        lo = in_sum;
        hi = grid * grid - out_sum;
        return;
    }
    for (int r = b0; r <= b1; ++r) {
        const int bh = span(oy, y, r);
        if (bh == 0) continue;
        const bool row_in = r >= 0 && r < ny;
        const uint32_t* row = words + (size_t)(row_in ? r : 0) * pitch;
        uint32_t v = 0;
        int vw = -1;
        for (int c = a0; c <= a1; ++c) {
            const int aw = span(ox, x, c);
            if (aw == 0) continue;
            int code = 0;  // outside the raster: clean outside
            if (row_in && c >= 0 && c < nx) {
                if ((c >> 4) != vw) {
                    vw = c >> 4;
                    v = __ldg(row + vw);
                }
                code = (v >> (2 * (c & 15))) & 3u;
            }
            if (code == 1) in_sum += aw * bh;
            else if (code == 0) out_sum += aw * bh;
        }
    }
    lo = in_sum;
    hi = grid * grid - out_sum;
}

// Smallest covered-cell count c with c / grid^2 >= min_fg in the reference's FP64 arithmetic
// (the division it performs, so the comparison is exact); grid^2 + 1 if none.
// Host and device agree: both divide in IEEE binary64 round-to-nearest.
__host__ __device__ inline int accept_cells(int grid, double min_fg) {
#ifdef __CUDA_ARCH__
#define PF_DDIV(a, b) __ddiv_rn((a), (b))
#else
#define PF_DDIV(a, b) ((a) / (b))
#endif
    const double g2 = (double)grid * (double)grid;
    int c = (int)fmax(0.0, fmin(g2, ceil(min_fg * g2)));
    while (c > 0 && PF_DDIV((double)(c - 1), g2) >= min_fg) --c;
    while (c <= (int)g2 && !(PF_DDIV((double)c, g2) >= min_fg)) ++c;
#undef PF_DDIV
    return c;
}

// overlap_fraction(rect) >= min_fg, decided without finishing the lattice when the covered
// cells so far already reach the threshold, or the rows left cannot (the sampler only needs
// the acceptance bit, pkg/sampler.py:174-179).  All lanes return the same value.
// `need` = accept_cells(grid, min_fg), hoisted out of the per-candidate path by the caller.
__device__ inline bool warp_overlap_accept(const PolyView& P, double x, double y, double w, double h, int grid,
                                           uint32_t* smem, double min_fg, int need) {
    const int c = warp_overlap_count_upto(P, x, y, w, h, grid, smem, need);
    return c < 0 ? 0.0 >= min_fg : c >= need;  // c < 0: bbox early-out, fraction 0.0
}

__device__ inline bool warp_overlap_accept(const PolyView& P, double x, double y, double w, double h, int grid,
                                           uint32_t* smem, double min_fg) {
    return warp_overlap_accept(P, x, y, w, h, grid, smem, min_fg, accept_cells(grid, min_fg));
}

}  // namespace pf
