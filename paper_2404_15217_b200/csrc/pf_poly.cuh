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

__device__ __forceinline__ double edge_x_at(const PolyView& P, int e, double py) {
    const double x1 = __ldg(P.edges + 4 * e), y1 = __ldg(P.edges + 4 * e + 1);
    const double x2 = __ldg(P.edges + 4 * e + 2), y2 = __ldg(P.edges + 4 * e + 3);
    return __dadd_rn(x1, __ddiv_rn(__dmul_rn(__dsub_rn(py, y1), __dsub_rn(x2, x1)), __dsub_rn(y2, y1)));
}

// Lattice coordinate k of a row: corner rows use edges e_k = x0 + k*step,
// centre rows (e_k + e_{k+1}) / 2.
__device__ __forceinline__ double lattice(double x0, double step, int k, bool centre) {
    const double ek = __dadd_rn(x0, __dmul_rn((double)k, step));
    if (!centre) return ek;
    const double ek1 = __dadd_rn(x0, __dmul_rn((double)(k + 1), step));
    return __dmul_rn(__dadd_rn(ek, ek1), 0.5);  // == / 2.0 exactly (no subnormals here)
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
    const int i_hi = a;
    if ((e1 - i_hi) & 1) {
        for (int j = 0; j < nw; ++j) {
            const int rem = n_pts - 32 * j;
            words[j] = rem >= 32 ? 0xffffffffu : (rem > 0 ? ((1u << rem) - 1u) : 0u);
        }
    }
    const double inv = 1.0 / step;  // estimate only: the walk below is exact
    for (int i = i_lo; i < i_hi; ++i) {
        const double X = edge_x_at(P, __ldg(P.slab_edge + i), py);
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

constexpr int kMaxGrid = 256;
constexpr int kMaxWords = (kMaxGrid + 1 + 31) / 32;  // 9

__host__ __device__ constexpr int overlap_words(int grid) { return (grid + 1 + 31) / 32; }
// shared bytes one warp needs for a grid
__host__ __device__ constexpr int overlap_smem_bytes(int grid) {
    return (2 * grid + 1) * overlap_words(grid) * 4;
}
// ... when it only counts with a stop (rows traced in chunks of 32: warp_overlap_accept)
__host__ __device__ constexpr int overlap_smem_bytes_chunked(int grid) {
    return (2 * (grid < 32 ? grid : 32) + 1) * overlap_words(grid) * 4;
}

// Covered cells of lattice cell rows [r_lo, r_hi): corner rows r_lo..r_hi and centre rows
// r_lo..r_hi-1 are traced into `smem`, then counted.  With stop >= 0 the rows are taken in
// chunks of 32 and the count returns early once it reaches `stop` or can no longer reach it
// (the returned value is then only compared against `stop`).
__device__ inline int warp_overlap_rows(const PolyView& P, double x, double y, double sx, double sy, int grid,
                                        uint32_t* smem, int r_lo, int r_hi, int stop) {
    const int lane = threadIdx.x & 31;
    const int nw = overlap_words(grid);
    const int chunk = stop >= 0 ? 32 : grid;
    uint32_t* corner = smem;                    // chunk + 1 rows
    uint32_t* centre = smem + (chunk + 1) * nw;  // chunk rows
    uint32_t words[kMaxWords];
    int total = 0;
    for (int c0 = r_lo; c0 < r_hi; c0 += chunk) {
        const int nrow = min(chunk, r_hi - c0);
        const int n_rows = 2 * nrow + 1;
        for (int ri = lane; ri < n_rows; ri += 32) {
            const bool is_centre = ri > nrow;
            const int r = is_centre ? ri - nrow - 1 : ri;
            const double py = lattice(y, sy, c0 + r, is_centre);
            row_mask(P, py, x, sx, is_centre, is_centre ? grid : grid + 1, nw, words);
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
        const int ka = y >= Yfirst ? slab_of(P, y) : 0;
        const int kb = ylast < Ylast ? slab_of(P, ylast) : P.n_y - 2;
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
    }
    return warp_overlap_rows(P, x, y, sx, sy, grid, smem, 0, grid, stop);
}

__device__ inline int warp_overlap_count(const PolyView& P, double x, double y, double w, double h, int grid,
                                         uint32_t* smem) {
    return warp_overlap_count_upto(P, x, y, w, h, grid, smem, -1);
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
