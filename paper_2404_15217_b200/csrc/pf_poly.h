// Polygon slab index blob shared by the host builder (pf_polygon.cpp) and the
// device even-odd test (pf_poly.cuh).
#pragma once
#include <stdint.h>

namespace pf {

// Blob = header | edges (x1,y1,x2,y2 f64)[n_edges] | Y f64[n_y] |
//        slab_off i32[n_y] | slab_edge i32[n_entries] | slab_lo f64[n_entries] |
//        slab_hi f64[n_entries] | row_lut i32[lut_len]
// Slab k (0 <= k < n_y-1) is [Y[k], Y[k+1]); its edges are
// slab_edge[slab_off[k] .. slab_off[k+1]) ordered left to right, with
// conservative x-bounds made monotone (lo: suffix-min, hi: prefix-max) so
// that "entirely right of x" / "entirely left of x" are a suffix / prefix.
// row_lut[i] = largest k with Y[k] <= lut_base + i.
struct PolyHeader {
    int64_t total_bytes;
    int32_t n_edges, n_y, n_entries, lut_len;
    int32_t lut_base, magic;
    double bbox[4];
    int64_t off_edges, off_y, off_slab_off, off_slab_edge, off_slab_lo, off_slab_hi, off_lut;
};

constexpr int32_t kPolyMagic = 0x50464231;  // "PFB1"

// Classification raster (pf_polygon_raster_build): header | uint32 words[ny][pitch], 16
// cells of 2 bits per word (cell c of a row at bits 2(c%16), 2(c%16)+1 of word c/16).
struct RasterHeader {
    double ox, oy, cell, inv_cell;  // cell (i, j) covers [ox + i*cell, ox + (i+1)*cell) x ...
    int32_t nx, ny, pitch, magic;
    int64_t coarse;                 // byte offset of the next (4x coarser) level's header, or 0
    int64_t _reserved;
};
constexpr int kRasterLevels = 2;   // cell and 4 * cell: windows up to ~15 cells wide at either
constexpr int32_t kRasterMagic = 0x50465231;  // "PFR1"
constexpr uint32_t kRasterInside = 0x55555555u;

inline int64_t align16(int64_t v) { return (v + 15) & ~int64_t(15); }

}  // namespace pf
