// Classification raster of a ForegroundPolygon (include/pf_b200.h pf_polygon_raster_build):
// a precomputed filter in front of the sampler's overlap test (pkg/foreground.py:246-286,
// called from sample_patch, pkg/sampler.py:174-179).
//
// Two levels, cells of `cell` and 4 `cell` px (wide windows read the coarse one), each covering
// the polygon's bounding box plus one cell on every side.  A cell is
// "dirty" when some edge comes within 1 px of it; otherwise no edge meets the cell grown by
// 1 px, the even-odd parity is the same at every point of that grown cell, and the cell's
// centre (traced with the device even-odd test) gives it.  The sampler's evaluation warps
// read the 2-bit codes under a candidate window: all inside means overlap_fraction == 1.0,
// all outside 0.0, exactly; anything else falls through to the slab test and the lattice.
//
//   raster_mark_kernel      one thread per edge: every cell whose 1 px growth the edge's
//                           part inside that cell row's band (also grown) can reach -> bit 1
//   raster_classify_kernel  one thread per (cell row, 256 cells): centre parity -> bit 0
#include <cuda_runtime.h>

#include <cmath>

#include "pf_common.cuh"
#include "pf_poly.cuh"

namespace pf {
namespace {

constexpr double kEps = 1e-3;  // slack on the edge's clipped x-range (rounding of the clip)

__global__ void raster_mark_kernel(const void* blob, RasterHeader hdr, uint32_t* words) {
    const PolyHeader* h = reinterpret_cast<const PolyHeader*>(blob);
    const double* edges = reinterpret_cast<const double*>(reinterpret_cast<const uint8_t*>(blob) + h->off_edges);
    const int n_edges = h->n_edges;
    const double C = hdr.cell, ic = hdr.inv_cell;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_edges; e += gridDim.x * blockDim.x) {
        const double x1 = edges[4 * e], y1 = edges[4 * e + 1], x2 = edges[4 * e + 2], y2 = edges[4 * e + 3];
        const double ymin = fmin(y1, y2), ymax = fmax(y1, y2);
        // rows whose grown band [oy + rC - 1, oy + (r+1)C + 1] meets [ymin, ymax]
        const int r0 = max(0, (int)floor((ymin - 1.0 - hdr.oy) * ic) - 1);
        const int r1 = min(hdr.ny - 1, (int)floor((ymax + 1.0 - hdr.oy) * ic));
        for (int r = r0; r <= r1; ++r) {
            const double lo = hdr.oy + r * C - 1.0, hi = hdr.oy + (r + 1) * C + 1.0;
            const double ya = fmax(ymin, lo), yb = fmin(ymax, hi);
            if (ya > yb) continue;
            double xa, xb;
            if (y1 == y2) {
                xa = fmin(x1, x2);
                xb = fmax(x1, x2);
            } else {
                const double ta = (ya - y1) / (y2 - y1), tb = (yb - y1) / (y2 - y1);
                const double pa = x1 + ta * (x2 - x1), pb = x1 + tb * (x2 - x1);
                xa = fmin(pa, pb);
                xb = fmax(pa, pb);
            }
            // cells whose grown x-range [ox + cC - 1, ox + (c+1)C + 1] meets [xa, xb]
            const int c0 = max(0, (int)ceil((xa - kEps - 1.0 - hdr.ox) * ic) - 1);
            const int c1 = min(hdr.nx - 1, (int)floor((xb + kEps + 1.0 - hdr.ox) * ic));
            uint32_t* row = words + (size_t)r * hdr.pitch;
            PF_CHECK(r >= 0 && r < hdr.ny && (c1 < c0 || (c0 >= 0 && c1 < hdr.nx)));
            for (int c = c0; c <= c1; ++c) atomicOr(row + (c >> 4), 2u << (2 * (c & 15)));
        }
    }
}

__global__ void raster_classify_kernel(const void* blob, RasterHeader hdr, uint32_t* words) {
    const int segs = (hdr.nx + 255) / 256;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= segs * hdr.ny) return;
    const int r = t / segs, s = t % segs;
    const int n_pts = min(256, hdr.nx - 256 * s);
    const PolyView P = poly_view(blob);
    uint32_t bits[kMaxWords];
    const double py = hdr.oy + (r + 0.5) * hdr.cell;
    const double x0 = hdr.ox + (256 * s + 0.5) * hdr.cell;
    row_mask(P, py, x0, hdr.cell, false, n_pts, 8, bits);
    uint32_t* row = words + (size_t)r * hdr.pitch + 16 * s;
    for (int w = 0; w < 16 && 16 * w < n_pts; ++w) {
        const uint32_t b = (bits[w >> 1] >> (16 * (w & 1))) & 0xffffu;  // 16 cells
        uint32_t spread = 0;  // cell k's inside bit -> bit 2k
        for (int k = 0; k < 16; ++k) spread |= ((b >> k) & 1u) << (2 * k);
        row[w] |= spread;
    }
}

bool raster_geometry(const double* bbox, double cell, RasterHeader* h) {
    if (!bbox || !(cell >= 8.0) || !(cell <= 65536.0) || std::ldexp(1.0, std::ilogb(cell)) != cell) return false;
    for (int i = 0; i < 4; ++i)
        if (!std::isfinite(bbox[i])) return false;
    if (bbox[2] < bbox[0] || bbox[3] < bbox[1]) return false;
    const double fx0 = std::floor(bbox[0] / cell), fy0 = std::floor(bbox[1] / cell);
    const double nx = std::floor(bbox[2] / cell) - fx0 + 3.0, ny = std::floor(bbox[3] / cell) - fy0 + 3.0;
    if (nx * ny > (double)(1 << 28)) return false;
    *h = RasterHeader{};
    h->ox = (fx0 - 1.0) * cell;
    h->oy = (fy0 - 1.0) * cell;
    h->cell = cell;
    h->inv_cell = 1.0 / cell;
    h->nx = (int)nx;
    h->ny = (int)ny;
    h->pitch = (h->nx + 15) / 16;
    h->magic = kRasterMagic;
    return true;
}

// Levels: cell, 4 cell, ... (kRasterLevels), each header followed by its words, 16-byte aligned.
bool raster_levels(const double* bbox, double cell, RasterHeader (&hs)[kRasterLevels], int64_t (&offs)[kRasterLevels],
                   int64_t* total) {
    int64_t at = 0;
    for (int l = 0; l < kRasterLevels; ++l) {
        if (!raster_geometry(bbox, cell * (double)(1 << (2 * l)), &hs[l])) return false;
        offs[l] = at;
        at += (int64_t)sizeof(RasterHeader) + ((int64_t)hs[l].ny * hs[l].pitch * 4 + 15) / 16 * 16;
    }
    for (int l = 0; l + 1 < kRasterLevels; ++l) hs[l].coarse = offs[l + 1] - offs[l];
    *total = at;
    return true;
}

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" int pf_polygon_raster_bytes(const double* bbox, double cell, int64_t* bytes) {
    RasterHeader hs[kRasterLevels];
    int64_t offs[kRasterLevels];
    if (!bytes || !raster_levels(bbox, cell, hs, offs, bytes))
        return fail(PF_ERR_INVALID_ARG, "pf_polygon_raster_bytes: bad bbox or cell (power of two, 8..16384)");
    return PF_OK;
}

extern "C" int pf_polygon_raster_build(const void* poly_blob_dev, const double* bbox, double cell, void* raster_dev,
                                       int64_t raster_bytes, void* stream) {
    RasterHeader hs[kRasterLevels];
    int64_t offs[kRasterLevels], need = 0;
    if (!poly_blob_dev || !raster_dev || !raster_levels(bbox, cell, hs, offs, &need))
        return fail(PF_ERR_INVALID_ARG, "pf_polygon_raster_build: bad arguments");
    if (raster_bytes < need) return fail(PF_ERR_INVALID_ARG, "pf_polygon_raster_build: raster buffer too small");
    cudaStream_t st = as_stream(stream);
    int rc = PF_OK;
    for (int l = 0; l < kRasterLevels; ++l) {
        const RasterHeader& h = hs[l];
        uint8_t* out = reinterpret_cast<uint8_t*>(raster_dev) + offs[l];
        uint32_t* words = reinterpret_cast<uint32_t*>(out + sizeof(RasterHeader));
        if ((rc = check_cuda(cudaMemcpyAsync(out, &h, sizeof(h), cudaMemcpyHostToDevice, st), "cudaMemcpyAsync")))
            return rc;
        if ((rc = check_cuda(cudaMemsetAsync(words, 0, (size_t)h.ny * h.pitch * 4, st), "cudaMemsetAsync"))) return rc;
        raster_mark_kernel<<<592, 256, 0, st>>>(poly_blob_dev, h, words);
        if ((rc = after_launch("raster_mark_kernel"))) return rc;
        const int threads = ((h.nx + 255) / 256) * h.ny;
        raster_classify_kernel<<<(threads + 127) / 128, 128, 0, st>>>(poly_blob_dev, h, words);
        if ((rc = after_launch("raster_classify_kernel"))) return rc;
    }
    // the headers are copied from this stack frame: finish before returning
    return check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize");
}
