// Host side of the foreground polygon: marching-squares tracing
// (polygon_from_mask, pkg/foreground.py:169-220) and the slab index the
// device even-odd test walks.
//
// The tracer restates the published marching-squares contour algorithm that
// the reference calls as skimage.measure.find_contours(padded, 0.5)
// (scikit-image >= 0.20, pyproject.toml:13; not installed here, so parity
// with it is unpinned): per 2x2 square in row-major order emit oriented
// segments between edge midpoints (saddles resolved with the low value
// fully connected), then assemble segments into contours in creation order,
// joining onto existing heads/tails and keeping the older contour's index.
// Built with -ffp-contract=off so every FP64 expression rounds like numpy.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/pf_b200.h"
#include "pf_poly.h"

namespace pf {
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
}  // namespace pf

namespace {

// Points are edge midpoints: store doubled (row, col) as integers.
struct Pt {
    int64_t r2, c2;
    bool operator==(const Pt& o) const { return r2 == o.r2 && c2 == o.c2; }
};
inline uint64_t key_of(const Pt& p) { return ((uint64_t)(uint32_t)p.r2 << 32) | (uint32_t)p.c2; }

struct Contour {
    std::deque<Pt> pts;
    bool alive = true;
};

// find_contours(padded mask, 0.5) with fully_connected='low'.
std::vector<std::vector<Pt>> trace(const uint8_t* mask, int h, int w) {
    const int H = h + 2, W = w + 2;
    auto val = [&](int r, int c) -> int {
        if (r <= 0 || c <= 0 || r > h || c > w) return 0;
        return mask[(size_t)(r - 1) * w + (c - 1)] ? 1 : 0;
    };
    std::vector<Contour> contours;
    std::unordered_map<uint64_t, int> starts, ends;
    starts.reserve(1 << 12);
    ends.reserve(1 << 12);

    auto add_segment = [&](Pt from, Pt to) {
        if (from == to) return;
        int tail = -1, head = -1;
        auto it = starts.find(key_of(to));
        if (it != starts.end()) {
            tail = it->second;
            starts.erase(it);
        }
        auto jt = ends.find(key_of(from));
        if (jt != ends.end()) {
            head = jt->second;
            ends.erase(jt);
        }
        if (tail >= 0 && head >= 0) {
            if (tail == head) {
                contours[head].pts.push_back(to);  // close the contour
            } else if (tail > head) {
                // tail created second: append tail to head
                auto& hd = contours[head].pts;
                auto& tl = contours[tail].pts;
                hd.insert(hd.end(), tl.begin(), tl.end());
                contours[tail].alive = false;
                tl.clear();
                starts[key_of(hd.front())] = head;
                ends[key_of(hd.back())] = head;
            } else {
                // head created second: prepend head to tail
                auto& hd = contours[head].pts;
                auto& tl = contours[tail].pts;
                tl.insert(tl.begin(), hd.begin(), hd.end());
                starts.erase(key_of(hd.front()));
                contours[head].alive = false;
                hd.clear();
                starts[key_of(tl.front())] = tail;
                ends[key_of(tl.back())] = tail;
            }
        } else if (tail < 0 && head < 0) {
            Contour c;
            c.pts.push_back(from);
            c.pts.push_back(to);
            contours.push_back(std::move(c));
            const int idx = (int)contours.size() - 1;
            starts[key_of(from)] = idx;
            ends[key_of(to)] = idx;
        } else if (head < 0) {
            contours[tail].pts.push_front(from);
            starts[key_of(from)] = tail;
        } else {
            contours[head].pts.push_back(to);
            ends[key_of(to)] = head;
        }
    };

    for (int r0 = 0; r0 < H - 1; ++r0) {
        for (int c0 = 0; c0 < W - 1; ++c0) {
            const int ul = val(r0, c0), ur = val(r0, c0 + 1);
            const int ll = val(r0 + 1, c0), lr = val(r0 + 1, c0 + 1);
            const int sc = ul + 2 * ur + 4 * ll + 8 * lr;
            if (sc == 0 || sc == 15) continue;
            const Pt top{2 * r0, 2 * c0 + 1};
            const Pt bottom{2 * r0 + 2, 2 * c0 + 1};
            const Pt left{2 * r0 + 1, 2 * c0};
            const Pt right{2 * r0 + 1, 2 * c0 + 2};
            switch (sc) {
                case 1: add_segment(top, left); break;
                case 2: add_segment(right, top); break;
                case 3: add_segment(right, left); break;
                case 4: add_segment(left, bottom); break;
                case 5: add_segment(top, bottom); break;
                case 6:  // saddle, low fully connected
                    add_segment(right, top);
                    add_segment(left, bottom);
                    break;
                case 7: add_segment(right, bottom); break;
                case 8: add_segment(bottom, right); break;
                case 9:
                    add_segment(top, left);
                    add_segment(bottom, right);
                    break;
                case 10: add_segment(bottom, top); break;
                case 11: add_segment(bottom, left); break;
                case 12: add_segment(left, right); break;
                case 13: add_segment(top, right); break;
                case 14: add_segment(left, top); break;
            }
        }
    }
    std::vector<std::vector<Pt>> out;
    for (auto& c : contours)
        if (c.alive) out.emplace_back(c.pts.begin(), c.pts.end());
    return out;
}

double shoelace(const std::vector<double>& xy, size_t n) {
    // exact for marching-squares rings (half-integer coordinates); for
    // general rings numpy's pairwise sum may differ in the last ulp.
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const size_t j = (i + 1) % n;
        s += xy[2 * i] * xy[2 * j + 1] - xy[2 * j] * xy[2 * i + 1];
    }
    return 0.5 * s;
}

// points_in_polygon for one point against one ring (foreground.py:223-243).
bool point_in_ring(double px, double py, const double* xy, size_t n) {
    int hits = 0;
    for (size_t i = 0; i < n; ++i) {
        const size_t j = (i + 1) % n;
        const double x1 = xy[2 * i], y1 = xy[2 * i + 1], x2 = xy[2 * j], y2 = xy[2 * j + 1];
        const bool crosses = (y1 > py) != (y2 > py);
        if (!crosses) continue;
        const double x_at = x1 + (py - y1) * (x2 - x1) / (y2 - y1);
        if (px < x_at) ++hits;
    }
    return (hits & 1) != 0;
}

}  // namespace

using namespace pf;

extern "C" int pf_polygon_trace(const uint8_t* mask, int32_t h, int32_t w, double scale,
                                double min_region_px, double* xy, int64_t xy_cap_points,
                                int64_t* ring_off, int32_t ring_cap, int64_t* n_points,
                                int32_t* n_rings) {
    if (!mask || h < 1 || w < 1 || !n_points || !n_rings)
        return fail(PF_ERR_INVALID_ARG, "pf_polygon_trace: bad arguments");
    if (!(scale > 0.0 && scale <= 1.0))
        return fail(PF_ERR_INVALID_ARG, "scale must be in (0, 1]");
    bool any = false;
    for (size_t i = 0; i < (size_t)h * w && !any; ++i) any = mask[i] != 0;
    if (!any) return fail(PF_ERR_EMPTY_FOREGROUND, "mask contains no foreground pixels");

    const auto contours = trace(mask, h, w);
    // (row, col) -> (x, y) - 1; drop closing duplicate; filter.
    std::vector<std::vector<double>> rings;
    for (const auto& c : contours) {
        std::vector<double> r;
        r.reserve(c.size() * 2);
        for (const auto& p : c) {
            r.push_back((double)p.c2 * 0.5 - 1.0);
            r.push_back((double)p.r2 * 0.5 - 1.0);
        }
        size_t n = c.size();
        if (n >= 1 && r[0] == r[2 * (n - 1)] && r[1] == r[2 * (n - 1) + 1]) {
            n -= 1;
            r.resize(2 * n);
        }
        if (n < 3) continue;
        if (std::fabs(shoelace(r, n)) < min_region_px) continue;
        rings.push_back(std::move(r));
    }
    if (rings.empty())
        return fail(PF_ERR_EMPTY_FOREGROUND, "no region of at least " + std::to_string(min_region_px) +
                                                 " px^2 in the mask");
    // orient by nesting depth using each ring's mean point as the probe
    int64_t total = 0;
    for (auto& r : rings) total += (int64_t)(r.size() / 2);
    *n_points = total;
    *n_rings = (int32_t)rings.size();
    if (!xy || !ring_off || xy_cap_points < total || ring_cap < (int32_t)rings.size() + 1)
        return fail(PF_ERR_CAPACITY, "pf_polygon_trace: output capacity too small");
    std::vector<std::vector<double>> oriented(rings.size());
    for (size_t i = 0; i < rings.size(); ++i) {
        const auto& r = rings[i];
        const size_t n = r.size() / 2;
        double sx = 0.0, sy = 0.0;
        for (size_t k = 0; k < n; ++k) {
            sx += r[2 * k];
            sy += r[2 * k + 1];
        }
        const double mx = sx / (double)n, my = sy / (double)n;
        int depth = 0;
        for (size_t j = 0; j < rings.size(); ++j)
            if (j != i && point_in_ring(mx, my, rings[j].data(), rings[j].size() / 2)) ++depth;
        const bool want_positive = depth % 2 == 0;
        std::vector<double> o(r.size());
        if ((shoelace(r, n) > 0) != want_positive) {
            for (size_t k = 0; k < n; ++k) {
                o[2 * k] = r[2 * (n - 1 - k)];
                o[2 * k + 1] = r[2 * (n - 1 - k) + 1];
            }
        } else {
            o = r;
        }
        for (auto& v : o) v = v / scale;
        oriented[i] = std::move(o);
    }
    int64_t off = 0;
    ring_off[0] = 0;
    for (size_t i = 0; i < oriented.size(); ++i) {
        std::memcpy(xy + 2 * off, oriented[i].data(), oriented[i].size() * sizeof(double));
        off += (int64_t)(oriented[i].size() / 2);
        ring_off[i + 1] = off;
    }
    return PF_OK;
}

namespace {

struct Built {
    std::vector<double> edges;  // 4 per edge
    std::vector<double> Y;
    std::vector<int32_t> slab_off, slab_edge, lut;
    std::vector<double> slab_lo, slab_hi;
    int32_t lut_base = 0;
    double bbox[4];
};

int build_index(const double* xy, const int64_t* ring_off, int32_t n_rings, Built& b) {
    if (!xy || !ring_off || n_rings < 1) return fail(PF_ERR_INVALID_ARG, "polygon has no rings");
    const int64_t npts = ring_off[n_rings];
    b.bbox[0] = b.bbox[1] = INFINITY;
    b.bbox[2] = b.bbox[3] = -INFINITY;
    for (int64_t i = 0; i < npts; ++i) {
        b.bbox[0] = std::min(b.bbox[0], xy[2 * i]);
        b.bbox[1] = std::min(b.bbox[1], xy[2 * i + 1]);
        b.bbox[2] = std::max(b.bbox[2], xy[2 * i]);
        b.bbox[3] = std::max(b.bbox[3], xy[2 * i + 1]);
        b.Y.push_back(xy[2 * i + 1]);
    }
    std::sort(b.Y.begin(), b.Y.end());
    b.Y.erase(std::unique(b.Y.begin(), b.Y.end()), b.Y.end());
    for (int32_t r = 0; r < n_rings; ++r) {
        const int64_t s = ring_off[r], e = ring_off[r + 1];
        if (e - s < 3) return fail(PF_ERR_INVALID_ARG, "each ring needs >= 3 (x, y) points");
        for (int64_t i = s; i < e; ++i) {
            const int64_t j = (i + 1 < e) ? i + 1 : s;  // np.roll(-1)
            b.edges.push_back(xy[2 * i]);
            b.edges.push_back(xy[2 * i + 1]);
            b.edges.push_back(xy[2 * j]);
            b.edges.push_back(xy[2 * j + 1]);
        }
    }
    const int32_t n_y = (int32_t)b.Y.size();
    const int64_t n_edges = (int64_t)b.edges.size() / 4;
    std::vector<std::vector<int32_t>> slab(std::max(n_y - 1, 0));
    for (int64_t e = 0; e < n_edges; ++e) {
        const double y1 = b.edges[4 * e + 1], y2 = b.edges[4 * e + 3];
        if (y1 == y2) continue;  // never crosses a row
        const double lo = std::min(y1, y2), hi = std::max(y1, y2);
        const int32_t k0 = (int32_t)(std::lower_bound(b.Y.begin(), b.Y.end(), lo) - b.Y.begin());
        const int32_t k1 = (int32_t)(std::lower_bound(b.Y.begin(), b.Y.end(), hi) - b.Y.begin());
        for (int32_t k = k0; k < k1; ++k) slab[k].push_back((int32_t)e);
    }
    b.slab_off.assign(std::max(n_y, 1), 0);
    for (int32_t k = 0; k + 1 < n_y; ++k) {
        auto& v = slab[k];
        const double ya = b.Y[k], yb = b.Y[k + 1], ym = 0.5 * (ya + yb);
        auto x_on = [&](int32_t e, double yy) {
            const double x1 = b.edges[4 * e], y1 = b.edges[4 * e + 1];
            const double x2 = b.edges[4 * e + 2], y2 = b.edges[4 * e + 3];
            return x1 + (yy - y1) * (x2 - x1) / (y2 - y1);
        };
        std::vector<std::pair<double, int32_t>> order;
        order.reserve(v.size());
        for (int32_t e : v) order.emplace_back(x_on(e, ym), e);
        std::stable_sort(order.begin(), order.end(),
                         [](const auto& a, const auto& c) { return a.first < c.first; });
        const size_t base = b.slab_edge.size();
        for (auto& pr : order) {
            const int32_t e = pr.second;
            const double xa = x_on(e, ya), xb = x_on(e, yb);
            const double x1 = b.edges[4 * e], x2 = b.edges[4 * e + 2];
            // conservative bounds: clipped x-range, never outside the edge's own
            double lo = std::max(std::min(xa, xb), std::min(x1, x2));
            double hi = std::min(std::max(xa, xb), std::max(x1, x2));
            const double m = 1e-6 + 1e-9 * std::max(std::fabs(lo), std::fabs(hi));
            b.slab_edge.push_back(e);
            b.slab_lo.push_back(lo - m);
            b.slab_hi.push_back(hi + m);
        }
        const size_t cnt = b.slab_edge.size() - base;
        for (size_t i = 1; i < cnt; ++i)
            b.slab_hi[base + i] = std::max(b.slab_hi[base + i], b.slab_hi[base + i - 1]);
        for (size_t i = cnt; i-- > 1;)
            b.slab_lo[base + i - 1] = std::min(b.slab_lo[base + i - 1], b.slab_lo[base + i]);
        b.slab_off[k + 1] = (int32_t)b.slab_edge.size();
    }
    // integer-row lookup table
    if (n_y >= 1) {
        const double f0 = std::floor(b.Y[0]), f1 = std::floor(b.Y[n_y - 1]);
        const double len = f1 - f0 + 1.0;
        if (len >= 1.0 && len <= 8.0 * 1024 * 1024 && std::fabs(f0) < 1e9) {
            b.lut_base = (int32_t)f0;
            b.lut.resize((size_t)len);
            int32_t k = 0;
            for (size_t i = 0; i < b.lut.size(); ++i) {
                const double yy = f0 + (double)i;
                while (k + 1 < n_y && b.Y[k + 1] <= yy) ++k;
                b.lut[i] = (b.Y[k] <= yy) ? k : -1;
            }
        }
    }
    return PF_OK;
}

int64_t layout(const Built& b, PolyHeader& h) {
    std::memset(&h, 0, sizeof(h));
    h.magic = kPolyMagic;
    h.n_edges = (int32_t)(b.edges.size() / 4);
    h.n_y = (int32_t)b.Y.size();
    h.n_entries = (int32_t)b.slab_edge.size();
    h.lut_len = (int32_t)b.lut.size();
    h.lut_base = b.lut_base;
    for (int i = 0; i < 4; ++i) h.bbox[i] = b.bbox[i];
    int64_t o = align16(sizeof(PolyHeader));
    h.off_edges = o;
    o = align16(o + (int64_t)b.edges.size() * 8);
    h.off_y = o;
    o = align16(o + (int64_t)b.Y.size() * 8);
    h.off_slab_off = o;
    o = align16(o + (int64_t)b.slab_off.size() * 4);
    h.off_slab_edge = o;
    o = align16(o + (int64_t)b.slab_edge.size() * 4);
    h.off_slab_lo = o;
    o = align16(o + (int64_t)b.slab_lo.size() * 8);
    h.off_slab_hi = o;
    o = align16(o + (int64_t)b.slab_hi.size() * 8);
    h.off_lut = o;
    o = align16(o + (int64_t)b.lut.size() * 4);
    h.total_bytes = o;
    return o;
}

}  // namespace

extern "C" int pf_polygon_index_size(const double* xy, const int64_t* ring_off, int32_t n_rings,
                                     int64_t* bytes) {
    if (!bytes) return fail(PF_ERR_INVALID_ARG, "pf_polygon_index_size: null output");
    Built b;
    const int rc = build_index(xy, ring_off, n_rings, b);
    if (rc) return rc;
    PolyHeader h;
    *bytes = layout(b, h);
    return PF_OK;
}

extern "C" int pf_polygon_index_build(const double* xy, const int64_t* ring_off, int32_t n_rings,
                                      void* blob, int64_t bytes) {
    if (!blob) return fail(PF_ERR_INVALID_ARG, "pf_polygon_index_build: null blob");
    Built b;
    const int rc = build_index(xy, ring_off, n_rings, b);
    if (rc) return rc;
    PolyHeader h;
    const int64_t need = layout(b, h);
    if (bytes < need) return fail(PF_ERR_CAPACITY, "pf_polygon_index_build: blob too small");
    uint8_t* p = static_cast<uint8_t*>(blob);
    std::memset(p, 0, (size_t)need);
    std::memcpy(p, &h, sizeof(h));
    std::memcpy(p + h.off_edges, b.edges.data(), b.edges.size() * 8);
    std::memcpy(p + h.off_y, b.Y.data(), b.Y.size() * 8);
    std::memcpy(p + h.off_slab_off, b.slab_off.data(), b.slab_off.size() * 4);
    std::memcpy(p + h.off_slab_edge, b.slab_edge.data(), b.slab_edge.size() * 4);
    std::memcpy(p + h.off_slab_lo, b.slab_lo.data(), b.slab_lo.size() * 8);
    std::memcpy(p + h.off_slab_hi, b.slab_hi.data(), b.slab_hi.size() * 8);
    if (!b.lut.empty()) std::memcpy(p + h.off_lut, b.lut.data(), b.lut.size() * 4);
    return PF_OK;
}
