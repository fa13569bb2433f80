// On-GPU polygon_from_mask (pkg/foreground.py:169-220): the tissue mask
// never leaves HBM.  Same output as the host tracer (csrc/pf_polygon.cpp) and the reference run
// with the oracle's find_contours restatement, ring for ring and vertex for vertex:
//
//  1. marching squares on the 1-px zero-padded mask at iso 0.5, saddles low-connected: every
//     2x2 cell emits 0..2 directed segments between edge midpoints, in row-major cell order
//     (the order skimage.measure.find_contours scans, pkg/foreground.py:184);
//  2. every midpoint starts exactly one segment and ends exactly one, so the segments form
//     disjoint cycles: succ(k) = the segment starting where k ends;
//  3. find_contours' assembly (join onto existing heads / tails, keep the older contour's
//     index) is replaced by what it provably produces: a ring's index is that of its
//     first-scanned segment (rings ordered by it), and the ring is closed by its last-scanned
//     segment L, so the ring starts at L's end point and follows the segment direction.
//     Pointer jumping over succ gives every segment its cycle's first / last segment and its
//     distance to L (list ranking), i.e. its position in the ring;
//  4. (row, col) -> (x, y) - 1; rings with |shoelace area| < min_region_px dropped -- the area
//     is exact in integers (doubled coordinates), as is numpy's on half-integer vertices;
//  5. nesting depth of each kept ring's vertex-mean probe against every other kept ring with
//     the reference's FP64 even-odd test (foreground.py:223-243, same edge direction and
//     expression order), reversal when (area > 0) != (depth even), division by the scale.
#include <cuda_runtime.h>

#include <algorithm>
#include <cub/device/device_scan.cuh>
#include <string>

#include "pf_common.cuh"

namespace pf {
namespace {

constexpr int kTB = 256;

// Vertex ids of the padded H x W grid: horizontal-edge midpoints (r, c + 1/2), r < H, c < W - 1,
// then vertical-edge midpoints (r + 1/2, c), r < H - 1, c < W.
struct Grid {
    int h, w, H, W;
    __device__ int hid(int r, int c) const { return r * (W - 1) + c; }
    __device__ int vid(int r, int c) const { return H * (W - 1) + r * W + c; }
    // doubled (row, col) of a vertex id
    __device__ void coords2(int v, int& r2, int& c2) const {
        const int nh = H * (W - 1);
        if (v < nh) {
            const int r = v / (W - 1), c = v - r * (W - 1);
            r2 = 2 * r;
            c2 = 2 * c + 1;
        } else {
            v -= nh;
            const int r = v / W, c = v - r * W;
            r2 = 2 * r + 1;
            c2 = 2 * c;
        }
    }
    __device__ int val(const uint8_t* m, int r, int c) const {  // padded mask value
        return (r <= 0 || c <= 0 || r > h || c > w) ? 0 : (m[(size_t)(r - 1) * w + (c - 1)] ? 1 : 0);
    }
    __device__ int cell_case(const uint8_t* m, int r0, int c0) const {
        return val(m, r0, c0) | (val(m, r0, c0 + 1) << 1) | (val(m, r0 + 1, c0) << 2) | (val(m, r0 + 1, c0 + 1) << 3);
    }
};

__device__ __forceinline__ int seg_count(int sc) { return (sc == 0 || sc == 15) ? 0 : ((sc == 6 || sc == 9) ? 2 : 1); }

// segment `slot` of a cell case: (from, to) as top/bottom/left/right of the cell (the host
// tracer's table, pf_polygon.cpp)
__device__ void seg_of(const Grid& g, int r0, int c0, int sc, int slot, int& from, int& to) {
    const int top = g.hid(r0, c0), bottom = g.hid(r0 + 1, c0), left = g.vid(r0, c0), right = g.vid(r0, c0 + 1);
    switch (sc) {
        case 1: from = top, to = left; break;
        case 2: from = right, to = top; break;
        case 3: from = right, to = left; break;
        case 4: from = left, to = bottom; break;
        case 5: from = top, to = bottom; break;
        case 6: if (slot == 0) from = right, to = top; else from = left, to = bottom; break;
        case 7: from = right, to = bottom; break;
        case 8: from = bottom, to = right; break;
        case 9: if (slot == 0) from = top, to = left; else from = bottom, to = right; break;
        case 10: from = bottom, to = top; break;
        case 11: from = bottom, to = left; break;
        case 12: from = left, to = right; break;
        case 13: from = top, to = right; break;
        default: from = left, to = top; break;  // 14
    }
}

__global__ void count_kernel(Grid g, const uint8_t* mask, int* cnt, int ncells, int* any) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncells; i += gridDim.x * blockDim.x) {
        const int r0 = i / (g.W - 1), c0 = i - r0 * (g.W - 1);
        const int sc = g.cell_case(mask, r0, c0);
        cnt[i] = seg_count(sc);
        if (sc == 8) *any = 1;  // a foreground pixel's upper-left cell (the padding makes one exist)
    }
}

__global__ void emit_kernel(Grid g, const uint8_t* mask, const int* off, int ncells, int* sfrom, int* sto, int* start_of) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ncells; i += gridDim.x * blockDim.x) {
        const int r0 = i / (g.W - 1), c0 = i - r0 * (g.W - 1);
        const int sc = g.cell_case(mask, r0, c0);
        const int n = seg_count(sc);
        for (int s = 0; s < n; ++s) {
            int f, t;
            seg_of(g, r0, c0, sc, s, f, t);
            const int k = off[i] + s;
            sfrom[k] = f;
            sto[k] = t;
            start_of[f] = k;
        }
    }
}

__global__ void succ_kernel(const int* sto, const int* start_of, int n, int* succ, int* jmp, int* mn, int* mx) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int s = start_of[sto[k]];
        succ[k] = s;
        jmp[k] = s;
        mn[k] = min(k, s);
        mx[k] = max(k, s);
    }
}

// one doubling round of cycle min / max: covers 2^(r+1) consecutive segments afterwards
__global__ void minmax_round(int n, const int* jmp, const int* mn, const int* mx, int* jmp2, int* mn2, int* mx2) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int j = jmp[k];
        mn2[k] = min(mn[k], mn[j]);
        mx2[k] = max(mx[k], mx[j]);
        jmp2[k] = jmp[j];
    }
}

// list ranking towards the cycle's last-scanned segment L (terminal: a self loop of weight 0)
__global__ void rank_init(int n, const int* succ, const int* mx, int* nxt, int* d) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const bool last = mx[k] == k;
        nxt[k] = last ? k : succ[k];
        d[k] = last ? 0 : 1;
    }
}

__global__ void rank_round(int n, const int* nxt, const int* d, int* nxt2, int* d2) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int j = nxt[k];
        d2[k] = d[k] + d[j];
        nxt2[k] = nxt[j];
    }
}

// per ring (indexed by its first segment): length, exact doubled-coordinate sums
struct RingAcc {
    long long area8;  // 8 * shoelace area = sum of X_p Y_q - X_q Y_p over segments (X = 2x)
    long long sx2, sy2;  // sums of 2x, 2y over the ring's vertices
    int len;
    int last;  // last-scanned segment
};

__global__ void ring_flag_kernel(int n, const int* mn, int* is_first) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) is_first[k] = mn[k] == k;
}

__global__ void ring_acc_kernel(Grid g, int n, const int* sfrom, const int* sto, const int* mn, const int* mx,
                                const int* d, const int* ring_of_first, RingAcc* acc) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int ri = ring_of_first[mn[k]];
        int pr, pc, qr, qc;
        g.coords2(sfrom[k], pr, pc);
        g.coords2(sto[k], qr, qc);
        const long long Xp = pc - 2, Yp = pr - 2, Xq = qc - 2, Yq = qr - 2;  // 2 * ((col, row) - 1)
        atomicAdd(reinterpret_cast<unsigned long long*>(&acc[ri].area8), (unsigned long long)(Xp * Yq - Xq * Yp));
        atomicAdd(reinterpret_cast<unsigned long long*>(&acc[ri].sx2), (unsigned long long)Xp);
        atomicAdd(reinterpret_cast<unsigned long long*>(&acc[ri].sy2), (unsigned long long)Yp);
        if (mx[k] == k) {
            acc[ri].last = k;
        }
        atomicAdd(&acc[ri].len, 1);
        (void)d;
    }
}

__global__ void keep_kernel(int nr, const RingAcc* acc, double min_region_px, int* keep, int* keep_len) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += gridDim.x * blockDim.x) {
        const double area = (double)acc[i].area8 / 8.0;  // exact (|area8| < 2^53)
        const bool k = acc[i].len >= 3 && !(fabs(area) < min_region_px);
        keep[i] = k;
        keep_len[i] = k ? acc[i].len : 0;
    }
}

// parity[(i - i0) * nk + j]: crossings (mod 2) of kept ring i's probe, i in [i0, i1), with the
// edges of kept ring j -- points_in_polygon(probe, [ring_j]) (foreground.py:223-243)
__global__ void depth_kernel(Grid g, int n, const int* sfrom, const int* sto, const int* mn, const int* ring_of_first,
                             const int* keep, const int* kept_index, int nk, int i0, int i1, const double* probe,
                             int* parity) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int rj = ring_of_first[mn[k]];
        if (!keep[rj]) continue;
        const int j = kept_index[rj];
        int pr, pc, qr, qc;
        g.coords2(sfrom[k], pr, pc);
        g.coords2(sto[k], qr, qc);
        const double x1 = (double)pc * 0.5 - 1.0, y1 = (double)pr * 0.5 - 1.0;
        const double x2 = (double)qc * 0.5 - 1.0, y2 = (double)qr * 0.5 - 1.0;
        for (int i = i0; i < i1; ++i) {
            if (i == j) continue;
            const double px = probe[2 * i], py = probe[2 * i + 1];
            if ((y1 > py) == (y2 > py)) continue;
            const double x_at = __dadd_rn(x1, __ddiv_rn(__dmul_rn(__dsub_rn(py, y1), __dsub_rn(x2, x1)), __dsub_rn(y2, y1)));
            if (px < x_at) atomicXor(parity + (size_t)(i - i0) * nk + j, 1);
        }
    }
}

// depth[i] = number of other kept rings whose even-odd test contains probe i
__global__ void depth_reduce_kernel(int nk, int i0, int i1, const int* parity, int* depth) {
    for (int i = i0 + blockIdx.x * blockDim.x + threadIdx.x; i < i1; i += gridDim.x * blockDim.x) {
        int d = 0;
        for (int j = 0; j < nk; ++j) d += parity[(size_t)(i - i0) * nk + j];
        depth[i] = d;
    }
}

__global__ void probe_kernel(int nr, const RingAcc* acc, const int* keep, const int* kept_index, double* probe) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += gridDim.x * blockDim.x) {
        if (!keep[i]) continue;
        const int q = kept_index[i];
        const double n = (double)acc[i].len;
        probe[2 * q] = __ddiv_rn((double)acc[i].sx2 * 0.5, n);  // numpy mean: exact sum / n
        probe[2 * q + 1] = __ddiv_rn((double)acc[i].sy2 * 0.5, n);
    }
}

__global__ void write_kernel(Grid g, int n, const int* sfrom, const int* mn, const int* d, const int* ring_of_first,
                             const RingAcc* acc, const int* keep, const int* kept_index, const long long* pt_off,
                             const int* depth_of, double scale, double* xy) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int ri = ring_of_first[mn[k]];
        if (!keep[ri]) continue;
        const int q = kept_index[ri];
        const int len = acc[ri].len;
        int pos = len - 1 - d[k];  // the ring starts at the end point of its last-scanned segment
        const bool want_positive = (depth_of[q] & 1) == 0;
        if ((acc[ri].area8 > 0) != want_positive) pos = len - 1 - pos;  // ring[::-1]
        int r2, c2;
        g.coords2(sfrom[k], r2, c2);
        const long long o = pt_off[q] + pos;
        xy[2 * o] = __ddiv_rn((double)c2 * 0.5 - 1.0, scale);
        xy[2 * o + 1] = __ddiv_rn((double)r2 * 0.5 - 1.0, scale);
    }
}

__global__ void ring_off_kernel(int nk, const long long* pt_off, const int* keep_len_kept, long long* ring_off) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= nk; i += gridDim.x * blockDim.x)
        ring_off[i] = i < nk ? pt_off[i] : (nk ? pt_off[nk - 1] + keep_len_kept[nk - 1] : 0);
}

__global__ void gather_kept_kernel(int nr, const int* keep, const int* kept_index, const int* keep_len, long long* len_kept,
                                   int* len_kept32) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nr; i += gridDim.x * blockDim.x)
        if (keep[i]) {
            len_kept[kept_index[i]] = keep_len[i];
            len_kept32[kept_index[i]] = keep_len[i];
        }
}

int blocks_for(long long n) { return (int)std::min<long long>((n + kTB - 1) / kTB, 148LL * 16); }

// bump allocator over the caller's scratch
struct Bump {
    uint8_t* p;
    int64_t left;
    template <typename T>
    T* take(int64_t count) {
        const int64_t b = (count * (int64_t)sizeof(T) + 255) / 256 * 256;
        if (b > left) return nullptr;
        T* r = reinterpret_cast<T*>(p);
        p += b;
        left -= b;
        return r;
    }
};

}  // namespace
}  // namespace pf

using namespace pf;

extern "C" int pf_polygon_trace_device_scratch_bytes(int32_t h, int32_t w, int64_t* bytes) {
    if (h < 1 || w < 1 || !bytes) return fail(PF_ERR_INVALID_ARG, "pf_polygon_trace_device_scratch_bytes: bad arguments");
    const int64_t H = h + 2, W = w + 2;
    const int64_t cells = (H - 1) * (W - 1);
    const int64_t segs = 2 * cells, verts = H * (W - 1) + (H - 1) * W;
    size_t cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (int*)nullptr, (int*)nullptr, (int)segs);
    size_t cub2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub2, (long long*)nullptr, (long long*)nullptr, (int)segs);
    // cnt/off (cells), from/to/succ/jmp x2/mn x2/mx x2/d x2/nxt x2 (segs), start_of (verts),
    // is_first/ring_of_first (segs), per-ring arrays (<= segs / 4 rings), scans, parity
    const int64_t rings = segs / 4 + 1;
    *bytes = 2 * cells * 4 + 14 * segs * 4 + verts * 4 + rings * (int64_t)(sizeof(RingAcc) + 8 * 8) +
             (int64_t)std::max(cub_bytes, cub2) + 64 * 256 + 16 * 1024 * 1024;  // + parity blocks
    return PF_OK;
}

extern "C" int pf_polygon_trace_device(const uint8_t* mask_dev, int32_t h, int32_t w, double scale, double min_region_px,
                                       void* scratch, int64_t scratch_bytes, double* xy_dev, int64_t xy_cap_points,
                                       int64_t* ring_off_dev, int32_t ring_cap, int64_t* n_points, int32_t* n_rings,
                                       void* stream) {
    if (!mask_dev || h < 1 || w < 1 || !scratch || !n_points || !n_rings)
        return fail(PF_ERR_INVALID_ARG, "pf_polygon_trace_device: bad arguments");
    if (!(scale > 0.0 && scale <= 1.0)) return fail(PF_ERR_INVALID_ARG, "scale must be in (0, 1]");
    cudaStream_t st = as_stream(stream);
    Grid g{h, w, h + 2, w + 2};
    const int ncells = (g.H - 1) * (g.W - 1);
    const int64_t verts = (int64_t)g.H * (g.W - 1) + (int64_t)(g.H - 1) * g.W;
    Bump b{static_cast<uint8_t*>(scratch), scratch_bytes};
    int* cnt = b.take<int>(ncells + 1);
    int* off = b.take<int>(ncells + 1);
    int* start_of = b.take<int>(verts);
    int* flag = b.take<int>(64);
    size_t cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, cnt, off, ncells + 1, st);
    void* cub_tmp = b.take<uint8_t>((int64_t)cub_bytes + 256);
    if (!cnt || !off || !start_of || !flag || !cub_tmp)
        return fail(PF_ERR_CAPACITY, "pf_polygon_trace_device: scratch too small");
    int rc;
    if ((rc = check_cuda(cudaMemsetAsync(flag, 0, 64 * sizeof(int), st), "cudaMemsetAsync"))) return rc;
    if ((rc = check_cuda(cudaMemsetAsync(cnt + ncells, 0, sizeof(int), st), "cudaMemsetAsync"))) return rc;
    count_kernel<<<blocks_for(ncells), kTB, 0, st>>>(g, mask_dev, cnt, ncells, flag);
    if ((rc = after_launch("count_kernel"))) return rc;
    size_t tb = cub_bytes;
    if ((rc = check_cuda(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, cnt, off, ncells + 1, st), "cub scan"))) return rc;
    int host[2] = {0, 0};
    if ((rc = check_cuda(cudaMemcpyAsync(&host[0], off + ncells, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H")))
        return rc;
    if ((rc = check_cuda(cudaMemcpyAsync(&host[1], flag, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H"))) return rc;
    if ((rc = check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
    const int nseg = host[0];
    if (!host[1] || nseg == 0) return fail(PF_ERR_EMPTY_FOREGROUND, "mask contains no foreground pixels");
    int* sfrom = b.take<int>(nseg);
    int* sto = b.take<int>(nseg);
    int* succ = b.take<int>(nseg);
    int* jA = b.take<int>(nseg);
    int* jB = b.take<int>(nseg);
    int* mnA = b.take<int>(nseg);
    int* mnB = b.take<int>(nseg);
    int* mxA = b.take<int>(nseg);
    int* mxB = b.take<int>(nseg);
    int* dA = b.take<int>(nseg);
    int* dB = b.take<int>(nseg);
    int* is_first = b.take<int>(nseg + 1);
    int* ring_of_first = b.take<int>(nseg + 1);
    if (!sfrom || !sto || !succ || !jA || !jB || !mnA || !mnB || !mxA || !mxB || !dA || !dB || !is_first || !ring_of_first)
        return fail(PF_ERR_CAPACITY, "pf_polygon_trace_device: scratch too small");
    emit_kernel<<<blocks_for(ncells), kTB, 0, st>>>(g, mask_dev, off, ncells, sfrom, sto, start_of);
    if ((rc = after_launch("emit_kernel"))) return rc;
    succ_kernel<<<blocks_for(nseg), kTB, 0, st>>>(sto, start_of, nseg, succ, jA, mnA, mxA);
    if ((rc = after_launch("succ_kernel"))) return rc;
    int rounds = 1;
    while ((1LL << rounds) < (long long)nseg + 1) ++rounds;
    for (int r = 0; r < rounds; ++r) {  // now 2^(r+1) segments covered
        minmax_round<<<blocks_for(nseg), kTB, 0, st>>>(nseg, jA, mnA, mxA, jB, mnB, mxB);
        if ((rc = after_launch("minmax_round"))) return rc;
        std::swap(jA, jB);
        std::swap(mnA, mnB);
        std::swap(mxA, mxB);
    }
    int* nxA = jB;  // reuse
    int* nxB = mnB;
    rank_init<<<blocks_for(nseg), kTB, 0, st>>>(nseg, succ, mxA, nxA, dA);
    if ((rc = after_launch("rank_init"))) return rc;
    for (int r = 0; r < rounds; ++r) {
        rank_round<<<blocks_for(nseg), kTB, 0, st>>>(nseg, nxA, dA, nxB, dB);
        if ((rc = after_launch("rank_round"))) return rc;
        std::swap(nxA, nxB);
        std::swap(dA, dB);
    }
    // rings = cycles, indexed in scan order of their first segment
    ring_flag_kernel<<<blocks_for(nseg), kTB, 0, st>>>(nseg, mnA, is_first);
    if ((rc = after_launch("ring_flag_kernel"))) return rc;
    if ((rc = check_cuda(cudaMemsetAsync(is_first + nseg, 0, sizeof(int), st), "cudaMemsetAsync"))) return rc;
    tb = cub_bytes;
    if ((rc = check_cuda(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, is_first, ring_of_first, nseg + 1, st), "cub scan")))
        return rc;
    if ((rc = check_cuda(cudaMemcpyAsync(&host[0], ring_of_first + nseg, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H")))
        return rc;
    if ((rc = check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
    const int nr = host[0];
    RingAcc* acc = b.take<RingAcc>(nr);
    int* keep = b.take<int>(nr + 1);
    int* keep_len = b.take<int>(nr + 1);
    int* kept_index = b.take<int>(nr + 1);
    if (!acc || !keep || !keep_len || !kept_index) return fail(PF_ERR_CAPACITY, "pf_polygon_trace_device: scratch too small");
    if ((rc = check_cuda(cudaMemsetAsync(acc, 0, sizeof(RingAcc) * nr, st), "cudaMemsetAsync"))) return rc;
    ring_acc_kernel<<<blocks_for(nseg), kTB, 0, st>>>(g, nseg, sfrom, sto, mnA, mxA, dA, ring_of_first, acc);
    if ((rc = after_launch("ring_acc_kernel"))) return rc;
    keep_kernel<<<blocks_for(nr), kTB, 0, st>>>(nr, acc, min_region_px, keep, keep_len);
    if ((rc = after_launch("keep_kernel"))) return rc;
    if ((rc = check_cuda(cudaMemsetAsync(keep + nr, 0, sizeof(int), st), "cudaMemsetAsync"))) return rc;
    tb = cub_bytes;
    if ((rc = check_cuda(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, keep, kept_index, nr + 1, st), "cub scan"))) return rc;
    if ((rc = check_cuda(cudaMemcpyAsync(&host[0], kept_index + nr, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H")))
        return rc;
    if ((rc = check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
    const int nk = host[0];
    if (nk == 0)
        return fail(PF_ERR_EMPTY_FOREGROUND, "no region of at least " + std::to_string(min_region_px) + " px^2 in the mask");
    long long* len_kept = b.take<long long>(nk + 1);
    int* len_kept32 = b.take<int>(nk + 1);
    long long* pt_off = b.take<long long>(nk + 1);
    double* probe = b.take<double>(2 * nk);
    int* depth = b.take<int>(nk);
    // probes in chunks: the parity block holds chunk x nk words
    const int64_t par_words = std::max<int64_t>(nk, std::min<int64_t>((int64_t)nk * nk, (b.left - 4096) / 4));
    int* parity = b.take<int>(par_words);
    if (!len_kept || !len_kept32 || !pt_off || !probe || !depth || !parity)
        return fail(PF_ERR_CAPACITY, "pf_polygon_trace_device: scratch too small (too many rings)");
    const int chunk = (int)std::max<int64_t>(1, par_words / nk);
    gather_kept_kernel<<<blocks_for(nr), kTB, 0, st>>>(nr, keep, kept_index, keep_len, len_kept, len_kept32);
    if ((rc = after_launch("gather_kept_kernel"))) return rc;
    size_t cub3 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub3, len_kept, pt_off, nk, st);
    if (cub3 > cub_bytes + 256) return fail(PF_ERR_CAPACITY, "pf_polygon_trace_device: scan scratch");
    tb = cub_bytes + 256;
    if ((rc = check_cuda(cub::DeviceScan::ExclusiveSum(cub_tmp, tb, len_kept, pt_off, nk, st), "cub scan"))) return rc;
    long long tot[2] = {0, 0};
    if ((rc = check_cuda(cudaMemcpyAsync(&tot[0], pt_off + nk - 1, sizeof(long long), cudaMemcpyDeviceToHost, st), "D2H")))
        return rc;
    if ((rc = check_cuda(cudaMemcpyAsync(&tot[1], len_kept + nk - 1, sizeof(long long), cudaMemcpyDeviceToHost, st), "D2H")))
        return rc;
    if ((rc = check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
    *n_points = tot[0] + tot[1];
    *n_rings = nk;
    if (!xy_dev || !ring_off_dev || xy_cap_points < *n_points || ring_cap < nk + 1)
        return fail(PF_ERR_CAPACITY, "pf_polygon_trace_device: output capacity too small");
    probe_kernel<<<blocks_for(nr), kTB, 0, st>>>(nr, acc, keep, kept_index, probe);
    if ((rc = after_launch("probe_kernel"))) return rc;
    for (int i0 = 0; i0 < nk; i0 += chunk) {
        const int i1 = std::min(nk, i0 + chunk);
        if ((rc = check_cuda(cudaMemsetAsync(parity, 0, sizeof(int) * (size_t)(i1 - i0) * nk, st), "cudaMemsetAsync")))
            return rc;
        depth_kernel<<<blocks_for(nseg), kTB, 0, st>>>(g, nseg, sfrom, sto, mnA, ring_of_first, keep, kept_index, nk, i0,
                                                       i1, probe, parity);
        if ((rc = after_launch("depth_kernel"))) return rc;
        depth_reduce_kernel<<<blocks_for(i1 - i0), kTB, 0, st>>>(nk, i0, i1, parity, depth);
        if ((rc = after_launch("depth_reduce_kernel"))) return rc;
    }
    write_kernel<<<blocks_for(nseg), kTB, 0, st>>>(g, nseg, sfrom, mnA, dA, ring_of_first, acc, keep, kept_index, pt_off,
                                                   depth, scale, xy_dev);
    if ((rc = after_launch("write_kernel"))) return rc;
    ring_off_kernel<<<blocks_for(nk + 1), kTB, 0, st>>>(nk, pt_off, len_kept32, reinterpret_cast<long long*>(ring_off_dev));
    return after_launch("ring_off_kernel");
}
