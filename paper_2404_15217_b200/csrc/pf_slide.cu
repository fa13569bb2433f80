// Library-owned slide handles (SURVEY.md §8(b) "Ownership"): a C caller without torch creates a
// slide, uploads level-0 pixels or store tiles, builds the pyramid and passes the descriptor to
// the batched entry points.  Replaces the reference's Slide object lifecycle (open_slide /
// SlideRecord, pkg/store.py:123-237, 727-751) for an HBM-resident pyramid: the reference reads
// tiles on demand through TileCache (pkg/store.py:270-319); here every level lives in HBM.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>

#include "pf_common.cuh"

struct pf_slide {
    pf_slide_desc desc;
    int32_t factor;
    int32_t* status_dev;
    std::vector<void*> allocs;
};

namespace pf {

// level-0 HWC rows [y0, y0 + rows) (row stride `stride` bytes, device) -> tiles of level 0
__global__ void tile_rows_kernel(pf_slide_desc s, const uint8_t* src, int64_t stride, int y0, int rows) {
    const int y = y0 + blockIdx.y;
    if (blockIdx.y >= rows) return;
    const int W = s.width[0], T = s.tile_size;
    const int ty = y / T, v = y - ty * T;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < W * 3; b += gridDim.x * blockDim.x) {
        const int x = b / 3, c = b - x * 3;
        const int tx = x / T, u = x - tx * T;
        uint8_t* dst = const_cast<uint8_t*>(tile_ptr(s, 0, tx, ty)) + ((size_t)v * T + u) * 3 + c;
        *dst = src[(size_t)blockIdx.y * stride + b];
    }
}

}  // namespace pf

using namespace pf;

extern "C" int pf_slide_create(int32_t width, int32_t height, double base_mpp, int32_t tile_size,
                               int32_t downsample_factor, pf_slide** out) {
    if (!out || width < 1 || height < 1 || !(base_mpp > 0.0) || tile_size < 16 || tile_size % 16 != 0 ||
        downsample_factor < 2)
        return fail(PF_ERR_INVALID_ARG, "pf_slide_create: bad arguments");
    *out = nullptr;
    pf_slide* s = new (std::nothrow) pf_slide();
    if (!s) return fail(PF_ERR_INTERNAL, "pf_slide_create: out of host memory");
    std::memset(&s->desc, 0, sizeof(s->desc));
    s->factor = downsample_factor;
    // ingest_image's pyramid (pkg/store.py:496-498): ceil-divide until max(dim) <= tile
    int64_t w = width, h = height, ds = 1;
    int n = 0;
    while (true) {
        if (n == PF_MAX_LEVELS) {
            delete s;
            return fail(PF_ERR_INVALID_ARG, "pf_slide_create: more than PF_MAX_LEVELS levels");
        }
        s->desc.width[n] = (int32_t)w;
        s->desc.height[n] = (int32_t)h;
        s->desc.downsample[n] = (int32_t)ds;
        s->desc.mpp[n] = base_mpp * (double)ds;
        s->desc.tiles_x[n] = (int32_t)((w + tile_size - 1) / tile_size);
        s->desc.tiles_y[n] = (int32_t)((h + tile_size - 1) / tile_size);
        ++n;
        if (std::max(w, h) <= tile_size) break;
        w = (w + downsample_factor - 1) / downsample_factor;
        h = (h + downsample_factor - 1) / downsample_factor;
        ds *= downsample_factor;
    }
    s->desc.n_levels = n;
    s->desc.tile_size = tile_size;
    s->desc.base_mpp = base_mpp;
    for (int l = 0; l < n; ++l) {
        const size_t bytes = (size_t)s->desc.tiles_x[l] * s->desc.tiles_y[l] * tile_size * tile_size * 3;
        void* p = nullptr;
        int rc = check_cuda(cudaMalloc(&p, bytes), "pf_slide_create: cudaMalloc");
        if (!rc) rc = check_cuda(cudaMemset(p, 0, bytes), "pf_slide_create: cudaMemset");
        if (rc) {
            if (p) cudaFree(p);
            for (void* q : s->allocs) cudaFree(q);
            delete s;
            return rc;
        }
        s->allocs.push_back(p);
        s->desc.level_ptr[l] = reinterpret_cast<uint64_t>(p);
    }
    void* st = nullptr;
    int rc = check_cuda(cudaMalloc(&st, 4), "pf_slide_create: cudaMalloc");
    if (!rc) rc = check_cuda(cudaMemset(st, 0, 4), "pf_slide_create: cudaMemset");
    if (rc) {
        if (st) cudaFree(st);
        for (void* q : s->allocs) cudaFree(q);
        delete s;
        return rc;
    }
    s->allocs.push_back(st);
    s->status_dev = static_cast<int32_t*>(st);
    s->desc.status_word = reinterpret_cast<uint64_t>(st);
    *out = s;
    return PF_OK;
}

extern "C" int pf_slide_destroy(pf_slide* s) {
    if (!s) return PF_OK;
    int rc = check_cuda(cudaDeviceSynchronize(), "pf_slide_destroy: cudaDeviceSynchronize");
    for (void* p : s->allocs) {
        const int r = check_cuda(cudaFree(p), "pf_slide_destroy: cudaFree");
        if (!rc) rc = r;
    }
    delete s;
    return rc;
}

extern "C" int pf_slide_get_desc(const pf_slide* s, pf_slide_desc* out) {
    if (!s || !out) return fail(PF_ERR_INVALID_ARG, "pf_slide_get_desc: bad arguments");
    *out = s->desc;
    return PF_OK;
}

extern "C" int pf_slide_upload_level0(pf_slide* s, const uint8_t* hwc, int64_t row_stride, int32_t on_host,
                                      void* stream) {
    if (!s || !hwc) return fail(PF_ERR_INVALID_ARG, "pf_slide_upload_level0: bad arguments");
    const int W = s->desc.width[0], H = s->desc.height[0];
    if (row_stride == 0) row_stride = (int64_t)W * 3;
    if (row_stride < (int64_t)W * 3) return fail(PF_ERR_INVALID_ARG, "pf_slide_upload_level0: row stride < 3 * width");
    cudaStream_t st = as_stream(stream);
    const int chunk = on_host ? 256 : H;  // host rows are staged through a bounded device buffer
    uint8_t* stage = nullptr;
    int rc = PF_OK;
    if (on_host) {
        if ((rc = check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&stage), (size_t)chunk * W * 3, st),
                             "pf_slide_upload_level0: cudaMallocAsync")))
            return rc;
    }
    for (int y0 = 0; y0 < H; y0 += chunk) {
        const int rows = std::min(chunk, H - y0);
        const uint8_t* src;
        int64_t stride;
        if (on_host) {
            if ((rc = check_cuda(cudaMemcpy2DAsync(stage, (size_t)W * 3, hwc + (size_t)y0 * row_stride, (size_t)row_stride,
                                                   (size_t)W * 3, rows, cudaMemcpyHostToDevice, st),
                                 "pf_slide_upload_level0: cudaMemcpy2DAsync")))
                break;
            src = stage;
            stride = (int64_t)W * 3;
        } else {
            src = hwc + (size_t)y0 * row_stride;
            stride = row_stride;
        }
        const dim3 grid((unsigned)std::min<int64_t>(((int64_t)W * 3 + 255) / 256, 64), rows);
        tile_rows_kernel<<<grid, 256, 0, st>>>(s->desc, src, stride, y0, rows);
        if ((rc = after_launch("tile_rows_kernel"))) break;
        if (on_host && (rc = check_cuda(cudaStreamSynchronize(st), "pf_slide_upload_level0: sync"))) break;
    }
    if (on_host) cudaFreeAsync(stage, st);
    if (rc) return rc;
    for (int l = 1; l < s->desc.n_levels; ++l)
        if ((rc = pf_build_level(&s->desc, l, s->factor, stream))) return rc;
    return PF_OK;
}

extern "C" int pf_slide_upload_tile(pf_slide* s, int32_t level, int32_t tx, int32_t ty, const uint8_t* tile_hwc_host,
                                    int32_t tw, int32_t th, void* stream) {
    if (!s || !tile_hwc_host || level < 0 || level >= s->desc.n_levels)
        return fail(PF_ERR_INVALID_ARG, "pf_slide_upload_tile: bad arguments");
    if (tx < 0 || ty < 0 || tx >= s->desc.tiles_x[level] || ty >= s->desc.tiles_y[level])
        return fail(PF_ERR_OUT_OF_BOUNDS, "pf_slide_upload_tile: tile index outside the level grid");
    const int T = s->desc.tile_size;
    // tile_dims (pkg/store.py:140-149): edge tiles are cropped
    const int ew = std::min(T, s->desc.width[level] - tx * T), eh = std::min(T, s->desc.height[level] - ty * T);
    if (tw != ew || th != eh) return fail(PF_ERR_INTEGRITY, "pf_slide_upload_tile: tile dims != tile_dims");
    uint8_t* dst = reinterpret_cast<uint8_t*>(s->desc.level_ptr[level]) +
                   ((size_t)ty * s->desc.tiles_x[level] + tx) * T * T * 3;
    return check_cuda(cudaMemcpy2DAsync(dst, (size_t)T * 3, tile_hwc_host, (size_t)tw * 3, (size_t)tw * 3, th,
                                        cudaMemcpyHostToDevice, as_stream(stream)),
                      "pf_slide_upload_tile: cudaMemcpy2DAsync");
}

extern "C" int pf_slide_build_pyramid(pf_slide* s, void* stream) {
    if (!s) return fail(PF_ERR_INVALID_ARG, "pf_slide_build_pyramid: bad arguments");
    for (int l = 1; l < s->desc.n_levels; ++l) {
        const int rc = pf_build_level(&s->desc, l, s->factor, stream);
        if (rc) return rc;
    }
    return PF_OK;
}

extern "C" int pf_slide_status(const pf_slide_desc* desc, int32_t clear, void* stream) {
    if (!desc) return fail(PF_ERR_INVALID_ARG, "pf_slide_status: bad arguments");
    if (!desc->status_word) return PF_OK;
    cudaStream_t st = as_stream(stream);
    int32_t v = 0;
    int rc = check_cuda(cudaMemcpyAsync(&v, reinterpret_cast<const void*>(desc->status_word), 4,
                                        cudaMemcpyDeviceToHost, st),
                        "pf_slide_status: cudaMemcpyAsync");
    if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "pf_slide_status: cudaStreamSynchronize");
    if (rc) return rc;
    if (v != PF_OK && clear) {
        rc = check_cuda(cudaMemsetAsync(reinterpret_cast<void*>(desc->status_word), 0, 4, st), "pf_slide_status: clear");
        if (rc) return rc;
    }
    if (v == PF_ERR_OUT_OF_BOUNDS)
        return fail(PF_ERR_OUT_OF_BOUNDS, "a read reached a tile that is not HBM-resident (zero hole of a compacted level)");
    return v == PF_OK ? PF_OK : fail(v, "slide status word set");
}
