// Store read path on the HBM pyramid: pyramid build / thumbnail box filter,
// region planning and batched read_region (gather + PIL resample + normalise).
//
// Reference: pkg/store.py — _box_downsample 429-441, ingest_image pyramid loop
// 496-498, Slide.thumbnail 604-609, read_region 651-688, _read_window 690-724.
#include <cuda_bf16.h>

#include "pf_common.cuh"
#include "pf_resample.cuh"

namespace pf {

// ---------------------------------------------------------------------------
// _box_downsample: out = floor(sum / count + 0.5) over factor x factor blocks,
// edge blocks averaging only the pixels they contain.  The FP64 expression is
// exactly floor((2*sum + count) / (2*count)) in integers (sum/count is never
// within one ulp of a half-integer it does not equal), so integers are used.
// One thread per output pixel; dst is either a tiled level or a dense HWC image.
// ---------------------------------------------------------------------------
template <bool kDstTiled>
__global__ void box_downsample_kernel(pf_slide_desc s, int src_level, int dst_level, int factor,
                                      int out_w, int out_h, uint8_t* dst_hwc) {
    const int ox = blockIdx.x * blockDim.x + threadIdx.x;
    const int oy = blockIdx.y;
    if (ox >= out_w || oy >= out_h) return;
    const int W = s.width[src_level], H = s.height[src_level];
    const int x0 = ox * factor, y0 = oy * factor;
    const int x1 = min(x0 + factor, W), y1 = min(y0 + factor, H);
    uint32_t acc0 = 0, acc1 = 0, acc2 = 0;
    for (int y = y0; y < y1; ++y) {
        for (int x = x0; x < x1; ++x) {
            const uint8_t* p = level_pixel(s, src_level, x, y);
            acc0 += p[0];
            acc1 += p[1];
            acc2 += p[2];
        }
    }
    const uint32_t cnt = (uint32_t)(x1 - x0) * (uint32_t)(y1 - y0);
    uint8_t* out = kDstTiled ? level_pixel_mut(s, dst_level, ox, oy)
                             : dst_hwc + ((size_t)oy * out_w + ox) * 3;
    out[0] = (uint8_t)((2 * acc0 + cnt) / (2 * cnt));
    out[1] = (uint8_t)((2 * acc1 + cnt) / (2 * cnt));
    out[2] = (uint8_t)((2 * acc2 + cnt) / (2 * cnt));
}

// Thumbnail with factor 32 over a 256-tile level: one warp per output pixel,
// lane = source row, 6 x 16-byte loads per lane (96 contiguous bytes).
__global__ void box32_warp_kernel(pf_slide_desc s, int src_level, int out_w, int out_h,
                                  uint8_t* dst_hwc) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= out_w * out_h) return;
    const int ox = warp % out_w, oy = warp / out_w;
    const int W = s.width[src_level], H = s.height[src_level];
    const int x0 = ox * 32, y0 = oy * 32;
    const int x1 = min(x0 + 32, W), y1 = min(y0 + 32, H);
    uint32_t a0 = 0, a1 = 0, a2 = 0;
    const int y = y0 + lane;
    if (y < y1) {
        if (x1 - x0 == 32) {
            const uint4* p = reinterpret_cast<const uint4*>(level_pixel(s, src_level, x0, y));
#pragma unroll
            for (int k = 0; k < 6; ++k) {
                const uint4 q = __ldg(p + k);
                const uint32_t words[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const uint32_t byte = (words[j] >> (8 * b)) & 0xffu;
                        const int c = (k * 16 + j * 4 + b) % 3;
                        if (c == 0) a0 += byte;
                        else if (c == 1) a1 += byte;
                        else a2 += byte;
                    }
                }
            }
        } else {
            for (int x = x0; x < x1; ++x) {
                const uint8_t* p = level_pixel(s, src_level, x, y);
                a0 += p[0];
                a1 += p[1];
                a2 += p[2];
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        a1 += __shfl_xor_sync(0xffffffffu, a1, o);
        a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (lane == 0) {
        const uint32_t cnt = (uint32_t)(x1 - x0) * (uint32_t)(y1 - y0);
        uint8_t* out = dst_hwc + ((size_t)oy * out_w + ox) * 3;
        out[0] = (uint8_t)((2 * a0 + cnt) / (2 * cnt));
        out[1] = (uint8_t)((2 * a1 + cnt) / (2 * cnt));
        out[2] = (uint8_t)((2 * a2 + cnt) / (2 * cnt));
    }
}

// sx, sy = round_half_away(x / ds), store.py:680-681 (x >= 0).
__global__ void plan_regions_kernel(const pf_slide_desc* slides, pf_patch_spec* specs, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    pf_patch_spec& sp = specs[i];
    const double ds = (double)slides[sp.slide].downsample[sp.level];
    sp.sx = (int32_t)floor((double)sp.x / ds + 0.5);
    sp.sy = (int32_t)floor((double)sp.y / ds + 0.5);
}

// ---------------------------------------------------------------------------
// read_region epilogue: (v/255 - mean)/std in FP32, the op order of
// normalize_patch (pkg/pipeline.py:152-155) and torchvision Normalize.
// ---------------------------------------------------------------------------
struct NormParams {
    float mean[3], stdv[3];
};

template <int kDtype>
__device__ __forceinline__ void store_px(void* out, size_t idx, uint8_t v, int c,
                                         const NormParams& np) {
    if (kDtype == PF_U8) {
        reinterpret_cast<uint8_t*>(out)[idx] = v;
    } else {
        const float f = __fdiv_rn(__fdiv_rn((float)v, 255.0f) - np.mean[c], np.stdv[c]);
        if (kDtype == PF_F32) reinterpret_cast<float*>(out)[idx] = f;
        else reinterpret_cast<__nv_bfloat16*>(out)[idx] = __float2bfloat16_rn(f);
    }
}

template <int kDtype>
__device__ __forceinline__ void write_out(void* out, int layout, int n_idx, int S, int y, int x,
                                          const uint8_t* rgb, const NormParams& np) {
    for (int c = 0; c < 3; ++c) {
        size_t idx;
        if (layout == PF_HWC) idx = (((size_t)n_idx * S + y) * S + x) * 3 + c;
        else idx = (((size_t)n_idx * 3 + c) * S + y) * S + x;
        store_px<kDtype>(out, idx, rgb[c], c, np);
    }
}

// One CTA per spec.  Passthrough copies the clamped window; otherwise the
// PIL two-pass resample runs in bands of output rows with a uint8
// intermediate in shared memory.
constexpr int kRRThreads = 256;
constexpr int kRRInterBytes = 48 * 1024;

template <int kDtype>
__global__ void __launch_bounds__(kRRThreads) read_regions_kernel(const pf_slide_desc* slides,
                                                                  const pf_patch_spec* specs,
                                                                  int out_size, int layout,
                                                                  NormParams np, void* out) {
    extern __shared__ __align__(16) uint8_t smem[];
    const pf_patch_spec sp = specs[blockIdx.x];
    const pf_slide_desc& s = slides[sp.slide];
    const int L = sp.level;
    const int W = s.width[L], H = s.height[L];
    const int side = sp.side, S = out_size;
    const bool skip_pass = layout & PF_SKIP_PASSTHROUGH;
    layout &= 0xff;

    if (side == S) {
        if (skip_pass) return;
        for (int p = threadIdx.x; p < S * S; p += blockDim.x) {
            const int y = p / S, x = p - y * S;
            const int X = clampi(sp.sx + x, 0, W - 1), Y = clampi(sp.sy + y, 0, H - 1);
            const uint8_t* src = level_pixel(s, L, X, Y);
            const uint8_t rgb[3] = {src[0], src[1], src[2]};
            write_out<kDtype>(out, layout, blockIdx.x, S, y, x, rgb, np);
        }
        return;
    }

    // coefficient table (square window: one table serves both axes)
    const AxisPlan ap = axis_plan(side, S);
    int* s_xmin = reinterpret_cast<int*>(smem);
    int* s_xsize = s_xmin + S;
    int32_t* s_w = s_xsize + S;
    double* s_red = reinterpret_cast<double*>(smem + (((size_t)(2 * S + S * ap.ksize) * 4 + 15) & ~size_t(15)));
    uint8_t* s_inter = reinterpret_cast<uint8_t*>(s_red + 2);
    build_axis_table(side, S, RS_PIL, s_xmin, s_xsize, s_w, s_red);
    const int K = ap.ksize;
    const int row_bytes = S * 3;
    const int max_rows = kRRInterBytes / row_bytes;

    int y0 = 0;
    while (y0 < S) {
        // grow the band while its source rows fit the intermediate buffer
        const int r0 = s_xmin[y0];
        int y1 = y0 + 1;
        while (y1 < S && s_xmin[y1] + s_xsize[y1] - r0 <= max_rows) ++y1;
        const int r1 = s_xmin[y1 - 1] + s_xsize[y1 - 1];
        // horizontal pass: source rows [r0, r1) -> s_inter
        for (int p = threadIdx.x; p < (r1 - r0) * S; p += blockDim.x) {
            const int rr = p / S, x = p - rr * S;
            const int Y = clampi(sp.sy + r0 + rr, 0, H - 1);
            const int xmin = s_xmin[x], xs = s_xsize[x];
            int32_t a0 = 1 << 21, a1 = 1 << 21, a2 = 1 << 21;
            for (int k = 0; k < xs; ++k) {
                const int X = clampi(sp.sx + xmin + k, 0, W - 1);
                const uint8_t* src = level_pixel(s, L, X, Y);
                const int32_t wk = s_w[x * K + k];
                a0 += (int32_t)src[0] * wk;
                a1 += (int32_t)src[1] * wk;
                a2 += (int32_t)src[2] * wk;
            }
            uint8_t* d = s_inter + (size_t)rr * row_bytes + x * 3;
            d[0] = clip_shift(a0, 22);
            d[1] = clip_shift(a1, 22);
            d[2] = clip_shift(a2, 22);
        }
        __syncthreads();
        // vertical pass: output rows [y0, y1)
        for (int p = threadIdx.x; p < (y1 - y0) * S; p += blockDim.x) {
            const int yy = p / S, x = p - yy * S;
            const int y = y0 + yy;
            const int ymin = s_xmin[y] - r0, ys = s_xsize[y];
            int32_t a0 = 1 << 21, a1 = 1 << 21, a2 = 1 << 21;
            for (int k = 0; k < ys; ++k) {
                const uint8_t* src = s_inter + (size_t)(ymin + k) * row_bytes + x * 3;
                const int32_t wk = s_w[y * K + k];
                a0 += (int32_t)src[0] * wk;
                a1 += (int32_t)src[1] * wk;
                a2 += (int32_t)src[2] * wk;
            }
            const uint8_t rgb[3] = {clip_shift(a0, 22), clip_shift(a1, 22), clip_shift(a2, 22)};
            write_out<kDtype>(out, layout, blockIdx.x, S, y, x, rgb, np);
        }
        __syncthreads();
        y0 = y1;
    }
}

template <int kDtype>
__global__ void normalize_kernel(const uint8_t* in, int64_t n, NormParams np, void* out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int c = (int)(i % 3);
    store_px<kDtype>(out, (size_t)i, in[i], c, np);
}

}  // namespace pf

using namespace pf;

extern "C" int pf_normalize(const uint8_t* in_hwc, int64_t n_pixels, int32_t dtype, const float* mean3,
                            const float* std3, void* out, void* stream) {
    if (n_pixels < 0 || (n_pixels > 0 && (!in_hwc || !out)))
        return fail(PF_ERR_INVALID_ARG, "pf_normalize: bad arguments");
    if (n_pixels == 0) return PF_OK;
    NormParams np;
    for (int c = 0; c < 3; ++c) {
        np.mean[c] = mean3 ? mean3[c] : 0.5f;
        np.stdv[c] = std3 ? std3[c] : 0.5f;
    }
    const int64_t n = n_pixels * 3;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (dtype == PF_F32) normalize_kernel<PF_F32><<<blocks, 256, 0, as_stream(stream)>>>(in_hwc, n, np, out);
    else if (dtype == PF_BF16) normalize_kernel<PF_BF16><<<blocks, 256, 0, as_stream(stream)>>>(in_hwc, n, np, out);
    else return fail(PF_ERR_INVALID_ARG, "pf_normalize: dtype must be f32 or bf16");
    return after_launch("normalize_kernel");
}

extern "C" int pf_build_level(const pf_slide_desc* slide, int32_t level, int32_t factor,
                              void* stream) {
    if (!slide || level < 1 || level >= slide->n_levels || factor < 2)
        return fail(PF_ERR_INVALID_ARG, "pf_build_level: bad level/factor");
    const int ow = slide->width[level], oh = slide->height[level];
    if (ow != (slide->width[level - 1] + factor - 1) / factor ||
        oh != (slide->height[level - 1] + factor - 1) / factor)
        return fail(PF_ERR_INTEGRITY, "pf_build_level: level dims != ceil(prev / factor)");
    dim3 grid((ow + 127) / 128, oh);
    box_downsample_kernel<true><<<grid, 128, 0, as_stream(stream)>>>(*slide, level - 1, level, factor,
                                                                      ow, oh, nullptr);
    return after_launch("box_downsample_kernel");
}

extern "C" int pf_thumbnail(const pf_slide_desc* slide, int32_t src_level, int32_t factor,
                            uint8_t* out_hwc, void* stream) {
    if (!slide || src_level < 0 || src_level >= slide->n_levels || factor < 1 || !out_hwc)
        return fail(PF_ERR_INVALID_ARG, "pf_thumbnail: bad arguments");
    const int W = slide->width[src_level], H = slide->height[src_level];
    const int ow = (W + factor - 1) / factor, oh = (H + factor - 1) / factor;
    if (factor == 32 && slide->tile_size % 32 == 0) {
        const long long warps = (long long)ow * oh;
        const int threads = 256;
        const long long blocks = (warps * 32 + threads - 1) / threads;
        box32_warp_kernel<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(*slide, src_level, ow, oh,
                                                                                out_hwc);
        return after_launch("box32_warp_kernel");
    }
    dim3 grid((ow + 127) / 128, oh);
    box_downsample_kernel<false><<<grid, 128, 0, as_stream(stream)>>>(*slide, src_level, 0, factor, ow,
                                                                       oh, out_hwc);
    return after_launch("box_downsample_kernel");
}

extern "C" int pf_plan_regions(const pf_slide_desc* slides_dev, pf_patch_spec* specs_dev, int32_t n,
                               void* stream) {
    if (n < 0 || (n > 0 && (!slides_dev || !specs_dev)))
        return fail(PF_ERR_INVALID_ARG, "pf_plan_regions: bad arguments");
    if (n == 0) return PF_OK;
    plan_regions_kernel<<<(n + 255) / 256, 256, 0, as_stream(stream)>>>(slides_dev, specs_dev, n);
    return after_launch("plan_regions_kernel");
}

extern "C" int pf_read_regions(const pf_slide_desc* slides_dev, const pf_patch_spec* specs_dev,
                               int32_t n, int32_t out_size, int32_t dtype, int32_t layout,
                               const float* mean3, const float* std3, void* out, void* stream) {
    if (n < 0 || out_size < 1 || out_size > 4096 || (n > 0 && (!slides_dev || !specs_dev || !out)))
        return fail(PF_ERR_INVALID_ARG, "pf_read_regions: bad arguments");
    if ((layout & 0xff) != PF_HWC && (layout & 0xff) != PF_NCHW)
        return fail(PF_ERR_INVALID_ARG, "pf_read_regions: bad layout");
    if (out_size > 512)
        return fail(PF_ERR_INVALID_ARG, "pf_read_regions: out_size > 512 unsupported");
    if (n == 0) return PF_OK;
    NormParams np;
    for (int c = 0; c < 3; ++c) {
        np.mean[c] = mean3 ? mean3[c] : 0.5f;
        np.stdv[c] = std3 ? std3[c] : 0.5f;
    }
    // worst-case ksize for down-ratios up to 15x
    const int ksize_max = 32;
    const size_t smem = ((size_t)(2 * out_size + out_size * ksize_max) * 4 + 15) / 16 * 16 + 16 + kRRInterBytes;
    cudaStream_t st = as_stream(stream);
    int rc;
    switch (dtype) {
        case PF_U8:
            rc = check_cuda(cudaFuncSetAttribute(read_regions_kernel<PF_U8>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                            "cudaFuncSetAttribute");
            if (rc) return rc;
            read_regions_kernel<PF_U8><<<n, kRRThreads, smem, st>>>(slides_dev, specs_dev, out_size, layout, np, out);
            break;
        case PF_F32:
            rc = check_cuda(cudaFuncSetAttribute(read_regions_kernel<PF_F32>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                            "cudaFuncSetAttribute");
            if (rc) return rc;
            read_regions_kernel<PF_F32><<<n, kRRThreads, smem, st>>>(slides_dev, specs_dev, out_size, layout, np, out);
            break;
        case PF_BF16:
            rc = check_cuda(cudaFuncSetAttribute(read_regions_kernel<PF_BF16>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                            "cudaFuncSetAttribute");
            if (rc) return rc;
            read_regions_kernel<PF_BF16><<<n, kRRThreads, smem, st>>>(slides_dev, specs_dev, out_size, layout, np, out);
            break;
        default:
            return fail(PF_ERR_INVALID_ARG, "pf_read_regions: bad dtype");
    }
    return after_launch("read_regions_kernel");
}
