// Store read path on the HBM pyramid: pyramid build / thumbnail box filter,
// region planning and batched read_region (gather + PIL resample + normalise).
//
// Reference: pkg/store.py — _box_downsample 429-441, ingest_image pyramid loop
// 496-498, Slide.thumbnail 604-609, read_region 651-688, _read_window 690-724.
#include <cuda_bf16.h>

#include <array>
#include <cstring>
#include <map>
#include <mutex>

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

// read_region on device.  Grid: (spec, band of kRRBand output rows).
//  * passthrough (side == out): the band's source rows are staged from the
//    tile pyramid with 16-byte cp.async (whole tile rows; clamped per-pixel
//    gather only when the window touches the level edge), then written with
//    the normalising epilogue (3x256 LUT) as 16-byte NCHW rows or HWC words;
//  * resample (side != out): each band CTA runs the PIL two-pass fixed-point
//    resample for its output rows (coefficients built in shared memory, the
//    band's source rows staged in sub-bands, horizontal pass into planar uint8,
//    vertical pass straight into the epilogue).
constexpr int kRRThreads = 256;
constexpr int kRRBand = 32;
constexpr int kRRSmem = 96 * 1024;

__device__ __forceinline__ void rr_cp_async16(void* smem_dst, const void* gmem_src) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src));
}
__device__ __forceinline__ void rr_cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Stage level rows Y0+r, r in [0, nr), columns [X0, X0+w) into stg (row stride row_bytes);
// returns the byte offset of column X0 inside a staged row.
__device__ int stage_level_rows(const pf_slide_desc& sd, int L, int X0, int Y0, int w, int nr, uint8_t* stg,
                                int row_bytes, bool fast) {
    const int T = sd.tile_size;
    const int LW = sd.width[L], LH = sd.height[L];
    if (fast) {
        // only the 16-byte aligned span of each window row: [a0, a0 + 16 * nch) of the level row,
        // chunk by chunk from whichever tile holds it (a tile row is 3T bytes, a multiple of 16)
        const int a0 = (X0 * 3) & ~15;
        const int nch = (X0 * 3 + w * 3 - a0 + 15) / 16;
        const int cpr = T * 3 / 16;
        const int c0 = a0 / 16;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int rr = warp; rr < nr; rr += blockDim.x / 32) {
            const int Y = Y0 + rr;
            const int ty = Y / T, v = Y - ty * T;
            uint8_t* srow = stg + rr * row_bytes;
            for (int ch = lane; ch < nch; ch += 32) {
                const int c = c0 + ch, tx = c / cpr, e = c - tx * cpr;
                rr_cp_async16(srow + ch * 16, tile_ptr(sd, L, tx, ty) + (size_t)v * T * 3 + e * 16);
            }
        }
        rr_cp_async_wait_all();
        return X0 * 3 - a0;
    }
    for (int q = threadIdx.x; q < nr * w; q += blockDim.x) {
        const int rr = q / w, xx = q - rr * w;
        const uint8_t* s = level_pixel(sd, L, clampi(X0 + xx, 0, LW - 1), clampi(Y0 + rr, 0, LH - 1));
        uint8_t* d = stg + rr * row_bytes + xx * 3;
        d[0] = s[0];
        d[1] = s[1];
        d[2] = s[2];
    }
    return 0;
}

// PIL horizontal pass of one output column over staged rows [rr0, rr1) (22-bit int taps,
// planar uint8 out).  K > 0: taps unrolled and kept in registers (zero beyond xsize).
template <int K>
__device__ __forceinline__ void pil_h_rows(const uint8_t* stg, int pitch, int off, int xmin, int xs, const int32_t* w,
                                           int rr0, int rr1, uint8_t* hb_col, int S, int hplane) {
    const uint8_t* s0 = stg + off + xmin * 3;
    if constexpr (K > 0) {
        int32_t wk[K];
#pragma unroll
        for (int k = 0; k < K; ++k) wk[k] = k < xs ? w[k] : 0;
        for (int rr = rr0; rr < rr1; ++rr) {
            const uint8_t* p = s0 + rr * pitch;
            int32_t a0 = 1 << 21, a1 = 1 << 21, a2 = 1 << 21;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (k < xs) {  // taps past xsize may lie beyond the staged span
                    a0 += (int32_t)p[3 * k] * wk[k];
                    a1 += (int32_t)p[3 * k + 1] * wk[k];
                    a2 += (int32_t)p[3 * k + 2] * wk[k];
                }
            }
            uint8_t* d = hb_col + rr * S;
            d[0] = clip_shift(a0, 22);
            d[hplane] = clip_shift(a1, 22);
            d[2 * hplane] = clip_shift(a2, 22);
        }
    } else {
        for (int rr = rr0; rr < rr1; ++rr) {
            const uint8_t* p = s0 + rr * pitch;
            int32_t a0 = 1 << 21, a1 = 1 << 21, a2 = 1 << 21;
            for (int k = 0; k < xs; ++k) {
                a0 += (int32_t)p[3 * k] * w[k];
                a1 += (int32_t)p[3 * k + 1] * w[k];
                a2 += (int32_t)p[3 * k + 2] * w[k];
            }
            uint8_t* d = hb_col + rr * S;
            d[0] = clip_shift(a0, 22);
            d[hplane] = clip_shift(a1, 22);
            d[2 * hplane] = clip_shift(a2, 22);
        }
    }
}

template <int kDtype>
struct RROut;
template <>
struct RROut<PF_U8> {
    using T = uint8_t;
};
template <>
struct RROut<PF_F32> {
    using T = float;
};
template <>
struct RROut<PF_BF16> {
    using T = __nv_bfloat16;
};

// ---------------------------------------------------------------------------
// Exact 2:1 PIL BILINEAR (side == 2 * out, window inside the level): BASELINE config 3's
// 448 -> 224 reads.  Every interior output's taps are PIL's own 22-bit weights
// (0.125, 0.375, 0.375, 0.125) * 2^22 = 2^19 * (1, 3, 3, 1), so
//   (2^21 + sum w_k p_k) >> 22 == (p0 + 3 (p1 + p2) + p3 + 4) >> 3      (never clips),
// computed on 16-bit lanes of packed words; the first and last output of each axis (3 clipped
// taps, renormalised) take the table weights.  Bit-exact with the general path / Pillow.
// Grid: (spec, band of kR2Rows output rows); specs it does not take exit at once.
// ---------------------------------------------------------------------------
#ifndef PF_R2_ROWS
#define PF_R2_ROWS 12  // measured: 4 rows 0.66 ms, 8 0.52, 12 0.49, 16 0.50, 24 0.53 per C3 read_regions call
#endif
constexpr int kR2Rows = PF_R2_ROWS;
#ifndef PF_R2_BANDS
#define PF_R2_BANDS 1
#endif
constexpr int kR2Bands = PF_R2_BANDS;  // bands per block
constexpr int kR2Threads = 256;

__device__ __forceinline__ bool is_2x(const pf_patch_spec& sp, const pf_slide_desc& sd, int S) {
    const int L = sp.level;
    return sp.side == 2 * S && S >= 8 && (S % 4) == 0 && sp.sx >= 0 && sp.sy >= 0 && sp.sx + sp.side <= sd.width[L] &&
           sp.sy + sp.side <= sd.height[L] && (sd.tile_size % 16) == 0;
}

// generic 3-tap PIL output of an axis edge: weights w[0..2] (22-bit), bytes p0..p2
__device__ __forceinline__ uint32_t pil3(const int32_t* w, uint32_t p0, uint32_t p1, uint32_t p2) {
    const int32_t a = (1 << 21) + (int32_t)p0 * w[0] + (int32_t)p1 * w[1] + (int32_t)p2 * w[2];
    return clip_shift(a, 22);
}

template <int kDtype, int kS>
__global__ void __launch_bounds__(kR2Threads) resample2x_kernel(const pf_slide_desc* slides, const pf_patch_spec* specs,
                                                                int S_rt, int layout, int n_bands, NormParams np,
                                                                void* out_v) {
    using OT = typename RROut<kDtype>::T;
    const int S = kS ? kS : S_rt;  // compile-time for the BASELINE size: index math without divisions
    extern __shared__ __align__(16) uint8_t smem[];
    // block = (spec, group of kR2Bands bands, taken one after the other)
    const int n_groups = (n_bands + kR2Bands - 1) / kR2Bands;
    const int spec_i = blockIdx.x / n_groups, group = blockIdx.x - spec_i * n_groups;
    const pf_patch_spec sp = specs[spec_i];
    const pf_slide_desc& sd = slides[sp.slide];
    if (!is_2x(sp, sd, S)) return;
    const int lay = layout & 0xff;
    const int L = sp.level, T = sd.tile_size;
    const int side = 2 * S;
    // edge weights (first / last output of an axis), PIL's own computation
    __shared__ int32_t s_w0[3], s_wl[3];
    if (threadIdx.x < 2) {
        const AxisPlan ap = axis_plan(side, S);
        double w[8];
        int xmin;
        const int xs = axis_weights(ap, side, threadIdx.x == 0 ? 0 : S - 1, &xmin, w);
        for (int k = 0; k < 3; ++k) (threadIdx.x == 0 ? s_w0 : s_wl)[k] = k < xs ? quantise_weight(w[k], 22) : 0;
    }
    OT* lut = reinterpret_cast<OT*>(smem);
    uint8_t* stg = smem + ((3 * 256 * sizeof(OT) + 15) & ~size_t(15));
    if constexpr (kDtype != PF_U8)
        for (int i = threadIdx.x; i < 3 * 256; i += kR2Threads) {
            const int c = i >> 8;
            const float f = __fdiv_rn(__fdiv_rn((float)(i & 255), 255.0f) - np.mean[c], np.stdv[c]);
            if constexpr (kDtype == PF_F32) lut[i] = f;
            else lut[i] = __float2bfloat16_rn(f);
        }
    // one TMA bulk copy per (staged row, tile the row crosses) on one mbarrier (phase per band):
    // per-16-byte cp.async with its tile address math was ~30 % of this kernel's instructions
    __shared__ __align__(8) uint64_t s_bar;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();  // initialised before any copy completes on it
    for (int it = 0; it < kR2Bands; ++it) {
    const int band = group * kR2Bands + it;
    const int Y0 = band * kR2Rows, Y1 = min(S, Y0 + kR2Rows);
    if (Y0 >= S) break;
    // source rows of the band: output y uses rows 2y - 1 .. 2y + 2 (y = 0: 0..2; y = S-1: 2S-3..2S-1)
    const int R0 = max(0, 2 * Y0 - 1), R1 = min(side, 2 * (Y1 - 1) + 3);
    const int nr = R1 - R0;
    const int a0 = (sp.sx * 3) & ~15, off = sp.sx * 3 - a0;
    const int nch = (off + side * 3 + 15) / 16;
    const int pitch = nch * 16 + 16;  // the last group's 9-word load reads <= 12 bytes past the span
    uint8_t* hb = stg + (size_t)nr * pitch;  // [3][nr][S] horizontal-pass output
    PF_CHECK(nr <= 2 * kR2Rows + 2 && (int)((3 * 256 * sizeof(OT) + 15) & ~size_t(15)) + nr * pitch + 3 * nr * S <=
             (int)(3 * 256 * 4 + (2 * kR2Rows + 2) * ((15 + 6 * S + 15) / 16 * 16 + 16) + 3 * (2 * kR2Rows + 2) * S + 64));
    const int cpr = T * 3 / 16, c0 = a0 / 16;
    const int tx0 = c0 / cpr, e0 = c0 - tx0 * cpr;
    {
        // the arrive (thread 0) keeps the phase open until it has happened, so copies that
        // complete before it only take the transaction count negative
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                         "r"((uint32_t)(nr * nch * 16))
                         : "memory");
        const int n_tiles = (e0 + nch + cpr - 1) / cpr;
        for (int q = threadIdx.x; q < nr * n_tiles; q += kR2Threads) {
            const int rr = q / n_tiles, t = q - rr * n_tiles;
            const int Y = sp.sy + R0 + rr;
            const int ty = Y / T, v = Y - ty * T;
            const int ch0 = max(0, t * cpr - e0), ch1 = min(nch, (t + 1) * cpr - e0);
            if (ch1 <= ch0) continue;
            const uint8_t* src = tile_ptr(sd, L, tx0 + t, ty) + (size_t)v * T * 3 + (size_t)(e0 + ch0 - t * cpr) * 16;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    (uint32_t)__cvta_generic_to_shared(stg + rr * pitch + ch0 * 16)),
                "l"(src), "r"((uint32_t)((ch1 - ch0) * 16)), "r"(bar)
                : "memory");
        }
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                         : "=r"(done)
                         : "r"(bar), "r"((uint32_t)(it & 1))
                         : "memory");
    }
    __syncthreads();
    // horizontal pass: item = (staged row, 4 output columns): source pixels 2x0-1 .. 2x0+8 as
    // 32 bytes from 9 aligned words + funnel shifts, 4 outputs per channel packed into one word;
    // the first and last group (clipped taps at x = 0 and x = S-1) per column
    const int G4h = S / 4;
    auto store3 = [&](int rr, int x0, const uint32_t (&w)[3]) {
#pragma unroll
        for (int c = 0; c < 3; ++c) *reinterpret_cast<uint32_t*>(hb + (size_t)c * nr * S + rr * S + x0) = w[c];
    };
    // interior groups (x0 = 4 .. S-8): no per-column branches inside a warp
    for (int q = threadIdx.x; q < nr * (G4h - 2); q += kR2Threads) {
        const int rr = q / (G4h - 2), x0 = (q - rr * (G4h - 2) + 1) * 4;
        const int b0 = off + (2 * x0 - 1) * 3;  // 30 bytes: pixels 2x0-1 .. 2x0+8
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(stg + rr * pitch + (b0 & ~3));
        const uint32_t sh = (uint32_t)(b0 & 3) * 8;
        uint32_t r[9], A[8], outw[3];
#pragma unroll
        for (int i = 0; i < 9; ++i) r[i] = wp[i];
#pragma unroll
        for (int i = 0; i < 8; ++i) A[i] = __funnelshift_r(r[i], r[i + 1], sh);
        // outputs k and k + 2 of a channel in the two 16-bit lanes of one word: tap t of output k
        // is byte 6k + c + 3t of A, and of output k + 2 the byte 12 further, i.e. the same byte of
        // the word three on -- one byte_perm per tap pair
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            uint32_t pair[2];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                uint32_t tap[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int b = 6 * k + c + 3 * t, i = b >> 2, o = b & 3;
                    tap[t] = __byte_perm(A[i], A[i + 3], (uint32_t)(o | ((o + 4) << 8))) & 0x00ff00ffu;
                }
                pair[k] = ((tap[0] + tap[3] + 3u * (tap[1] + tap[2]) + 0x00040004u) >> 3) & 0x00ff00ffu;
            }
            outw[c] = __byte_perm(pair[0], pair[1], 0x6240u);  // bytes k = 0, 1, 2, 3
        }
        store3(rr, x0, outw);
    }
    // the first and last group of every row: the clipped edge taps at x = 0 and x = S-1
    for (int q = threadIdx.x; q < 2 * nr; q += kR2Threads) {
        const int rr = q >> 1, x0 = (q & 1) ? S - 4 : 0;
        const uint8_t* row = stg + rr * pitch + off;
        uint32_t o[3] = {0u, 0u, 0u};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int x = x0 + k;
            if (x == 0 || x == S - 1) {
                const uint8_t* p = row + (x == 0 ? 0 : (side - 3) * 3);
                const int32_t* w = x == 0 ? s_w0 : s_wl;
#pragma unroll
                for (int c = 0; c < 3; ++c) o[c] |= pil3(w, p[c], p[3 + c], p[6 + c]) << (8 * k);
            } else {
                const uint8_t* p = row + (2 * x - 1) * 3;
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    o[c] |= (((uint32_t)p[c] + p[9 + c] + 3u * ((uint32_t)p[3 + c] + p[6 + c]) + 4u) >> 3) << (8 * k);
            }
        }
        store3(rr, x0, o);
    }
    __syncthreads();
    // vertical pass: item = (output row, 4 columns); 16-bit lanes of packed words
    const size_t plane = (size_t)S * S;
    OT* o = reinterpret_cast<OT*>(out_v) + (size_t)spec_i * 3 * plane;
    const int G = S / 4;
    for (int q = threadIdx.x; q < (Y1 - Y0) * G; q += kR2Threads) {
        const int yy = q / G, x0 = (q - yy * G) * 4;
        const int y = Y0 + yy;
        uint32_t px[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const uint8_t* col = hb + (size_t)c * nr * S + x0;
            if (y == 0 || y == S - 1) {
                const int rb = (y == 0 ? 0 : side - 3) - R0;
                const int32_t* w = y == 0 ? s_w0 : s_wl;
                uint32_t v = 0;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    v |= pil3(w, col[(rb) * S + k], col[(rb + 1) * S + k], col[(rb + 2) * S + k]) << (8 * k);
                px[c] = v;
            } else {
                const int rb = 2 * y - 1 - R0;
                const uint32_t w0 = *reinterpret_cast<const uint32_t*>(col + rb * S);
                const uint32_t w1 = *reinterpret_cast<const uint32_t*>(col + (rb + 1) * S);
                const uint32_t w2 = *reinterpret_cast<const uint32_t*>(col + (rb + 2) * S);
                const uint32_t w3 = *reinterpret_cast<const uint32_t*>(col + (rb + 3) * S);
                const uint32_t m = 0x00ff00ffu;
                const uint32_t lo = ((w0 & m) + (w3 & m) + 3u * ((w1 & m) + (w2 & m)) + 0x00040004u) >> 3;
                const uint32_t hi = (((w0 >> 8) & m) + ((w3 >> 8) & m) + 3u * (((w1 >> 8) & m) + ((w2 >> 8) & m)) +
                                     0x00040004u) >> 3;
                px[c] = (lo & m) | ((hi & m) << 8);
            }
        }
        if (kDtype == PF_U8 && lay == PF_HWC) {  // 4 pixels x RGB = 12 bytes = 3 words (offset a multiple of 12)
            const uint32_t R = px[0], Gc = px[1], B = px[2];
            uint32_t* dst = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(o) + ((size_t)y * S + x0) * 3);
            // r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3
            dst[0] = __byte_perm(__byte_perm(R, Gc, 0x1040u), B, 0x3410u);
            dst[1] = __byte_perm(__byte_perm(Gc, B, 0x2051u), R, 0x3610u);
            dst[2] = __byte_perm(__byte_perm(B, R, 0x3072u), Gc, 0x3710u);
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const uint8_t v = (uint8_t)(px[c] >> (8 * k));
                    const size_t idx = lay == PF_HWC ? ((size_t)y * S + x0 + k) * 3 + c : c * plane + (size_t)y * S + x0 + k;
                    if constexpr (kDtype == PF_U8) reinterpret_cast<uint8_t*>(o)[idx] = v;
                    else o[idx] = lut[c * 256 + v];
                }
        }
    }
    __syncthreads();  // the next band restages the buffers
    }
}

// Passthrough epilogue of one staged band: nr rows of S px (RGB, byte offset `base` in rows of
// `row_bytes`) -> output rows [y0, y0 + nr) of `o`, through the normalising LUT (smem, or the
// global table read with __ldg when kLdg).
template <int kDtype, bool kLdg>
__device__ __forceinline__ void passthrough_out(const uint8_t* work, int row_bytes, int base, int nr, int y0, int S,
                                                int lay, const typename RROut<kDtype>::T* lut,
                                                typename RROut<kDtype>::T* o) {
    using OT = typename RROut<kDtype>::T;
    const size_t plane = (size_t)S * S;
    auto L = [&](int i) -> OT {
        if constexpr (kLdg) return __ldg(lut + i);
        else return lut[i];
    };
#ifndef PF_PT_ITEM_CH
    if constexpr (kLdg) {
        // lean kernel: one item = 4 pixels x 3 channels; its 12 staged bytes are read as 4
        // aligned words and funnel-shifted (4 LDS instead of 12 byte loads), then one 4-wide
        // store per channel plane.  The staged band has >= 16 B of slack after its last row
        // (host smem size), so the 4th word is always inside the allocation.
        if (lay == PF_NCHW && (S % 4) == 0) {
            const int G = S / 4;
            for (int q = threadIdx.x; q < nr * G; q += blockDim.x) {
                const int rr = q / G, x0 = (q - rr * G) * 4;
                const int off = rr * row_bytes + base + x0 * 3;
                const uint32_t* w = reinterpret_cast<const uint32_t*>(work + (off & ~3));
                const uint32_t a0 = w[0], a1 = w[1], a2 = w[2], a3 = w[3];
                const uint32_t sh = (uint32_t)(off & 3) * 8;
                const uint32_t b[3] = {__funnelshift_r(a0, a1, sh), __funnelshift_r(a1, a2, sh),
                                       __funnelshift_r(a2, a3, sh)};
                OT* dst = o + (size_t)(y0 + rr) * S + x0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    OT v[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int j = 3 * k + c;  // byte j of the 12: pixel k, channel c
                        v[k] = L(c * 256 + (int)((b[j >> 2] >> ((j & 3) * 8)) & 0xffu));
                    }
                    OT* d = dst + c * plane;
                    if constexpr (sizeof(OT) == 4) *reinterpret_cast<uint4*>(d) = *reinterpret_cast<const uint4*>(v);
                    else if constexpr (sizeof(OT) == 2) *reinterpret_cast<uint2*>(d) = *reinterpret_cast<const uint2*>(v);
                    else *reinterpret_cast<uint32_t*>(d) = *reinterpret_cast<const uint32_t*>(v);
                }
            }
            return;
        }
    }
#endif
    if (lay == PF_NCHW && (S % 4) == 0) {
        const int G = S / 4;
        for (int q = threadIdx.x; q < 3 * nr * G; q += blockDim.x) {
            const int c = q / (nr * G);
            const int rem = q - c * nr * G;
            const int rr = rem / G, x0 = (rem - rr * G) * 4;
            const uint8_t* s = work + rr * row_bytes + base + x0 * 3 + c;
            OT v[4] = {L(c * 256 + s[0]), L(c * 256 + s[3]), L(c * 256 + s[6]), L(c * 256 + s[9])};
            OT* dst = o + c * plane + (size_t)(y0 + rr) * S + x0;
            if constexpr (sizeof(OT) == 4) *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(v);
            else if constexpr (sizeof(OT) == 2) *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(v);
            else *reinterpret_cast<uint32_t*>(dst) = *reinterpret_cast<const uint32_t*>(v);
        }
    } else if (lay == PF_HWC && kDtype == PF_U8 && (S * 3) % 4 == 0) {
        const int W4 = S * 3 / 4;
        for (int q = threadIdx.x; q < nr * W4; q += blockDim.x) {
            const int rr = q / W4, b0 = (q - rr * W4) * 4;
            const uint8_t* s = work + rr * row_bytes + base + b0;
            const uint32_t w = (uint32_t)s[0] | ((uint32_t)s[1] << 8) | ((uint32_t)s[2] << 16) | ((uint32_t)s[3] << 24);
            *reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(o) + (size_t)(y0 + rr) * S * 3 + b0) = w;
        }
    } else {
        for (int q = threadIdx.x; q < nr * S; q += blockDim.x) {
            const int rr = q / S, x = q - rr * S;
            const uint8_t* s = work + rr * row_bytes + base + x * 3;
            for (int c = 0; c < 3; ++c) {
                const size_t idx = lay == PF_HWC ? ((size_t)(y0 + rr) * S + x) * 3 + c : c * plane + (size_t)(y0 + rr) * S + x;
                o[idx] = L(c * 256 + s[c]);
            }
        }
    }
}

// One (spec, band) of the general read, block-uniform (every return leaves the item); `lut`
// built by the caller.
template <int kDtype>
__device__ __forceinline__ void read_region_item(const pf_slide_desc* slides, const pf_patch_spec& sp, int spec_i,
                                                 int band, int S, int layout,
                                                 const typename RROut<kDtype>::T* lut, uint8_t* work, int work_bytes,
                                                 void* out_v) {
    using OT = typename RROut<kDtype>::T;
    const int lay = layout & 0xff;
    const pf_slide_desc& sd = slides[sp.slide];
    const int L = sp.level;
    const int LW = sd.width[L], LH = sd.height[L];
    const int side = sp.side;
    const bool pass = side == S;
    if (band * kRRBand >= S) return;
    OT* out = reinterpret_cast<OT*>(out_v);
    const size_t plane = (size_t)S * S;
    OT* o = out + (size_t)spec_i * 3 * plane;
    const int T = sd.tile_size;

    if (pass) {
        const int y0 = band * kRRBand, y1 = min(S, y0 + kRRBand);
        if (y0 >= S) return;
        const int nr = y1 - y0;
        const int X0 = sp.sx, Y0 = sp.sy + y0;
        const bool fast = X0 >= 0 && Y0 >= 0 && X0 + S <= LW && Y0 + nr <= LH && (T % 16) == 0;
        const int row_bytes = fast ? (((X0 * 3) & 15) + S * 3 + 15) & ~15 : ((S * 3 + 15) & ~15);
        const int base = stage_level_rows(sd, L, X0, Y0, S, nr, work, row_bytes, fast);
        __syncthreads();
        passthrough_out<kDtype, false>(work, row_bytes, base, nr, y0, S, lay, lut, o);
        return;
    }

    // ---- PIL resample of the whole window (one CTA per spec): fixed output-row bands, the
    // 16-byte aligned span of each window row staged with cp.async one band ahead, horizontal
    // pass with the row's taps in registers, vertical pass into the epilogue
    const AxisPlan ap = axis_plan(side, S);
    const int K = ap.ksize;
    int* s_xmin = reinterpret_cast<int*>(work);
    int* s_xsize = s_xmin + S;
    int32_t* s_w = s_xsize + S;
    double* s_red = reinterpret_cast<double*>(work + (((size_t)(2 * S + S * K) * 4 + 15) & ~size_t(15)));
    uint8_t* buf = reinterpret_cast<uint8_t*>(s_red + 2);
    const int buf_bytes = work_bytes - (int)(buf - work);
    build_axis_table(side, S, RS_PIL, s_xmin, s_xsize, s_w, s_red);  // ends with __syncthreads
    const int sx = sp.sx, sy = sp.sy;
    const bool fast = sx >= 0 && sy >= 0 && sx + side <= LW && sy + side <= LH && (T % 16) == 0;
    const int a0 = fast ? (sx * 3) & ~15 : 0;
    const int off = fast ? sx * 3 - a0 : 0;
    const int nch = (off + side * 3 + 15) / 16;
    const int pitch = nch * 16 + 16;
    const int cap = (buf_bytes - 3 * S * 4) / (2 * pitch + 3 * S);  // source rows per band
    PF_CHECK(cap >= 4);  // pf_read_region_fits keeps such windows off this kernel
    if (cap < 4) return;  // host checks the window fits (out_size <= 512)
    uint8_t* hb = buf + 2 * cap * pitch;  // [3][cap + 4][S]
    const int hplane = (cap + 4) * S;
    int R = (int)floor(((double)cap - 1.0 - 2.0 * ap.support) / ap.scale) + 1;
    R = R < 1 ? 1 : (R > S ? S : R);
    // this CTA's output rows: its kRRBand-row band of the patch (band-parallel across CTAs),
    // resampled in internal bands of R rows that fit the staging ring
    const int Yb0 = band * kRRBand, Yb1 = min(S, Yb0 + kRRBand);
    const int nb = (Yb1 - Yb0 + R - 1) / R;
    auto rows_of = [&](int bnd, int& r0, int& r1) {  // axis_weights' own xmin / xmax bounds
        const int y0 = Yb0 + bnd * R, y1 = min(Yb1, y0 + R);
        r0 = (int)(ap.scale * ((double)y0 + 0.5) - ap.support + 0.5);
        r0 = r0 < 0 ? 0 : r0;
        r1 = (int)(ap.scale * ((double)(y1 - 1) + 0.5) + ap.support + 0.5);
        r1 = r1 > side ? side : r1;
    };
    const int cpr = T * 3 / 16;
    auto stage = [&](int bnd) {
        int r0, r1;
        rows_of(bnd, r0, r1);
        const int nr = r1 - r0;
        uint8_t* stg = buf + (bnd & 1) * cap * pitch;
        if (fast) {
            const int c0 = a0 / 16, tx0 = c0 / cpr, e0 = c0 - tx0 * cpr;
            const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
            for (int rr = warp; rr < nr; rr += kRRThreads / 32) {
                const int Y = sy + r0 + rr;
                const int ty = Y / T, v = Y - ty * T;
                for (int ch = lane; ch < nch; ch += 32) {
                    const int e = e0 + ch, t = e / cpr;
                    rr_cp_async16(stg + rr * pitch + ch * 16, tile_ptr(sd, L, tx0 + t, ty) + (size_t)v * T * 3 + (e - t * cpr) * 16);
                }
            }
        } else {  // window touches the level edge: clamped per-pixel gather
            for (int q = threadIdx.x; q < nr * side; q += kRRThreads) {
                const int rr = q / side, xx = q - rr * side;
                const uint8_t* p = level_pixel(sd, L, clampi(sx + xx, 0, LW - 1), clampi(sy + r0 + rr, 0, LH - 1));
                uint8_t* d = stg + rr * pitch + xx * 3;
                d[0] = p[0];
                d[1] = p[1];
                d[2] = p[2];
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    stage(0);
    for (int bnd = 0; bnd < nb; ++bnd) {
        const int y0 = Yb0 + bnd * R, y1 = min(Yb1, y0 + R);
        int r0, r1;
        rows_of(bnd, r0, r1);
        const int nr = r1 - r0;
        if (bnd + 1 < nb) stage(bnd + 1);
        else asm volatile("cp.async.commit_group;\n" ::: "memory");
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        __syncthreads();
        const uint8_t* stg = buf + (bnd & 1) * cap * pitch;
        // horizontal pass: item = (4 source rows, output column)
        const int ngr = (nr + 3) >> 2;
        for (int q = threadIdx.x; q < ngr * S; q += kRRThreads) {
            const int g = q / S, x = q - g * S;
            const int rr0 = g * 4, rr1 = min(nr, rr0 + 4);
            switch (K) {
                case 3: pil_h_rows<3>(stg, pitch, off, s_xmin[x], s_xsize[x], s_w + x * K, rr0, rr1, hb + x, S, hplane); break;
                case 5: pil_h_rows<5>(stg, pitch, off, s_xmin[x], s_xsize[x], s_w + x * K, rr0, rr1, hb + x, S, hplane); break;
                case 7: pil_h_rows<7>(stg, pitch, off, s_xmin[x], s_xsize[x], s_w + x * K, rr0, rr1, hb + x, S, hplane); break;
                case 9: pil_h_rows<9>(stg, pitch, off, s_xmin[x], s_xsize[x], s_w + x * K, rr0, rr1, hb + x, S, hplane); break;
                default: pil_h_rows<0>(stg, pitch, off, s_xmin[x], s_xsize[x], s_w + x * K, rr0, rr1, hb + x, S, hplane); break;
            }
        }
        __syncthreads();
        // vertical pass -> output rows [y0, y1)
        for (int q = threadIdx.x; q < (y1 - y0) * S; q += kRRThreads) {
            const int yy = q / S, x = q - yy * S;
            const int y = y0 + yy;
            const int ymin = s_xmin[y] - r0, ys = s_xsize[y];
            const int32_t* wy = s_w + y * K;
            int32_t a[3] = {1 << 21, 1 << 21, 1 << 21};
            const uint8_t* col = hb + ymin * S + x;
            for (int k = 0; k < ys; ++k) {
                const int32_t wk = wy[k];
                a[0] += (int32_t)col[k * S] * wk;
                a[1] += (int32_t)col[hplane + k * S] * wk;
                a[2] += (int32_t)col[2 * hplane + k * S] * wk;
            }
            for (int c = 0; c < 3; ++c) {
                const size_t idx = lay == PF_HWC ? ((size_t)y * S + x) * 3 + c : c * plane + (size_t)y * S + x;
                o[idx] = lut[c * 256 + clip_shift(a[c], 22)];
            }
        }
        __syncthreads();
    }
}

// Block = (spec, kRRBand-row band); with PF_SKIP_PASSTHROUGH (the multi-crop loaders: the
// general path is then only for the rare resampled windows the exact 2:1 kernel cannot take)
// a block takes a whole spec's bands, so the many specs other kernels take cost one block each
// instead of n_bands.
template <int kDtype>
__global__ void __launch_bounds__(kRRThreads) read_regions_kernel(const pf_slide_desc* slides,
                                                                  const pf_patch_spec* specs, int S, int layout,
                                                                  int n_bands, NormParams np, void* out_v) {
    using OT = typename RROut<kDtype>::T;
    extern __shared__ __align__(16) uint8_t smem[];
    const bool per_spec = layout & PF_SKIP_PASSTHROUGH;
    const int spec_i = per_spec ? (int)blockIdx.x : (int)blockIdx.x / n_bands;
    const int band0 = per_spec ? 0 : (int)blockIdx.x - spec_i * n_bands;
    const pf_patch_spec sp = specs[spec_i];
    const bool pass = sp.side == S;
    if (pass && per_spec) return;
    if (!pass && is_2x(sp, slides[sp.slide], S)) return;  // resample2x_kernel takes it
    OT* lut = reinterpret_cast<OT*>(smem);
    uint8_t* work = smem + ((3 * 256 * sizeof(OT) + 15) & ~size_t(15));
    const int work_bytes = kRRSmem - (int)(work - smem);
    for (int i = threadIdx.x; i < 3 * 256; i += kRRThreads) {
        const int c = i >> 8;
        const uint8_t v = (uint8_t)(i & 255);
        if constexpr (kDtype == PF_U8) lut[i] = v;
        else {
            const float f = __fdiv_rn(__fdiv_rn((float)v, 255.0f) - np.mean[c], np.stdv[c]);
            if constexpr (kDtype == PF_F32) lut[i] = f;
            else lut[i] = __float2bfloat16_rn(f);
        }
    }
    for (int band = band0; band < (per_spec ? n_bands : band0 + 1); ++band) {
        read_region_item<kDtype>(slides, sp, spec_i, band, S, layout, lut, work, work_bytes, out_v);
        __syncthreads();  // the band's staging / planes are reused by the next
    }
}

// PF_SKIP_RESAMPLED launches (every spec a passthrough, e.g. BASELINE config 1): a lean
// kernel of kPTBand-row bands with only the band's staged rows in shared memory (~19 KB at 224 px: 8
// CTAs per SM instead of read_regions_kernel's 2) and the normalising LUT read from a global
// table through L1 instead of 768 divided entries built per CTA.  28-row bands (8 per 224 px
// patch: 2048 CTAs for C1's 256 patches, ~19 KB so still 8 CTAs per SM) measured 4 % faster than
// 16 (C1 4.04 -> 4.21 M patches/s); 12, 20, 24 and 32 rows no better than 16, and 32 rows exceed
// the 48 KB default dynamic shared memory at out_size 512.  Streaming (.cs) stores, and 6 or 8
// CTAs per SM forced by __launch_bounds__ (5 at 48 registers): neutral.  A
// persistent grid double-buffering the next band's rows was no faster.
#ifndef PF_PT_BAND
#define PF_PT_BAND 28
#endif
constexpr int kPTBand = PF_PT_BAND;
template <int kDtype>
__global__ void __launch_bounds__(256) passthrough_kernel(const pf_slide_desc* slides, const pf_patch_spec* specs,
                                                          int S, int layout, int n_bands,
                                                          const typename RROut<kDtype>::T* glut, void* out_v) {
    using OT = typename RROut<kDtype>::T;
    extern __shared__ __align__(16) uint8_t smem[];
    const int spec_i = (int)blockIdx.x / n_bands;
    const int band = (int)blockIdx.x - spec_i * n_bands;
    const pf_patch_spec sp = specs[spec_i];
    if (sp.side != S) return;  // resampled specs are left untouched (PF_SKIP_RESAMPLED)
    const pf_slide_desc& sd = slides[sp.slide];
    const int L = sp.level, T = sd.tile_size;
    const int y0 = band * kPTBand, y1 = min(S, y0 + kPTBand);
    if (y0 >= S) return;
    const int nr = y1 - y0, X0 = sp.sx, Y0 = sp.sy + y0;
    const bool fast = X0 >= 0 && Y0 >= 0 && X0 + S <= sd.width[L] && Y0 + nr <= sd.height[L] && (T % 16) == 0;
    const int row_bytes = fast ? (((X0 * 3) & 15) + S * 3 + 15) & ~15 : ((S * 3 + 15) & ~15);
    const int base = stage_level_rows(sd, L, X0, Y0, S, nr, smem, row_bytes, fast);
    __syncthreads();
    OT* o = reinterpret_cast<OT*>(out_v) + (size_t)spec_i * 3 * S * S;
    passthrough_out<kDtype, true>(smem, row_bytes, base, nr, y0, S, layout & 0xff, glut, o);
}

// normalising LUT [3][256] of pf_read_regions, built once per (device, dtype, mean, std)
template <int kDtype>
__global__ void rr_lut_kernel(typename RROut<kDtype>::T* lut, NormParams np) {
    const int i = threadIdx.x + blockIdx.x * blockDim.x;
    if (i >= 3 * 256) return;
    const int c = i >> 8;
    const uint8_t v = (uint8_t)(i & 255);
    if constexpr (kDtype == PF_U8) lut[i] = v;
    else {
        const float f = __fdiv_rn(__fdiv_rn((float)v, 255.0f) - np.mean[c], np.stdv[c]);
        if constexpr (kDtype == PF_F32) lut[i] = f;
        else lut[i] = __float2bfloat16_rn(f);
    }
}

// ---------------------------------------------------------------------------
// General read_region for one spec whose window does not fit the fused kernel's shared-memory
// plan (down-ratio above ~15, or out_size > 512): PIL's two passes (Resample.c,
// ImagingResampleHorizontal / Vertical, 22-bit taps) through a global uint8 intermediate.
// Rare requests (the reference's PIL path accepts any ratio); not on the training hot path.
// ---------------------------------------------------------------------------
// coefficient table of one axis (side -> S): xmin[S], xsize[S], w[S * K] (int32, zero padded);
// the double weights are staged in w as doubles first (K doubles per output, 2K int32 slots)
__global__ void generic_coeffs_kernel(int side, int S, int K, int* xmin_t, int* xsize_t, int32_t* w_t, double* wd) {
    const AxisPlan p = axis_plan(side, S);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
        const double center = p.scale * ((double)i + 0.5);
        int xmin = (int)(center - p.support + 0.5);
        if (xmin < 0) xmin = 0;
        int xmax = (int)(center + p.support + 0.5);
        if (xmax > side) xmax = side;
        int xs = xmax - xmin;
        if (xs < 0) xs = 0;
        if (xs > K) xs = K;
        double* w = wd + (size_t)i * K;
        double ww = 0.0;
        for (int x = 0; x < xs; ++x) {
            const double v = triangle(((double)(x + xmin) - center + 0.5) * p.invscale);
            w[x] = v;
            ww += v;
        }
        if (ww != 0.0)
            for (int x = 0; x < xs; ++x) w[x] = w[x] / ww;
        xmin_t[i] = xmin;
        xsize_t[i] = xs;
        for (int k = 0; k < K; ++k) w_t[(size_t)i * K + k] = k < xs ? quantise_weight(w[k], 22) : 0;
    }
}

// horizontal pass: window rows [0, side) -> inter[side][S][3] (rows clamped: _read_window's
// +-1 px edge replication; columns clamped likewise)
__global__ void generic_hpass_kernel(const pf_slide_desc* slides, pf_patch_spec sp, int S, int K, const int* xmin_t,
                                     const int* xsize_t, const int32_t* w_t, uint8_t* inter) {
    const pf_slide_desc& sd = slides[sp.slide];
    const int L = sp.level, LW = sd.width[L], LH = sd.height[L];
    const int r = blockIdx.y;
    const int Y = clampi(sp.sy + r, 0, LH - 1);
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < S; x += gridDim.x * blockDim.x) {
        const int xm = xmin_t[x], xs = xsize_t[x];
        const int32_t* w = w_t + (size_t)x * K;
        int32_t a0 = 1 << 21, a1 = 1 << 21, a2 = 1 << 21;
        for (int k = 0; k < xs; ++k) {
            const uint8_t* p = level_pixel(sd, L, clampi(sp.sx + xm + k, 0, LW - 1), Y);
            a0 += (int32_t)p[0] * w[k];
            a1 += (int32_t)p[1] * w[k];
            a2 += (int32_t)p[2] * w[k];
        }
        uint8_t* d = inter + ((size_t)r * S + x) * 3;
        d[0] = clip_shift(a0, 22);
        d[1] = clip_shift(a1, 22);
        d[2] = clip_shift(a2, 22);
    }
}

// vertical pass (or the passthrough copy when the window already is S x S) -> normalised output
template <int kDtype>
__global__ void generic_vpass_kernel(const pf_slide_desc* slides, pf_patch_spec sp, int S, int K, const int* xmin_t,
                                     const int* xsize_t, const int32_t* w_t, const uint8_t* inter, int layout,
                                     NormParams np, void* out) {
    const int y = blockIdx.y;
    const size_t plane = (size_t)S * S;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < S; x += gridDim.x * blockDim.x) {
        uint8_t px[3];
        if (inter) {
            const int ym = xmin_t[y], ys = xsize_t[y];
            const int32_t* w = w_t + (size_t)y * K;
            int32_t a[3] = {1 << 21, 1 << 21, 1 << 21};
            for (int k = 0; k < ys; ++k) {
                const uint8_t* p = inter + ((size_t)(ym + k) * S + x) * 3;
                a[0] += (int32_t)p[0] * w[k];
                a[1] += (int32_t)p[1] * w[k];
                a[2] += (int32_t)p[2] * w[k];
            }
            for (int c = 0; c < 3; ++c) px[c] = clip_shift(a[c], 22);
        } else {  // side == S: the window itself (clamped at the level edge)
            const pf_slide_desc& sd = slides[sp.slide];
            const int L = sp.level;
            const uint8_t* p = level_pixel(sd, L, clampi(sp.sx + x, 0, sd.width[L] - 1), clampi(sp.sy + y, 0, sd.height[L] - 1));
            px[0] = p[0], px[1] = p[1], px[2] = p[2];
        }
        for (int c = 0; c < 3; ++c) {
            const size_t idx = layout == PF_HWC ? ((size_t)y * S + x) * 3 + c : c * plane + (size_t)y * S + x;
            store_px<kDtype>(out, idx, px[c], c, np);
        }
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
    if (n < 0 || out_size < 1 || (n > 0 && (!slides_dev || !specs_dev || !out)))
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
    if ((layout & PF_SKIP_RESAMPLED) && (layout & PF_SKIP_PASSTHROUGH)) return PF_OK;
    if (layout & PF_SKIP_RESAMPLED) {  // passthrough specs only: the lean kernel
        cudaStream_t st = as_stream(stream);
        int rc;
        const void* lut = nullptr;
        {
            static std::mutex mu;
            static std::map<std::array<uint32_t, 8>, void*> luts;
            int cur = 0;
            if ((rc = check_cuda(cudaGetDevice(&cur), "cudaGetDevice"))) return rc;
            std::array<uint32_t, 8> key{(uint32_t)cur, (uint32_t)dtype};
            std::memcpy(key.data() + 2, np.mean, 12);
            std::memcpy(key.data() + 5, np.stdv, 12);
            std::lock_guard<std::mutex> lock(mu);
            auto it = luts.find(key);
            if (it == luts.end()) {
                void* p = nullptr;
                const size_t elt = dtype == PF_F32 ? 4 : (dtype == PF_BF16 ? 2 : 1);
                if ((rc = check_cuda(cudaMalloc(&p, 3 * 256 * elt), "cudaMalloc"))) return rc;
                if (dtype == PF_U8) rr_lut_kernel<PF_U8><<<3, 256, 0, st>>>(static_cast<uint8_t*>(p), np);
                else if (dtype == PF_F32) rr_lut_kernel<PF_F32><<<3, 256, 0, st>>>(static_cast<float*>(p), np);
                else rr_lut_kernel<PF_BF16><<<3, 256, 0, st>>>(static_cast<__nv_bfloat16*>(p), np);
                if ((rc = after_launch("rr_lut_kernel"))) return rc;
                // later calls may come from other streams: complete before it is shared
                if ((rc = check_cuda(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return rc;
                it = luts.emplace(key, p).first;
            }
            lut = it->second;
        }
        const int nbp = (out_size + kPTBand - 1) / kPTBand;
        const int smem = kPTBand * (((15 + out_size * 3 + 15) & ~15) + 16);  // <= 44 KB (out_size <= 512)
        const unsigned grid = (unsigned)((long long)n * nbp);
        switch (dtype) {
            case PF_U8:
                passthrough_kernel<PF_U8><<<grid, 256, smem, st>>>(slides_dev, specs_dev, out_size, layout, nbp,
                                                                    static_cast<const uint8_t*>(lut), out);
                break;
            case PF_F32:
                passthrough_kernel<PF_F32><<<grid, 256, smem, st>>>(slides_dev, specs_dev, out_size, layout, nbp,
                                                                     static_cast<const float*>(lut), out);
                break;
            case PF_BF16:
                passthrough_kernel<PF_BF16><<<grid, 256, smem, st>>>(slides_dev, specs_dev, out_size, layout, nbp,
                                                                      static_cast<const __nv_bfloat16*>(lut), out);
                break;
            default: return fail(PF_ERR_INVALID_ARG, "pf_read_regions: bad dtype");
        }
        return after_launch("passthrough_kernel");
    }
    // every spec is split into kRRBand-row output bands across CTAs (passthrough and PIL resample
    // alike); with PF_SKIP_PASSTHROUGH the passthrough specs' CTAs exit at once
    const int n_bands = (out_size + kRRBand - 1) / kRRBand;
    const long long grid = (layout & PF_SKIP_PASSTHROUGH) ? (long long)n : (long long)n * n_bands;
    cudaStream_t st = as_stream(stream);
    int rc;
    // the exact 2:1 kernel's shared memory: LUT + (2 * kR2Rows + 2) staged rows + planar H output
    const int r2_rows = 2 * kR2Rows + 2;
    const int r2_smem = 3 * 256 * 4 + r2_rows * ((15 + 6 * out_size + 15) / 16 * 16 + 16) + 3 * r2_rows * out_size + 64;
    const int r2_bands = (out_size + kR2Rows - 1) / kR2Rows;
    const int r2_groups = (r2_bands + kR2Bands - 1) / kR2Bands;
    const bool r2 = r2_smem <= 160 * 1024;
#define PF_RR_LAUNCH(DT)                                                                                          \
    rc = check_cuda(cudaFuncSetAttribute(read_regions_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                         kRRSmem),                                                                \
                    "cudaFuncSetAttribute");                                                                      \
    if (rc) return rc;                                                                                            \
    read_regions_kernel<DT><<<(unsigned)grid, kRRThreads, kRRSmem, st>>>(slides_dev, specs_dev, out_size, layout,  \
                                                                          n_bands, np, out);                      \
    if (r2) {                                                                                                     \
        if ((rc = after_launch("read_regions_kernel"))) return rc;                                                \
        if (out_size == 224) {                                                                                    \
            rc = check_cuda(cudaFuncSetAttribute(resample2x_kernel<DT, 224>,                                      \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, r2_smem),           \
                            "cudaFuncSetAttribute");                                                              \
            if (rc) return rc;                                                                                    \
            resample2x_kernel<DT, 224><<<(unsigned)((long long)n * r2_groups), kR2Threads, r2_smem, st>>>(        \
                slides_dev, specs_dev, out_size, layout, r2_bands, np, out);                                      \
        } else {                                                                                                  \
            rc = check_cuda(cudaFuncSetAttribute(resample2x_kernel<DT, 0>,                                        \
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, r2_smem),           \
                            "cudaFuncSetAttribute");                                                              \
            if (rc) return rc;                                                                                    \
            resample2x_kernel<DT, 0><<<(unsigned)((long long)n * r2_groups), kR2Threads, r2_smem, st>>>(          \
                slides_dev, specs_dev, out_size, layout, r2_bands, np, out);                                      \
        }                                                                                                         \
    }
    switch (dtype) {
        case PF_U8: PF_RR_LAUNCH(PF_U8) break;
        case PF_F32: PF_RR_LAUNCH(PF_F32) break;
        case PF_BF16: PF_RR_LAUNCH(PF_BF16) break;
        default: return fail(PF_ERR_INVALID_ARG, "pf_read_regions: bad dtype");
    }
#undef PF_RR_LAUNCH
    return after_launch("read_regions_kernel");
}


namespace {
// The fused kernel's shared-memory plan for a resampled window (read_regions_kernel above):
// whether a band of >= 4 staged source rows fits.
bool fused_fits(int side, int S, int dtype) {
    if (S > 512) return false;
    if (side == S) return true;
    const AxisPlan ap = axis_plan(side, S);
    const int K = ap.ksize;
    if (K > 32) return false;
    const int osz = dtype == PF_F32 ? 4 : (dtype == PF_BF16 ? 2 : 1);
    const int lut = (3 * 256 * osz + 15) & ~15;
    const int work_bytes = kRRSmem - lut;
    const int tab = (((2 * S + S * K) * 4) + 15) & ~15;
    const int buf_bytes = work_bytes - (tab + 16);
    const int nch = (15 + side * 3 + 15) / 16;  // worst-case offset 15
    const int pitch = nch * 16 + 16;
    const int cap = (buf_bytes - 3 * S * 4) / (2 * pitch + 3 * S);
    return cap >= 4;
}
}  // namespace

extern "C" int pf_read_region_fits(int32_t side, int32_t out_size, int32_t dtype, int32_t* fits) {
    if (side < 1 || out_size < 1 || !fits) return fail(PF_ERR_INVALID_ARG, "pf_read_region_fits: bad arguments");
    *fits = fused_fits(side, out_size, dtype) ? 1 : 0;
    return PF_OK;
}

extern "C" int pf_read_region_generic_scratch_bytes(int32_t side, int32_t out_size, int64_t* bytes) {
    if (side < 1 || out_size < 1 || !bytes) return fail(PF_ERR_INVALID_ARG, "pf_read_region_generic_scratch_bytes: bad arguments");
    const int64_t K = axis_plan(side, out_size).ksize;
    const int64_t S = out_size;
    *bytes = 2 * S * 4 + S * K * 4 + S * K * 8 + (int64_t)side * S * 3 + 64;
    return PF_OK;
}

extern "C" int pf_read_region_generic(const pf_slide_desc* slides_dev, const pf_patch_spec* spec, int32_t out_size,
                                      int32_t dtype, int32_t layout, const float* mean3, const float* std3,
                                      void* scratch_dev, int64_t scratch_bytes, void* out, void* stream) {
    if (!slides_dev || !spec || out_size < 1 || !out || spec->side < 1)
        return fail(PF_ERR_INVALID_ARG, "pf_read_region_generic: bad arguments");
    if (layout != PF_HWC && layout != PF_NCHW) return fail(PF_ERR_INVALID_ARG, "pf_read_region_generic: bad layout");
    if (dtype != PF_U8 && dtype != PF_F32 && dtype != PF_BF16)
        return fail(PF_ERR_INVALID_ARG, "pf_read_region_generic: bad dtype");
    const int S = out_size, side = spec->side;
    NormParams np;
    for (int c = 0; c < 3; ++c) {
        np.mean[c] = mean3 ? mean3[c] : 0.5f;
        np.stdv[c] = std3 ? std3[c] : 0.5f;
    }
    cudaStream_t st = as_stream(stream);
    const int K = axis_plan(side, S).ksize;
    int* xmin_t = nullptr;
    int* xsize_t = nullptr;
    int32_t* w_t = nullptr;
    uint8_t* inter = nullptr;
    if (side != S) {
        int64_t need = 0;
        pf_read_region_generic_scratch_bytes(side, S, &need);
        if (!scratch_dev || scratch_bytes < need)
            return fail(PF_ERR_CAPACITY, "pf_read_region_generic: scratch too small");
        uint8_t* base = static_cast<uint8_t*>(scratch_dev);
        double* wd = reinterpret_cast<double*>(base);
        xmin_t = reinterpret_cast<int*>(base + (size_t)S * K * 8);
        xsize_t = xmin_t + S;
        w_t = xsize_t + S;
        inter = reinterpret_cast<uint8_t*>(w_t + (size_t)S * K);
        generic_coeffs_kernel<<<(S + 127) / 128, 128, 0, st>>>(side, S, K, xmin_t, xsize_t, w_t, wd);
        int rc = after_launch("generic_coeffs_kernel");
        if (rc) return rc;
        generic_hpass_kernel<<<dim3((S + 127) / 128, side), 128, 0, st>>>(slides_dev, *spec, S, K, xmin_t, xsize_t,
                                                                         w_t, inter);
        if ((rc = after_launch("generic_hpass_kernel"))) return rc;
    }
    const dim3 grid((S + 127) / 128, S);
    switch (dtype) {
        case PF_U8:
            generic_vpass_kernel<PF_U8><<<grid, 128, 0, st>>>(slides_dev, *spec, S, K, xmin_t, xsize_t, w_t, inter, layout, np, out);
            break;
        case PF_F32:
            generic_vpass_kernel<PF_F32><<<grid, 128, 0, st>>>(slides_dev, *spec, S, K, xmin_t, xsize_t, w_t, inter, layout, np, out);
            break;
        default:
            generic_vpass_kernel<PF_BF16><<<grid, 128, 0, st>>>(slides_dev, *spec, S, K, xmin_t, xsize_t, w_t, inter, layout, np, out);
            break;
    }
    return after_launch("generic_vpass_kernel");
}
