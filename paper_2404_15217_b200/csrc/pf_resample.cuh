// Separable antialiased bilinear ("triangle") resampling with fixed-point
// integer taps, in the two flavours the hot path must reproduce bit-exactly:
//
//  * PIL Image.resize(BILINEAR) — Pillow Resample.c precompute_coeffs +
//    normalize_coeffs_8bpc: 22-bit int32 weights.  Used by Slide.read_region
//    when the window side != out_size (pkg/store.py:685-687).
//  * torch uint8 antialiased bilinear (aten upsample AA, the CPU path under
//    torchvision.transforms.v2.functional.resized_crop): the same double
//    weights quantised to int16 with a per-axis precision p chosen from the
//    largest weight.  Used by RandomResizedCrop in the multi-crop kernel.
//
// Both compute out = clamp((2^(p-1) + sum_k w_k * in[xmin+k]) >> p, 0, 255)
// per axis, horizontal pass first, with a uint8 intermediate.  Every double
// operation below is a single IEEE op (the library is built -fmad=false), in
// the evaluation order of the C sources they restate.
#pragma once

#include <math.h>
#include <stdint.h>

namespace pf {

enum ResampleFlavour { RS_PIL = 0, RS_TORCH = 1 };

struct AxisPlan {
    double scale, support, invscale;
    int ksize;
};

__host__ __device__ inline AxisPlan axis_plan(int in_size, int out_size) {
    AxisPlan p;
    p.scale = (double)in_size / (double)out_size;
    const double filterscale = p.scale < 1.0 ? 1.0 : p.scale;
    p.support = 1.0 * filterscale;  // bilinear support 1.0
    p.invscale = 1.0 / filterscale;
    p.ksize = (int)ceil(p.support) * 2 + 1;
    return p;
}

__host__ __device__ inline double triangle(double x) {
    if (x < 0.0) x = -x;
    if (x < 1.0) return 1.0 - x;
    return 0.0;
}

// Bounds and normalised double weights of output index i.  Returns xsize.
__host__ __device__ inline int axis_weights(const AxisPlan& p, int in_size, int i, int* xmin_out,
                                            double* w /* [ksize] */) {
    const double center = p.scale * ((double)i + 0.5);
    int xmin = (int)(center - p.support + 0.5);
    if (xmin < 0) xmin = 0;
    int xmax = (int)(center + p.support + 0.5);
    if (xmax > in_size) xmax = in_size;
    int xsize = xmax - xmin;
    if (xsize < 0) xsize = 0;
    if (xsize > p.ksize) xsize = p.ksize;
    double ww = 0.0;
    for (int x = 0; x < xsize; ++x) {
        const double v = triangle(((double)(x + xmin) - center + 0.5) * p.invscale);
        w[x] = v;
        ww += v;
    }
    if (ww != 0.0)
        for (int x = 0; x < xsize; ++x) w[x] = w[x] / ww;
    *xmin_out = xmin;
    return xsize;
}

__host__ __device__ inline int32_t quantise_weight(double v, int prec) {
    const double s = v * (double)(1 << prec);
    return v < 0 ? (int32_t)(-0.5 + s) : (int32_t)(0.5 + s);
}

// torch: largest p < 22 with (int)(0.5 + wmax * 2^(p+1)) < 2^15.
__host__ __device__ inline int torch_precision(double wmax) {
    int p = 0;
    for (p = 0; p < 22; ++p) {
        const int next = (int)(0.5 + wmax * (double)(1 << (p + 1)));
        if (next >= (1 << 15)) break;
    }
    return p;
}

__device__ __forceinline__ uint8_t clip_shift(int32_t acc, int prec) {
    int32_t v = acc >> prec;  // arithmetic shift (floor)
    return (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
}

// CTA-cooperative coefficient table for one axis, into shared memory:
// xmin[out], xsize[out], w[out * ksize] (int32, zero padded).  Returns the
// precision (22 for PIL).  `red` is >= 1 double of shared scratch.  Must be
// called by all threads of the block.
__device__ inline int build_axis_table(int in_size, int out_size, int flavour, int* s_xmin,
                                       int* s_xsize, int32_t* s_w, double* s_red) {
    const AxisPlan p = axis_plan(in_size, out_size);
    double w[32];  // ksize <= 32 supports down-ratios up to 15x
    int prec = 22;
    if (flavour == RS_TORCH) {
        double local_max = 0.0;
        for (int i = threadIdx.x; i < out_size; i += blockDim.x) {
            int xmin;
            const int xs = axis_weights(p, in_size, i, &xmin, w);
            for (int k = 0; k < xs; ++k) local_max = fmax(local_max, w[k]);
        }
        // block max (non-negative doubles: compare as int64 bit patterns)
        if (threadIdx.x == 0) *s_red = 0.0;
        __syncthreads();
        atomicMax(reinterpret_cast<unsigned long long*>(s_red),
                  (unsigned long long)__double_as_longlong(local_max));
        __syncthreads();
        prec = torch_precision(*s_red);
    }
    for (int i = threadIdx.x; i < out_size; i += blockDim.x) {
        int xmin;
        const int xs = axis_weights(p, in_size, i, &xmin, w);
        s_xmin[i] = xmin;
        s_xsize[i] = xs;
        for (int k = 0; k < p.ksize; ++k) s_w[i * p.ksize + k] = k < xs ? quantise_weight(w[k], prec) : 0;
    }
    __syncthreads();
    return prec;
}

}  // namespace pf
