// Tissue mask on a thumbnail.
//
// PF_MASK_LUMINANCE restates mask_from_rgb (pkg/foreground.py:141-158):
//   lum = arr.astype(f64) @ [.2126, .7152, .0722] / 255 < thr
// numpy hands the (N,3)@(3,) product to BLAS, whose per-row order on this
// image's OpenBLAS is fma(B, .0722, fma(R, .2126, G * .7152)) — verified over
// all 2^24 colours (tests/test_oracle.py pins it) — so the kernel evaluates
// exactly that expression in FP64.
// PF_MASK_SATURATION is the BASELINE rule: HSV saturation (max-min)/max > thr
// (FP64 IEEE division, 0 where max == 0), optionally followed by binary
// opening then closing with a (2r+1)^2 square and zero border
// (scipy.ndimage.binary_opening / binary_closing semantics).
#include "pf_common.cuh"

namespace pf {

__global__ void mask_kernel(const uint8_t* img, int n, int mode, double thr, uint8_t* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t r = img[3 * i], g = img[3 * i + 1], b = img[3 * i + 2];
    bool fg;
    if (mode == PF_MASK_LUMINANCE) {
        const double lum = __fma_rn((double)b, 0.0722, __fma_rn((double)r, 0.2126, __dmul_rn((double)g, 0.7152)));
        fg = __ddiv_rn(lum, 255.0) < thr;
    } else {
        const int mx = max(r, max(g, b)), mn = min(r, min(g, b));
        const double s = mx == 0 ? 0.0 : __ddiv_rn((double)(mx - mn), (double)mx);
        fg = s > thr;
    }
    out[i] = fg ? 1 : 0;
}

// erosion (is_erode) / dilation with a (2r+1)^2 square, outside pixels = 0
__global__ void morph_kernel(const uint8_t* in, int h, int w, int r, int is_erode, uint8_t* out) {
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int y = blockIdx.y;
    if (x >= w || y >= h) return;
    int acc = is_erode ? 1 : 0;
    for (int dy = -r; dy <= r; ++dy) {
        for (int dx = -r; dx <= r; ++dx) {
            const int yy = y + dy, xx = x + dx;
            const int v = (yy >= 0 && yy < h && xx >= 0 && xx < w) ? in[yy * w + xx] : 0;
            if (is_erode) acc &= v;
            else acc |= v;
        }
    }
    out[y * w + x] = (uint8_t)acc;
}

}  // namespace pf

using namespace pf;

extern "C" int pf_mask(const uint8_t* img_hwc, int32_t h, int32_t w, int32_t mode, double threshold,
                       int32_t morph_radius, uint8_t* out, uint8_t* scratch, void* stream) {
    if (!img_hwc || !out || h < 1 || w < 1)
        return fail(PF_ERR_INVALID_ARG, "pf_mask: bad arguments");
    if (mode != PF_MASK_LUMINANCE && mode != PF_MASK_SATURATION)
        return fail(PF_ERR_INVALID_ARG, "pf_mask: unknown mode");
    if (mode == PF_MASK_LUMINANCE && !(threshold > 0.0 && threshold < 1.0))
        return fail(PF_ERR_INVALID_ARG, "luminance_threshold must be in (0, 1)");
    if (morph_radius < 0 || (morph_radius > 0 && (mode != PF_MASK_SATURATION || !scratch)))
        return fail(PF_ERR_INVALID_ARG, "pf_mask: morphology needs saturation mode and scratch");
    cudaStream_t st = as_stream(stream);
    const int n = h * w;
    uint8_t* first = morph_radius > 0 ? scratch : out;
    mask_kernel<<<(n + 255) / 256, 256, 0, st>>>(img_hwc, n, mode, threshold, first);
    int rc = after_launch("mask_kernel");
    if (rc || morph_radius == 0) return rc;
    uint8_t* a = scratch;
    uint8_t* b = scratch + (size_t)n;
    dim3 grid((w + 127) / 128, h);
    // opening: erode then dilate; closing: dilate then erode
    morph_kernel<<<grid, 128, 0, st>>>(a, h, w, morph_radius, 1, b);
    if ((rc = after_launch("morph_kernel"))) return rc;
    morph_kernel<<<grid, 128, 0, st>>>(b, h, w, morph_radius, 0, a);
    if ((rc = after_launch("morph_kernel"))) return rc;
    morph_kernel<<<grid, 128, 0, st>>>(a, h, w, morph_radius, 0, b);
    if ((rc = after_launch("morph_kernel"))) return rc;
    morph_kernel<<<grid, 128, 0, st>>>(b, h, w, morph_radius, 1, out);
    return after_launch("morph_kernel");
}
