// Synthetic H&E-like slide generator (BASELINE.json configs; stands in for
// TCGA WSIs).  Level 0 is written straight into the padded tile-major HBM
// layout; upper levels come from pf_build_level.  Deterministic in
// (field, threshold, seed).
#include "pf_common.cuh"

namespace pf {

__device__ __forceinline__ float hash_normal(uint64_t seed, uint64_t idx, int which) {
    const uint64_t h = mix64(seed ^ mix64(idx * 3ull + (uint64_t)which + 0x51ed2701ull));
    const float u1 = ((float)(uint32_t)(h >> 40) + 0.5f) * (1.0f / 16777216.0f);
    const float u2 = (float)(uint32_t)(h & 0xffffffu) * (1.0f / 16777216.0f);
    return sqrtf(-2.0f * __logf(u1)) * __cosf(6.28318530718f * u2);
}

__device__ __forceinline__ uint8_t to_u8(float v) {
    v = fminf(fmaxf(v, 0.0f), 255.0f);
    return (uint8_t)__float2int_rn(v);
}

__device__ __forceinline__ float sample_field(const float* field, int fh, int fw, int cell, int X,
                                              int Y) {
    const float fx = ((float)X + 0.5f) / (float)cell - 0.5f;
    const float fy = ((float)Y + 0.5f) / (float)cell - 0.5f;
    const float cx = fminf(fmaxf(fx, 0.0f), (float)(fw - 1));
    const float cy = fminf(fmaxf(fy, 0.0f), (float)(fh - 1));
    const int x0 = min((int)cx, fw - 1), y0 = min((int)cy, fh - 1);
    const int x1 = min(x0 + 1, fw - 1), y1 = min(y0 + 1, fh - 1);
    const float ax = cx - (float)x0, ay = cy - (float)y0;
    const float a = field[y0 * fw + x0], b = field[y0 * fw + x1];
    const float c = field[y1 * fw + x0], d = field[y1 * fw + x1];
    return (a * (1.0f - ax) + b * ax) * (1.0f - ay) + (c * (1.0f - ax) + d * ax) * ay;
}

// One thread per 4 consecutive pixels of a tile row (12 bytes, 3 words).
__global__ void synth_level0_kernel(pf_slide_desc s, const float* field, int fh, int fw, int cell,
                                    float thr, uint64_t seed) {
    const int T = s.tile_size;
    const int tx = blockIdx.x, ty = blockIdx.y;
    const int quads_per_row = T / 4;
    uint8_t* tile = reinterpret_cast<uint8_t*>(s.level_ptr[0]) +
                    ((size_t)ty * s.tiles_x[0] + tx) * (size_t)T * T * 3;
    const int W = s.width[0], H = s.height[0];
    for (int q = threadIdx.x; q < T * quads_per_row; q += blockDim.x) {
        const int v = q / quads_per_row, u0 = (q - v * quads_per_row) * 4;
        const int Y = ty * T + v;
        uint32_t words[3] = {0, 0, 0};
        uint8_t* bytes = reinterpret_cast<uint8_t*>(words);
        for (int k = 0; k < 4; ++k) {
            const int X = tx * T + u0 + k;
            uint8_t r = 255, g = 255, b = 255;
            if (X < W && Y < H) {
                const float f = sample_field(field, fh, fw, cell, X, Y);
                const uint64_t idx = (uint64_t)Y * (uint64_t)W + (uint64_t)X;
                const float n0 = 4.0f * hash_normal(seed, idx, 0);
                const float n1 = 4.0f * hash_normal(seed, idx, 1);
                const float n2 = 4.0f * hash_normal(seed, idx, 2);
                if (f > thr) {
                    // depth into the tissue: pink (R220,G140,B210) -> purple (R150,G60,B140)
                    const float t = fminf((f - thr) / fmaxf(1.0f - thr, 1e-6f) * 2.5f, 1.0f);
                    r = to_u8(220.0f - 70.0f * t + n0);
                    g = to_u8(140.0f - 80.0f * t + n1);
                    b = to_u8(210.0f - 70.0f * t + n2);
                } else {
                    // near-white background 230..250, same base on all channels
                    const float base = 230.0f + 20.0f * fminf(fmaxf(f / fmaxf(thr, 1e-6f), 0.0f), 1.0f);
                    r = to_u8(base + n0);
                    g = to_u8(base + n1);
                    b = to_u8(base + n2);
                }
            }
            bytes[k * 3 + 0] = r;
            bytes[k * 3 + 1] = g;
            bytes[k * 3 + 2] = b;
        }
        uint32_t* dst = reinterpret_cast<uint32_t*>(tile + ((size_t)v * T + u0) * 3);
        dst[0] = words[0];
        dst[1] = words[1];
        dst[2] = words[2];
    }
}

}  // namespace pf

using namespace pf;

extern "C" int pf_synth_level0(const pf_slide_desc* slide, const float* field, int32_t field_h,
                               int32_t field_w, int32_t field_cell, float threshold, uint64_t seed,
                               void* stream) {
    if (!slide || !field || field_h < 1 || field_w < 1 || field_cell < 1 || slide->n_levels < 1 ||
        slide->tile_size % 4 != 0)
        return fail(PF_ERR_INVALID_ARG, "pf_synth_level0: bad arguments");
    dim3 grid(slide->tiles_x[0], slide->tiles_y[0]);
    synth_level0_kernel<<<grid, 256, 0, as_stream(stream)>>>(*slide, field, field_h, field_w,
                                                              field_cell, threshold, seed);
    return after_launch("synth_level0_kernel");
}
