// Probe: packed hue (hue_b2) vs scalar hue (f_hue) over every RGB colour and a few shifts.
// Prints mismatch counts and the first mismatching colours.  Run on a B200.
#include <cstdio>
#include <cstdint>
#include "../paper_2404_15217_b200/csrc/pf_color.cuh"
using namespace pf;
__global__ void k(float hf, unsigned long long* bad, uint32_t* first) {
    const uint32_t c0 = 2u * (blockIdx.x * blockDim.x + threadIdx.x);  // colours c0, c0 + 1
    float R[2], G[2], B[2];
    float2 Rb, Gb, Bb;
    for (int e = 0; e < 2; ++e) {
        const uint32_t c = c0 + e;
        R[e] = (float)(c >> 16), G[e] = (float)((c >> 8) & 255), B[e] = (float)(c & 255);
    }
    Rb = make_float2(R[0] + kMagic, R[1] + kMagic);
    Gb = make_float2(G[0] + kMagic, G[1] + kMagic);
    Bb = make_float2(B[0] + kMagic, B[1] + kMagic);
    hue_b2(Rb, Gb, Bb, hf);
    const float pr[2] = {Rb.x, Rb.y}, pg[2] = {Gb.x, Gb.y}, pb[2] = {Bb.x, Bb.y};
    for (int e = 0; e < 2; ++e) {
        float r = R[e], g = G[e], b = B[e];
        f_hue(r, g, b, hf);
        if (r != pr[e] - kMagic || g != pg[e] - kMagic || b != pb[e] - kMagic) {
            const unsigned long long n = atomicAdd(bad, 1ull);
            if (n < 8) {
                first[4 * n] = c0 + e;
                first[4 * n + 1] = ((uint32_t)r << 16) | ((uint32_t)g << 8) | (uint32_t)b;
                first[4 * n + 2] = ((uint32_t)(pr[e] - kMagic) << 16) | ((uint32_t)(pg[e] - kMagic) << 8) | (uint32_t)(pb[e] - kMagic);
            }
        }
    }
}
int main() {
    unsigned long long* d;
    uint32_t* f;
    cudaMalloc(&d, 8);
    cudaMalloc(&f, 4 * 8 * 4);
    const float hs[] = {-0.46440213918685913f, -0.1f, 0.05f, 0.3f, 0.5f};
    for (float hf : hs) {
        cudaMemset(d, 0, 8);
        k<<<(1 << 23) / 256, 256>>>(hf, d, f);
        unsigned long long n;
        uint32_t h[32];
        cudaMemcpy(&n, d, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(h, f, sizeof h, cudaMemcpyDeviceToHost);
        printf("hf %.8f: %llu mismatches\n", hf, n);
        for (unsigned i = 0; i < (n < 8 ? n : 8); ++i)
            printf("  colour %06x scalar %06x packed %06x\n", h[4 * i], h[4 * i + 1], h[4 * i + 2]);
    }
    return 0;
}
