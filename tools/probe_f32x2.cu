// Probe: are the packed f32x2 ops (Blackwell FFMA2/FADD2/FMUL2) bit-identical to their scalar
// IEEE counterparts (fused fma, directed rounding, subnormals)?  nvcc -arch=sm_100a, run on a B200.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
__device__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n.reg .b64 A, B, Cc, D;\nmov.b64 A, {%2, %3};\nmov.b64 B, {%4, %5};\nmov.b64 Cc, {%6, %7};\n"
        "fma.rn.f32x2 D, A, B, Cc;\nmov.b64 {%0, %1}, D;\n}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
__device__ float2 addrm2(float2 a, float2 b) {
    float2 d;
    asm("{\n.reg .b64 A, B, D;\nmov.b64 A, {%2, %3};\nmov.b64 B, {%4, %5};\nadd.rm.f32x2 D, A, B;\nmov.b64 {%0, %1}, D;\n}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ float2 mul2(float2 a, float2 b) {
    float2 d;
    asm("{\n.reg .b64 A, B, D;\nmov.b64 A, {%2, %3};\nmov.b64 B, {%4, %5};\nmul.rn.f32x2 D, A, B;\nmov.b64 {%0, %1}, D;\n}"
        : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    return d;
}
__device__ uint32_t h(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; return x ^ (x >> 16); }
__global__ void k(unsigned long long* bad, int mode) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    float a = __uint_as_float((h(3 * i) & 0x3fffffffu) | 0x3f000000u) - 1.0f;  // ~[-0.5, 1)
    float b = __uint_as_float((h(3 * i + 1) & 0x007fffffu) | 0x3f800000u);     // [1, 2)
    float c = __uint_as_float((h(3 * i + 2) & 0x007fffffu) | 0x3f800000u) - 1.5f;
    if (mode == 1) { b = -b; }
    if (mode == 2) { a *= 1e-38f; }  // subnormal range products / sums
    const float2 r = fma2(make_float2(a, c), make_float2(b, b), make_float2(c, a));
    const float2 s = addrm2(make_float2(a, c), make_float2(b, c * 3.0f));
    const float2 m = mul2(make_float2(a, c), make_float2(b, a));
    if (__float_as_uint(r.x) != __float_as_uint(__fmaf_rn(a, b, c))) atomicAdd(bad + 0, 1ull);
    if (__float_as_uint(r.y) != __float_as_uint(__fmaf_rn(c, b, a))) atomicAdd(bad + 0, 1ull);
    if (__float_as_uint(s.x) != __float_as_uint(__fadd_rd(a, b))) atomicAdd(bad + 1, 1ull);
    if (__float_as_uint(s.y) != __float_as_uint(__fadd_rd(c, c * 3.0f))) atomicAdd(bad + 1, 1ull);
    if (__float_as_uint(m.x) != __float_as_uint(__fmul_rn(a, b))) atomicAdd(bad + 2, 1ull);
    if (__float_as_uint(m.y) != __float_as_uint(__fmul_rn(c, a))) atomicAdd(bad + 2, 1ull);
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 3 * sizeof(unsigned long long));
    for (int mode = 0; mode < 3; ++mode) {
        cudaMemset(d, 0, 3 * sizeof(unsigned long long));
        k<<<1 << 16, 256>>>(d, mode);
        unsigned long long hbad[3];
        cudaMemcpy(hbad, d, sizeof hbad, cudaMemcpyDeviceToHost);
        printf("mode %d: fma2 mismatches %llu, add.rm2 %llu, mul2 %llu (of %d)\n", mode, hbad[0], hbad[1], hbad[2], 2 << 24);
    }
    return 0;
}
