// Exhaustive-edge + random check of pf::mod_u64 and pf::randrange_accepts_n against the
// plain 64-bit operators (tests/test_gpu_modu64.py builds and runs this on the GPU box).
#include <cstdio>
#include <cstdint>
#include "pf_common.cuh"

__global__ void check_kernel(uint64_t seed, int iters, unsigned long long* bad, unsigned long long* first) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        const uint64_t r0 = pf::mix64(seed + (t * iters + i) * 0x9E3779B97F4A7C15ull);
        const uint64_t r1 = pf::mix64(r0 ^ 0xD1B54A32D192ED03ull);
        const uint64_t r2 = pf::mix64(r1 + 17);
        // divisors across every magnitude up to 2^50, biased to the sampler's range
        const int bits = 1 + (int)(r2 % 50);
        uint64_t n = (r1 >> (64 - bits)) | 1ull;
        if ((r2 >> 8) % 7 == 0) n = 1 + (r1 % 70000);
        if ((r2 >> 16) % 11 == 0) n = 1ull << (r1 % 50);
        uint64_t v = r0;
        const int vk = (int)((r2 >> 24) % 6);
        if (vk == 0) v = ~0ull - (r0 % 4096);          // top of the range
        if (vk == 1) v = r0 % (n * 4 + 1);             // small numerators
        if (vk == 2) v = (r0 / n) * n + (r0 & 1 ? 0 : n - 1);  // multiples and one below
        const uint64_t want = v % n, got = pf::mod_u64(v, n);
        const bool acc_want = pf::randrange_accepts(v, pf::randrange_limit(n));
        const bool acc_got = pf::randrange_accepts_n(v, n);
        if (want != got || acc_want != acc_got) {
            if (atomicAdd(bad, 1ull) == 0) { first[0] = v; first[1] = n; first[2] = got; first[3] = want; }
        }
    }
}

int main() {
    unsigned long long *bad, *first;
    cudaMallocManaged(&bad, 8);
    cudaMallocManaged(&first, 32);
    *bad = 0;
    for (int rep = 0; rep < 8; ++rep) check_kernel<<<1184, 256>>>(0x1234567ull + rep * 0x9999ull, 64, bad, first);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("cuda error\n"); return 2; }
    printf("checked %llu mismatches %llu\n", 8ull * 1184 * 256 * 64, (unsigned long long)*bad);
    if (*bad) printf("first v=%llu n=%llu got=%llu want=%llu\n", first[0], first[1], first[2], first[3]);
    return *bad ? 1 : 0;
}
