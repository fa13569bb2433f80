// Shared helpers for the pf_b200 kernels: status plumbing, launch accounting,
// pyramid addressing and the reference's rounding rules.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/pf_b200.h"

// PF_CHECKS builds (tools/build_variant.py checks ... -DPF_CHECKS; tests run against the result
// with PF_B200_LIB) trap on any staged-buffer / table index outside its allocation: the
// in-house substitute for compute-sanitizer, which this GPU pool does not allow.
#ifdef PF_CHECKS
#include <cstdio>
#define PF_CHECK(cond)                                                                                   \
    do {                                                                                                 \
        if (!(cond)) {                                                                                   \
            printf("PF_CHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__,      \
                   (int)blockIdx.x, (int)threadIdx.x);                                                   \
            __trap();                                                                                    \
        }                                                                                                \
    } while (0)
#else
#define PF_CHECK(cond) ((void)0)
#endif

namespace pf {

// Dynamic shared memory of the launch (for PF_CHECK bounds on carved shared layouts).
__device__ __forceinline__ uint32_t dynamic_smem_size() {
    uint32_t r;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}

// Thread-local last error; set by every failing entry point.
void set_error(const std::string& msg);
int fail(int status, const std::string& msg);
int check_cuda(cudaError_t err, const char* what);
void count_launch();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Launch-check helper used right after every <<<>>>.
inline int after_launch(const char* what) {
    count_launch();
    return check_cuda(cudaGetLastError(), what);
}

// round_half_away for x >= 0 (pkg/store.py:70-72): floor(x + 0.5).
__host__ __device__ inline int64_t rha_nonneg(double x) {
#ifdef __CUDA_ARCH__
    return (int64_t)floor(__dadd_rn(x, 0.5));
#else
    return (int64_t)floor(x + 0.5);
#endif
}

// First byte of tile (tx, ty) of a level: dense tile-major, or through the
// residency slot map (non-resident tiles -> the zero hole slot 0).
__device__ __forceinline__ const uint8_t* tile_ptr(const pf_slide_desc& s, int level, int tx, int ty) {
    const size_t tile_bytes = (size_t)s.tile_size * s.tile_size * 3;
    const uint8_t* base = reinterpret_cast<const uint8_t*>(s.level_ptr[level]);
    const size_t t = (size_t)ty * s.tiles_x[level] + tx;
    const int32_t* map = reinterpret_cast<const int32_t*>(s.tile_map[level]);
    if (!map) return base + t * tile_bytes;
    const int32_t slot = __ldg(map + t);
    if (slot == 0 && s.status_word)  // the zero hole: the read plan missed this tile (fail loudly;
        atomicCAS(reinterpret_cast<int*>(s.status_word), 0, PF_ERR_OUT_OF_BOUNDS);  // first fault sticks)
    return base + (size_t)slot * tile_bytes;
}

// Address of pixel (X, Y) in a padded tile-major level (see pf_b200.h).
__device__ __forceinline__ const uint8_t* level_pixel(const pf_slide_desc& s, int level, int X,
                                                      int Y) {
    const int T = s.tile_size;
    const int tx = X / T, ty = Y / T;
    const int u = X - tx * T, v = Y - ty * T;
    return tile_ptr(s, level, tx, ty) + ((size_t)v * T + u) * 3;
}

__device__ __forceinline__ uint8_t* level_pixel_mut(const pf_slide_desc& s, int level, int X,
                                                    int Y) {
    return const_cast<uint8_t*>(level_pixel(s, level, X, Y));
}

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// SplitMix64 finaliser (pkg/rng.py:25-30).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Draw `counter` (1-based) of a stream with key `key` (pkg/rng.py:60-62).
__host__ __device__ __forceinline__ uint64_t stream_u64(uint64_t key, uint64_t counter) {
    return mix64(key + counter * 0x9E3779B97F4A7C15ull);
}

// RandomStream.uniform(0, 1) (pkg/rng.py:64-67): (u >> 11) * 2^-53, exact.
__host__ __device__ __forceinline__ double u64_to_unit(uint64_t u) {
    return (double)(u >> 11) * 1.1102230246251565e-16;  // 2^-53
}

// randrange limit (pkg/rng.py:69-77): floor(2^64 / n) * n; returns 0 to mean 2^64.
__host__ __device__ __forceinline__ uint64_t randrange_limit(uint64_t n) {
    // 2^64 mod n == (2^64 - n) mod n
    const uint64_t rem = (0ull - n) % n;
    return 0ull - rem;  // 2^64 - rem, wraps to 0 when rem == 0
}
__host__ __device__ __forceinline__ bool randrange_accepts(uint64_t v, uint64_t limit) {
    return limit == 0ull || v < limit;
}

// randrange_accepts(v, randrange_limit(n)) without the 64-bit division on the common path:
// limit = 2^64 - (2^64 mod n) > 2^64 - n, so v < 2^64 - n accepts outright; only a draw in
// the top n values (probability n / 2^64) computes the exact limit.
__device__ __forceinline__ bool randrange_accepts_n(uint64_t v, uint64_t n) {
    return v < 0ull - n || randrange_accepts(v, randrange_limit(n));
}

// v % n (1 <= n < 2^50) without the 64-bit division subroutine: two FP64 quotient estimates
// and one exact correction.  Pass 1: q = trunc(rz(v) * rn(1/n)) is within 3*2^-52*v/n + 1 of
// v/n, so r1 = v - q*n (exact in wrapping arithmetic) has |r1| <= 3*2^12 + n.  Pass 2:
// rn(r1 * rn(1/n)) is within 2^-40 of r1/n, so its floor is floor(r1/n) or one off when r1/n
// is that close to an integer, and r2 = r1 - floor(.)*n lies in [-n, 2n).  (Written as loops,
// the correction is turned into a division by the compiler.)
__device__ __forceinline__ uint64_t mod_u64(uint64_t v, uint64_t n) {
    if (n >= (1ull << 50)) return v % n;
    const double inv = __drcp_rn((double)n);
    const uint64_t q = __double2ull_rz(__dmul_rn(__ull2double_rz(v), inv));
    int64_t r = (int64_t)(v - q * n);
    r -= __double2ll_rd(__dmul_rn((double)r, inv)) * (int64_t)n;
    if (r < 0) r += (int64_t)n;
    else if (r >= (int64_t)n) r -= (int64_t)n;
    return (uint64_t)r;
}

}  // namespace pf
