// On-GPU baseline JPEG tile decode (JPEG half; replaces
// decode_tile's Pillow path for JPEG stores, pkg/store.py:397-426).  Bit-exact with
// Pillow's libjpeg-turbo default decompression (restated and pinned in oracle/jpeg.py):
//   pf_jpeg_entropy: one warp per tile (lane 0) Huffman-decodes every block of the
//     scan (byte stuffing already removed on the host) into int16 coefficients;
//   pf_jpeg_idct: one thread per 8x8 block, dequantise + accurate integer IDCT
//     (13-bit constants, PASS1_BITS 2) into per-component sample planes;
//   pf_jpeg_color: one thread per output pixel, 2x2 "fancy" (triangle) chroma
//     upsampling (box replication for chroma <= 2 samples wide) + fixed-point
//     YCbCr -> RGB, straight into the tile's slot of the HBM pyramid.
#include <stdint.h>

#include "pf_common.cuh"
#include "pf_jpeg.h"

namespace pf {

__constant__ uint8_t kZigzag[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,
                                    12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,  7,  14, 21, 28,
                                    35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
                                    58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

struct JBits {
    const uint8_t* in;
    int32_t n, pos;
    uint32_t buf;  // MSB-aligned
    int cnt;
};

__device__ __forceinline__ void jfill(JBits& b) {
    while (b.cnt <= 24) {
        const uint32_t byte = b.pos < b.n ? b.in[b.pos] : 0xFFu;  // past the end: ones (libjpeg)
        ++b.pos;
        b.buf |= byte << (24 - b.cnt);
        b.cnt += 8;
    }
}
__device__ __forceinline__ int jbits(JBits& b, int s) {
    if (s == 0) return 0;
    jfill(b);
    const int v = (int)(b.buf >> (32 - s));
    b.buf <<= s;
    b.cnt -= s;
    return v;
}
__device__ __forceinline__ int jdecode(JBits& b, const JpegHuff& h) {
    jfill(b);
    const int e = h.fast[b.buf >> 23];
    if (e) {
        const int len = e >> 8;
        b.buf <<= len;
        b.cnt -= len;
        return e & 255;
    }
    int code = (int)(b.buf >> 22), len = 10;  // codes longer than 9 bits
    while (len <= 16 && code > h.maxcode[len]) {
        ++len;
        code = (int)(b.buf >> (32 - len));
    }
    if (len > 16) return -1;
    b.buf <<= len;
    b.cnt -= len;
    return h.huffval[(h.valoff[len] + code) & 255];
}
__device__ __forceinline__ int jextend(int v, int s) { return (s && v < (1 << (s - 1))) ? v - (1 << s) + 1 : v; }

__global__ void jpeg_entropy_kernel(const JpegTile* tiles, int n, const uint8_t* data, const JpegHuff* huff,
                                    int16_t* coef, int32_t* status) {
    const int t = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (t >= n || (threadIdx.x & 31)) return;
    const JpegTile tl = tiles[t];
    JBits b;
    b.in = data + tl.data_off;
    b.n = tl.data_len;
    b.pos = 0;
    b.buf = 0;
    b.cnt = 0;
    int pred[3] = {0, 0, 0};
    int rc = 0;
    for (int my = 0; my < tl.mcuy && !rc; ++my)
        for (int mx = 0; mx < tl.mcux && !rc; ++mx)
            for (int c = 0; c < tl.ncomp && !rc; ++c) {
                const JpegComp& cp = tl.comp[c];
                const JpegHuff& dc = huff[cp.dc];
                const JpegHuff& ac = huff[cp.ac];
                for (int v = 0; v < cp.vs && !rc; ++v)
                    for (int h = 0; h < cp.hs && !rc; ++h) {
                        int16_t* blk = coef + cp.coef_off + ((int64_t)(my * cp.vs + v) * cp.bw + mx * cp.hs + h) * 64;
                        for (int k = 0; k < 64; ++k) blk[k] = 0;
                        const int s = jdecode(b, dc);
                        if (s < 0 || s > 15) {
                            rc = -1;
                            break;
                        }
                        pred[c] += jextend(jbits(b, s), s);
                        blk[0] = (int16_t)pred[c];
                        for (int k = 1; k < 64;) {
                            const int rs = jdecode(b, ac);
                            if (rs < 0) {
                                rc = -1;
                                break;
                            }
                            const int r = rs >> 4, sz = rs & 15;
                            if (sz == 0) {
                                if (r == 15) {
                                    k += 16;
                                    continue;
                                }
                                break;
                            }
                            k += r;
                            if (k > 63) {
                                rc = -2;
                                break;
                            }
                            blk[kZigzag[k]] = (int16_t)jextend(jbits(b, sz), sz);
                            ++k;
                        }
                    }
            }
    if (!rc && b.pos > b.n + 4) rc = -3;  // ran far past the entropy-coded data
    status[t] = rc;
}

// ---- accurate integer IDCT (IJG "islow")
constexpr int kCB = 13, kP1 = 2;
__device__ __forceinline__ int jdescale(int64_t x, int n) { return (int)((x + ((int64_t)1 << (n - 1))) >> n); }

__device__ __forceinline__ void jbutterfly(int64_t i0, int64_t i1, int64_t i2, int64_t i3, int64_t i4, int64_t i5,
                                           int64_t i6, int64_t i7, int64_t (&o)[8]) {
    int64_t z1 = (i2 + i6) * 4433;
    const int64_t tmp2 = z1 + i6 * (-15137), tmp3 = z1 + i2 * 6270;
    const int64_t tmp0 = (i0 + i4) * (1 << kCB), tmp1 = (i0 - i4) * (1 << kCB);
    const int64_t tmp10 = tmp0 + tmp3, tmp13 = tmp0 - tmp3, tmp11 = tmp1 + tmp2, tmp12 = tmp1 - tmp2;
    int64_t t0 = i7, t1 = i5, t2 = i3, t3 = i1;
    z1 = t0 + t3;
    int64_t z2 = t1 + t2, z3 = t0 + t2, z4 = t1 + t3;
    const int64_t z5 = (z3 + z4) * 9633;
    t0 *= 2446;
    t1 *= 16819;
    t2 *= 25172;
    t3 *= 12299;
    z1 *= -7373;
    z2 *= -20995;
    z3 = z3 * (-16069) + z5;
    z4 = z4 * (-3196) + z5;
    t0 += z1 + z3;
    t1 += z2 + z4;
    t2 += z2 + z3;
    t3 += z1 + z4;
    o[0] = tmp10 + t3;
    o[1] = tmp11 + t2;
    o[2] = tmp12 + t1;
    o[3] = tmp13 + t0;
    o[4] = tmp13 - t0;
    o[5] = tmp12 - t1;
    o[6] = tmp11 - t2;
    o[7] = tmp10 - t3;
}

// one thread per block of a component (blocks enumerated over all tiles by the host)
__global__ void jpeg_idct_kernel(const JpegTile* tiles, const int32_t* blk_tile, const int32_t* blk_comp,
                                 const int32_t* blk_index, int nblk, const int16_t* coef, const uint16_t* qpool,
                                 uint8_t* planes, const int32_t* status) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nblk) return;
    const int t = blk_tile[g];
    if (status[t]) return;
    const JpegComp& cp = tiles[t].comp[blk_comp[g]];
    const int bi = blk_index[g];
    const int by = bi / cp.bw, bx = bi - by * cp.bw;
    const int16_t* in = coef + cp.coef_off + (int64_t)bi * 64;
    const uint16_t* q = qpool + cp.q * 64;
    int ws[64];
    for (int col = 0; col < 8; ++col) {  // pass 1: columns
        int64_t o[8];
        int64_t d[8];
        for (int r = 0; r < 8; ++r) d[r] = (int64_t)in[r * 8 + col] * q[r * 8 + col];
        jbutterfly(d[0], d[1], d[2], d[3], d[4], d[5], d[6], d[7], o);
        for (int r = 0; r < 8; ++r) ws[r * 8 + col] = jdescale(o[r], kCB - kP1);
    }
    uint8_t* out = planes + cp.plane_off + (int64_t)by * 8 * (cp.bw * 8) + bx * 8;
    for (int r = 0; r < 8; ++r) {  // pass 2: rows
        int64_t o[8];
        jbutterfly(ws[r * 8], ws[r * 8 + 1], ws[r * 8 + 2], ws[r * 8 + 3], ws[r * 8 + 4], ws[r * 8 + 5], ws[r * 8 + 6],
                   ws[r * 8 + 7], o);
        for (int c = 0; c < 8; ++c) out[r * cp.bw * 8 + c] = (uint8_t)min(max(jdescale(o[c], kCB + kP1 + 3) + 128, 0), 255);
    }
}

// 2x2 fancy upsampled chroma sample at output (yy, xx) of a plane with cw x ch samples
__device__ __forceinline__ int jchroma(const uint8_t* p, int pitch, int cw, int ch, int yy, int xx, bool sub) {
    if (!sub) return p[yy * pitch + xx];
    const int cy = yy >> 1, cx = xx >> 1;
    if (cw <= 2) return p[cy * pitch + cx];  // libjpeg-turbo: plain replication for narrow chroma
    const int ny = (yy & 1) ? min(cy + 1, ch - 1) : max(cy - 1, 0);
    auto colsum = [&](int x) { return 3 * (int)p[cy * pitch + x] + (int)p[ny * pitch + x]; };
    const int c0 = colsum(cx);
    if (!(xx & 1)) return cx == 0 ? (4 * c0 + 8) >> 4 : (3 * c0 + colsum(cx - 1) + 8) >> 4;
    return cx == cw - 1 ? (4 * c0 + 7) >> 4 : (3 * c0 + colsum(cx + 1) + 7) >> 4;
}

__global__ void jpeg_color_kernel(const JpegTile* tiles, const int64_t* px_off, int n, int64_t total,
                                  const uint8_t* planes, int T, const int32_t* status) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= total) return;
    int lo = 0, hi = n;  // tile of pixel g: px_off is the exclusive prefix sum of h * w
    while (hi - lo > 1) {
        const int m = (lo + hi) >> 1;
        if (px_off[m] <= g) lo = m;
        else hi = m;
    }
    const int t = lo;
    if (status[t]) return;
    const JpegTile& tl = tiles[t];
    const int i = (int)(g - px_off[t]);
    const int yy = i / tl.w, xx = i - yy * tl.w;
    uint8_t* o = reinterpret_cast<uint8_t*>(tl.dst) + ((int64_t)yy * T + xx) * 3;
    const JpegComp& cy = tl.comp[0];
    const int Y = planes[cy.plane_off + (int64_t)yy * cy.bw * 8 + xx];
    if (tl.ncomp == 1) {
        o[0] = o[1] = o[2] = (uint8_t)Y;
        return;
    }
    const JpegComp& cb = tl.comp[1];
    const bool sub = cb.hs * 2 == cy.hs && cb.vs * 2 == cy.vs;
    const int cw = (tl.w + 1) >> 1, chh = (tl.h + 1) >> 1;
    const int Cb = jchroma(planes + cb.plane_off, cb.bw * 8, cw, chh, yy, xx, sub) - 128;
    const int Cr = jchroma(planes + tl.comp[2].plane_off, tl.comp[2].bw * 8, cw, chh, yy, xx, sub) - 128;
    const int r = Y + ((91881 * Cr + 32768) >> 16);  // FIX(1.40200)
    const int bb = Y + ((116130 * Cb + 32768) >> 16);  // FIX(1.77200)
    const int gg = Y + ((-22554 * Cb + 32768 - 46802 * Cr) >> 16);  // FIX(0.34414), FIX(0.71414)
    o[0] = (uint8_t)min(max(r, 0), 255);
    o[1] = (uint8_t)min(max(gg, 0), 255);
    o[2] = (uint8_t)min(max(bb, 0), 255);
}

}  // namespace pf

using namespace pf;

extern "C" int pf_jpeg_decode(const void* tiles_dev, int32_t n, const uint8_t* data_dev, const void* huff_dev,
                              const uint16_t* quant_dev, int16_t* coef_dev, uint8_t* planes_dev,
                              const int32_t* blk_tile_dev, const int32_t* blk_comp_dev, const int32_t* blk_index_dev,
                              int32_t nblk, const int64_t* px_off_dev, int64_t total_px, int32_t tile_size,
                              int32_t* status_dev, void* stream) {
    if (n < 0 || nblk < 0 || total_px < 0 || tile_size < 1 ||
        (n > 0 && (!tiles_dev || !data_dev || !huff_dev || !quant_dev || !coef_dev || !planes_dev || !blk_tile_dev ||
                   !blk_comp_dev || !blk_index_dev || !px_off_dev || !status_dev)))
        return fail(PF_ERR_INVALID_ARG, "pf_jpeg_decode: bad arguments");
    if (n == 0) return PF_OK;
    cudaStream_t st = as_stream(stream);
    const JpegTile* tiles = static_cast<const JpegTile*>(tiles_dev);
    jpeg_entropy_kernel<<<(n + 3) / 4, 128, 0, st>>>(tiles, n, data_dev, static_cast<const JpegHuff*>(huff_dev),
                                                     coef_dev, status_dev);
    int rc = after_launch("jpeg_entropy_kernel");
    if (rc) return rc;
    if (nblk > 0) {
        jpeg_idct_kernel<<<(nblk + 127) / 128, 128, 0, st>>>(tiles, blk_tile_dev, blk_comp_dev, blk_index_dev, nblk,
                                                            coef_dev, quant_dev, planes_dev, status_dev);
        if ((rc = after_launch("jpeg_idct_kernel"))) return rc;
    }
    if (total_px > 0) {
        jpeg_color_kernel<<<(unsigned)((total_px + 255) / 256), 256, 0, st>>>(tiles, px_off_dev, n, total_px,
                                                                              planes_dev, tile_size, status_dev);
        rc = after_launch("jpeg_color_kernel");
    }
    return rc;
}

extern "C" int pf_jpeg_struct_sizes(int32_t* huff, int32_t* tile) {
    if (!huff || !tile) return fail(PF_ERR_INVALID_ARG, "pf_jpeg_struct_sizes: bad arguments");
    *huff = (int32_t)sizeof(JpegHuff);
    *tile = (int32_t)sizeof(JpegTile);
    return PF_OK;
}
