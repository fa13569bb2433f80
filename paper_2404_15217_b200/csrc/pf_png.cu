// On-GPU PNG tile decode (replaces decode_tile's Pillow
// path, pkg/store.py:397-416, for the store's default codec, pkg/store.py:470).
//
// Stage 1 (pf_png_inflate): one warp per tile (lane 0) inflates its zlib stream
// (RFC 1950/1951: stored, fixed and dynamic Huffman blocks, LZ77 copies) into
// the tile's filtered scanlines in device scratch.  Canonical-Huffman decoding
// looks codes of up to 9 bits up in a table and walks longer ones bit by bit
// against count/symbol arrays (the compact canonical scheme of zlib's reference
// decoder "puff"), so a tile's tables fit in 2.5 KB of shared memory.
// Stage 2 (pf_png_unfilter): three threads per tile (one per RGB channel: the
// PNG filters only reference the same channel of the left / upper pixels)
// undo the per-row filters (None, Sub, Up, Average, Paeth) straight into the
// tile's slot of the HBM pyramid.  PNG is lossless, so the result is the
// bytes Pillow decodes; streams that do not parse set a per-tile status.
#include <stdint.h>

#include "pf_common.cuh"

namespace pf {

constexpr int kPngWarps = 4;  // tiles per inflate block: one warp per tile (lane 0 decodes; per-thread
                              // decoders in one warp diverge and hit 32-way bank conflicts)
constexpr int kMaxLit = 288, kMaxDist = 30;

constexpr int kFastBits = 9;  // codes up to 9 bits decode with one table lookup
struct Huff {
    uint16_t count[16];
    uint16_t symbol[kMaxLit];
    uint16_t fast[1 << kFastBits];  // (len << 9) | symbol, indexed by the next 9 stream bits; 0: longer code
};
struct HuffD {
    uint16_t count[16];
    uint16_t symbol[kMaxDist + 2];
    uint16_t fast[1 << kFastBits];
};

struct BitIn {
    const uint8_t* in;
    int64_t n, pos;
    uint32_t buf;
    int cnt;
    int err;
};

__device__ __forceinline__ uint32_t getbits(BitIn& s, int need) {
    uint32_t v = s.buf;
    while (s.cnt < need) {
        if (s.pos >= s.n) {
            s.err = 1;
            return 0;
        }
        v |= (uint32_t)s.in[s.pos++] << s.cnt;
        s.cnt += 8;
    }
    s.buf = v >> need;
    s.cnt -= need;
    return v & ((1u << need) - 1u);
}

// canonical code construction; returns 0 if complete or incomplete-but-usable, <0 if over-subscribed
template <typename H>
__device__ int construct(H& h, const uint8_t* length, int n) {
    for (int len = 0; len < 16; ++len) h.count[len] = 0;
    for (int s = 0; s < n; ++s) h.count[length[s]]++;
    if (h.count[0] == n) return 0;
    int left = 1;
    for (int len = 1; len < 16; ++len) {
        left <<= 1;
        left -= h.count[len];
        if (left < 0) return left;
    }
    uint16_t offs[16];
    offs[1] = 0;
    for (int len = 1; len < 15; ++len) offs[len + 1] = offs[len] + h.count[len];
    for (int s = 0; s < n; ++s)
        if (length[s] != 0) h.symbol[offs[length[s]]++] = (uint16_t)s;
    // fast table: canonical codes of length <= 9, stored bit-reversed (the stream sends a
    // code's most significant bit first)
    for (int i = 0; i < (1 << kFastBits); ++i) h.fast[i] = 0;
    int code = 0, idx = 0;
    for (int len = 1; len <= kFastBits; ++len) {
        for (int k = 0; k < h.count[len]; ++k, ++code, ++idx) {
            const int rev = (int)(__brev((unsigned)code) >> (32 - len));
            for (int f = rev; f < (1 << kFastBits); f += 1 << len)
                h.fast[f] = (uint16_t)((len << 9) | h.symbol[idx]);
        }
        code <<= 1;
    }
    return left;
}

// One symbol: a 9-bit table lookup, or (longer codes / stream tail) the canonical walk bit
// by bit against the per-length counts.
template <typename H>
__device__ __forceinline__ int decode_sym(BitIn& s, const H& h) {
    while (s.cnt < kFastBits && s.pos < s.n) {
        s.buf |= (uint32_t)s.in[s.pos++] << s.cnt;
        s.cnt += 8;
    }
    const int e = h.fast[s.buf & ((1u << kFastBits) - 1u)];
    const int elen = e >> 9;
    if (e && elen <= s.cnt) {
        s.buf >>= elen;
        s.cnt -= elen;
        return e & 511;
    }
    int code = 0, first = 0, index = 0;
    for (int len = 1; len < 16; ++len) {
        if (s.cnt == 0) {
            if (s.pos >= s.n) {
                s.err = 1;
                return -1;
            }
            s.buf = s.in[s.pos++];
            s.cnt = 8;
        }
        code |= (int)(s.buf & 1u);
        s.buf >>= 1;
        s.cnt--;
        const int count = h.count[len];
        if (code - count < first) return h.symbol[index + (code - first)];
        index += count;
        first += count;
        first <<= 1;
        code <<= 1;
    }
    return -10;  // ran out of codes
}

__constant__ uint16_t kLenBase[29] = {3,  4,  5,  6,  7,  8,  9,  10, 11,  13,  15,  17,  19,  23, 27,
                                      31, 35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t kLenExtra[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t kDistBase[30] = {1,   2,   3,   4,   5,   7,    9,    13,   17,   25,   33,   49,   65,    97,    129,
                                       193, 257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t kDistExtra[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

// Huffman-coded block body: literals and LZ77 copies until end-of-block
__device__ int codes(BitIn& s, uint8_t* out, int64_t& olen, int64_t omax, const Huff& lc, const HuffD& dc) {
    while (true) {
        int sym = decode_sym(s, lc);
        if (sym < 0) return sym;
        if (sym < 256) {
            if (olen >= omax) return -2;
            out[olen++] = (uint8_t)sym;
        } else if (sym == 256) {
            return 0;
        } else {
            sym -= 257;
            if (sym >= 29) return -10;
            const int len = kLenBase[sym] + (int)getbits(s, kLenExtra[sym]);
            const int ds = decode_sym(s, dc);
            if (ds < 0) return ds;
            if (ds >= 30) return -11;
            const int64_t dist = kDistBase[ds] + (int64_t)getbits(s, kDistExtra[ds]);
            if (s.err) return -1;
            if (dist > olen) return -11;
            if (olen + len > omax) return -2;
            const uint8_t* src = out + olen - dist;
            for (int i = 0; i < len; ++i) out[olen + i] = src[i];
            olen += len;
        }
    }
}

struct PngTables {
    Huff lc;
    HuffD dc;
    uint8_t lengths[320];
};

// one warp per tile: zlib stream zin[zoff[t] .. zoff[t+1]) -> raw[roff[t] .. roff[t] + rlen[t])
__global__ void png_inflate_kernel(const uint8_t* zin, const int64_t* zoff, int n, uint8_t* raw, const int64_t* roff,
                                   const int64_t* rlen, int32_t* status) {
    __shared__ PngTables tabs[kPngWarps];
    const int t = blockIdx.x * kPngWarps + (threadIdx.x >> 5);
    if (t >= n || (threadIdx.x & 31)) return;
    PngTables& T = tabs[threadIdx.x >> 5];
    BitIn s;
    s.in = zin + zoff[t];
    s.n = zoff[t + 1] - zoff[t];
    s.pos = 0;
    s.buf = 0;
    s.cnt = 0;
    s.err = 0;
    uint8_t* out = raw + roff[t];
    const int64_t omax = rlen[t];
    int64_t olen = 0;
    int rc = 0;
    // zlib header (RFC 1950): CM 8, no preset dictionary, FCHECK
    if (s.n < 6) rc = -20;
    else {
        const int cmf = s.in[0], flg = s.in[1];
        if ((cmf & 15) != 8 || (cmf >> 4) > 7 || (flg & 32) || ((cmf << 8) | flg) % 31) rc = -20;
        s.pos = 2;
    }
    int last = 0;
    while (!rc && !last) {
        last = (int)getbits(s, 1);
        const int type = (int)getbits(s, 2);
        if (s.err) {
            rc = -1;
            break;
        }
        if (type == 0) {  // stored: back to the byte boundary, returning whole buffered bytes
            s.pos -= s.cnt >> 3;
            s.buf = 0;
            s.cnt = 0;
            if (s.pos + 4 > s.n) {
                rc = -1;
                break;
            }
            const int len = s.in[s.pos] | (s.in[s.pos + 1] << 8);
            const int nlen = s.in[s.pos + 2] | (s.in[s.pos + 3] << 8);
            s.pos += 4;
            if (len != (~nlen & 0xffff)) {
                rc = -21;
                break;
            }
            if (s.pos + len > s.n) {
                rc = -1;
                break;
            }
            if (olen + len > omax) {
                rc = -2;
                break;
            }
            for (int i = 0; i < len; ++i) out[olen + i] = s.in[s.pos + i];
            olen += len;
            s.pos += len;
        } else if (type == 1) {  // fixed Huffman
            int sym = 0;
            for (; sym < 144; ++sym) T.lengths[sym] = 8;
            for (; sym < 256; ++sym) T.lengths[sym] = 9;
            for (; sym < 280; ++sym) T.lengths[sym] = 7;
            for (; sym < 288; ++sym) T.lengths[sym] = 8;
            construct(T.lc, T.lengths, 288);
            for (sym = 0; sym < 30; ++sym) T.lengths[sym] = 5;
            construct(T.dc, T.lengths, 30);
            rc = codes(s, out, olen, omax, T.lc, T.dc);
        } else if (type == 2) {  // dynamic Huffman
            const int nlen = (int)getbits(s, 5) + 257, ndist = (int)getbits(s, 5) + 1, ncode = (int)getbits(s, 4) + 4;
            if (s.err || nlen > 286 || ndist > 30) {
                rc = -3;
                break;
            }
            const uint8_t order[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};
            for (int i = 0; i < 19; ++i) T.lengths[order[i]] = i < ncode ? (uint8_t)getbits(s, 3) : 0;
            if (s.err || construct(T.lc, T.lengths, 19) != 0) {
                rc = -4;
                break;
            }
            int idx = 0;
            while (idx < nlen + ndist) {
                int sym = decode_sym(s, T.lc);
                if (sym < 0) {
                    rc = sym;
                    break;
                }
                if (sym < 16) {
                    T.lengths[idx++] = (uint8_t)sym;
                } else {
                    int len = 0, rep;
                    if (sym == 16) {
                        if (idx == 0) {
                            rc = -5;
                            break;
                        }
                        len = T.lengths[idx - 1];
                        rep = 3 + (int)getbits(s, 2);
                    } else if (sym == 17) {
                        rep = 3 + (int)getbits(s, 3);
                    } else {
                        rep = 11 + (int)getbits(s, 7);
                    }
                    if (idx + rep > nlen + ndist) {
                        rc = -6;
                        break;
                    }
                    while (rep--) T.lengths[idx++] = (uint8_t)len;
                }
            }
            if (rc) break;
            if (T.lengths[256] == 0) {
                rc = -9;
                break;
            }
            if (construct(T.lc, T.lengths, nlen) < 0 || construct(T.dc, T.lengths + nlen, ndist) < 0) {
                rc = -7;
                break;
            }
            rc = codes(s, out, olen, omax, T.lc, T.dc);
        } else {
            rc = -22;
        }
        if (s.err && !rc) rc = -1;
    }
    if (!rc && olen != omax) rc = -23;  // the image data must fill the scanlines exactly
    status[t] = rc;
}

__device__ __forceinline__ int paeth(int a, int b, int c) {
    const int p = a + b - c;
    const int pa = abs(p - a), pb = abs(p - b), pc = abs(p - c);
    return (pa <= pb && pa <= pc) ? a : (pb <= pc ? b : c);
}

// three threads per tile (channel c): undo the row filters into the tile slot (pitch T * 3);
// the previous row of the channel stays in shared memory (no reload of just-written output)
constexpr int kUnfThreads = 96, kUnfMaxW = 256;
__global__ void png_unfilter_kernel(const uint8_t* raw, const int64_t* roff, const int32_t* tw_, const int32_t* th_,
                                    uint8_t* const* dst, int T, int n, int32_t* status) {
    __shared__ uint8_t prev_rows[kUnfMaxW][kUnfThreads];  // [x][thread]: lockstep lanes hit distinct banks
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = g / 3, c = g - 3 * (g / 3);
    if (t >= n || status[t] != 0) return;
    const int tw = tw_[t], th = th_[t];
    if (tw > kUnfMaxW) {
        if (c == 0) status[t] = -31;
        return;
    }
    uint8_t* prev = &prev_rows[0][threadIdx.x];  // element x at prev[x * kUnfThreads]
    for (int x = 0; x < tw; ++x) prev[x * kUnfThreads] = 0;
    const uint8_t* in = raw + roff[t];
    uint8_t* out = dst[t];
    const int stride = 1 + 3 * tw;
    for (int r = 0; r < th; ++r) {
        const int ft = in[(int64_t)r * stride];
        if (ft > 4) {
            if (c == 0) status[t] = -30;
            return;
        }
        const uint8_t* line = in + (int64_t)r * stride + 1 + c;
        uint8_t* o = out + (int64_t)r * T * 3 + c;
        int left = 0, upleft = 0;
        for (int x = 0; x < tw; ++x) {
            const int b = prev[x * kUnfThreads];
            int v = line[3 * x];
            switch (ft) {
                case 1: v += left; break;
                case 2: v += b; break;
                case 3: v += (left + b) >> 1; break;
                case 4: v += paeth(left, b, upleft); break;
                default: break;
            }
            v &= 255;
            o[3 * x] = (uint8_t)v;
            prev[x * kUnfThreads] = (uint8_t)v;
            left = v;
            upleft = b;
        }
    }
}

}  // namespace pf

using namespace pf;

extern "C" int pf_png_inflate(const uint8_t* zdata_dev, const int64_t* zoff_dev, int32_t n, uint8_t* raw_dev,
                              const int64_t* roff_dev, const int64_t* rlen_dev, int32_t* status_dev, void* stream) {
    if (n < 0 || (n > 0 && (!zdata_dev || !zoff_dev || !raw_dev || !roff_dev || !rlen_dev || !status_dev)))
        return fail(PF_ERR_INVALID_ARG, "pf_png_inflate: bad arguments");
    if (n == 0) return PF_OK;
    png_inflate_kernel<<<(n + kPngWarps - 1) / kPngWarps, 32 * kPngWarps, 0, as_stream(stream)>>>(
        zdata_dev, zoff_dev, n, raw_dev, roff_dev, rlen_dev, status_dev);
    return after_launch("png_inflate_kernel");
}

extern "C" int pf_png_unfilter(const uint8_t* raw_dev, const int64_t* roff_dev, const int32_t* tile_w_dev,
                               const int32_t* tile_h_dev, uint8_t* const* dst_dev, int32_t tile_size, int32_t n,
                               int32_t* status_dev, void* stream) {
    if (n < 0 || tile_size < 1 ||
        (n > 0 && (!raw_dev || !roff_dev || !tile_w_dev || !tile_h_dev || !dst_dev || !status_dev)))
        return fail(PF_ERR_INVALID_ARG, "pf_png_unfilter: bad arguments");
    if (n == 0) return PF_OK;
    png_unfilter_kernel<<<(3 * n + kUnfThreads - 1) / kUnfThreads, kUnfThreads, 0, as_stream(stream)>>>(
        raw_dev, roff_dev, tile_w_dev, tile_h_dev, dst_dev, tile_size, n, status_dev);
    return after_launch("png_unfilter_kernel");
}
