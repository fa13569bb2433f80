// Host preparation of JPEG tiles for the GPU decoder (pf_jpeg.cu): marker parsing
// (ITU-T T.81 B.2: DQT, DHT, SOF0, DRI, SOS), Huffman lookup records, de-duplicated
// table pools, byte-unstuffed entropy segments and the (tile, component, block) list.
// Native so that preparing thousands of tiles costs microseconds each.
#include <stdint.h>
#include <string.h>

#include <map>
#include <string>
#include <vector>

#include "pf_b200.h"
#include "pf_jpeg.h"

namespace pf {
int fail(int status, const std::string& msg);
}

namespace {

using namespace pf;

const uint8_t kZz[64] = {0,  1,  8,  16, 9,  2,  3,  10, 17, 24, 32, 25, 18, 11, 4,  5,  12, 19, 26, 33, 40, 48,
                         41, 34, 27, 20, 13, 6,  7,  14, 21, 28, 35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23,
                         30, 37, 44, 51, 58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63};

JpegHuff make_huff(const uint8_t* counts, const uint8_t* vals) {
    JpegHuff h;
    memset(&h, 0, sizeof h);
    for (int i = 0; i < 18; ++i) h.maxcode[i] = -1;
    int code = 0, k = 0;
    for (int len = 1; len <= 16; ++len) {
        const int c = counts[len - 1];
        if (c) {
            h.valoff[len] = k - code;
            for (int j = 0; j < c; ++j)
                if (len <= 9) {
                    const int lo = (code + j) << (9 - len);
                    for (int f = lo; f < lo + (1 << (9 - len)); ++f) h.fast[f] = (uint16_t)((len << 8) | vals[k + j]);
                }
            h.maxcode[len] = code + c - 1;
        }
        code = (code + c) << 1;
        k += c;
    }
    memcpy(h.huffval, vals, k > 256 ? 256 : k);
    h.maxcode[17] = 0x7fffffff;
    return h;
}

struct Parsed {
    uint16_t q[4][64];
    bool has_q[4] = {false, false, false, false};
    uint8_t hcounts[2][4][16], hvals[2][4][256];
    int hn[2][4] = {{0}};
    bool has_h[2][4] = {{false}};
    int h = 0, w = 0, nc = 0;
    int cid[3], hs[3], vs[3], tq[3], td[3], ta[3];
    const uint8_t* scan = nullptr;
    int64_t scan_len = 0;
};

// 0 ok, 1 unsupported (decode on the host), <0 malformed
int parse(const uint8_t* d, int64_t n, Parsed& P) {
    if (n < 4 || d[0] != 0xFF || d[1] != 0xD8) return -1;
    int64_t pos = 2;
    bool sof = false;
    while (pos + 4 <= n) {
        if (d[pos] != 0xFF) return -1;
        const int m = d[pos + 1];
        pos += 2;
        if (m == 0xD9) break;
        if (m == 0x01 || (m >= 0xD0 && m <= 0xD7)) continue;
        const int ln = (d[pos] << 8) | d[pos + 1];
        if (ln < 2 || pos + ln > n) return -1;
        const uint8_t* seg = d + pos + 2;
        const int sl = ln - 2;
        if (m == 0xDB) {
            for (int i = 0; i < sl;) {
                const int pq = seg[i] >> 4, t = seg[i] & 15;
                if (t > 3 || i + 1 + 64 * (pq ? 2 : 1) > sl) return -1;
                for (int k = 0; k < 64; ++k)
                    P.q[t][kZz[k]] = pq ? (uint16_t)((seg[i + 1 + 2 * k] << 8) | seg[i + 2 + 2 * k]) : seg[i + 1 + k];
                P.has_q[t] = true;
                i += 1 + 64 * (pq ? 2 : 1);
            }
        } else if (m == 0xC4) {
            for (int i = 0; i < sl;) {
                const int tc = seg[i] >> 4, t = seg[i] & 15;
                if (tc > 1 || t > 3 || i + 17 > sl) return -1;
                int k = 0;
                for (int j = 0; j < 16; ++j) k += seg[i + 1 + j];
                if (k > 256 || i + 17 + k > sl) return -1;
                memcpy(P.hcounts[tc][t], seg + i + 1, 16);
                memcpy(P.hvals[tc][t], seg + i + 17, k);
                P.hn[tc][t] = k;
                P.has_h[tc][t] = true;
                i += 17 + k;
            }
        } else if (m == 0xC0) {
            if (sl < 6) return -1;
            P.h = (seg[1] << 8) | seg[2];
            P.w = (seg[3] << 8) | seg[4];
            P.nc = seg[5];
            if (P.nc != 1 && P.nc != 3) return 1;
            if (sl < 6 + 3 * P.nc) return -1;
            for (int k = 0; k < P.nc; ++k) {
                P.cid[k] = seg[6 + 3 * k];
                P.hs[k] = seg[7 + 3 * k] >> 4;
                P.vs[k] = seg[7 + 3 * k] & 15;
                P.tq[k] = seg[8 + 3 * k] & 3;
            }
            sof = true;
        } else if (m >= 0xC1 && m <= 0xCF && m != 0xC4 && m != 0xC8 && m != 0xCC) {
            return 1;  // progressive / lossless / arithmetic
        } else if (m == 0xDD) {
            if (sl >= 2 && ((seg[0] << 8) | seg[1])) return 1;  // restart intervals
        } else if (m == 0xDA) {
            if (!sof || sl < 1) return -1;
            const int ns = seg[0];
            if (ns != P.nc || sl < 1 + 2 * ns) return 1;
            for (int k = 0; k < ns; ++k) {
                int c = -1;
                for (int j = 0; j < P.nc; ++j)
                    if (P.cid[j] == seg[1 + 2 * k]) c = j;
                if (c < 0) return -1;
                P.td[c] = seg[2 + 2 * k] >> 4;
                P.ta[c] = seg[2 + 2 * k] & 15;
            }
            P.scan = d + pos + ln;
            P.scan_len = n - (pos + ln);
            return 0;
        }
        pos += ln;
    }
    return -1;
}

}  // namespace

// tiles_in: n files at bytes[off[t] .. off[t+1]); dims (w, h) expected per tile; dst pointers.
// Outputs (caller-allocated, bounds from the sizes below): tiles_out[n] JpegTile, ok_out[n]
// (0 decoded on the GPU, 1 unsupported -> host), data_out (<= total input bytes), huff_out
// (<= 4 n tables), quant_out (<= 4 n * 64), blk_{tile,comp,index}_out (<= sum ceil(w/8)
// ceil(h/8) * 3), px_off_out[n] (pixels before tile t); counts_out = {n_huff, n_quant,
// n_blocks, data_bytes, coef_total, plane_total, total_px}.
extern "C" int pf_jpeg_prepare(const uint8_t* bytes, const int64_t* off, const int32_t* tw, const int32_t* th,
                               const uint64_t* dst, int32_t n, void* tiles_out, int32_t* ok_out, uint8_t* data_out,
                               void* huff_out, uint16_t* quant_out, int32_t* blk_tile_out, int32_t* blk_comp_out,
                               int32_t* blk_index_out, int64_t* px_off_out, int64_t* counts_out) {
    if (n < 0 || (n > 0 && (!bytes || !off || !tw || !th || !dst || !tiles_out || !ok_out || !data_out || !huff_out ||
                            !quant_out || !blk_tile_out || !blk_comp_out || !blk_index_out || !px_off_out)) ||
        !counts_out)
        return fail(PF_ERR_INVALID_ARG, "pf_jpeg_prepare: bad arguments");
    JpegTile* tiles = static_cast<JpegTile*>(tiles_out);
    JpegHuff* huff = static_cast<JpegHuff*>(huff_out);
    std::map<std::string, int> hmap, qmap;
    int64_t nh = 0, nq = 0, nblk = 0, data = 0, coef = 0, plane = 0, px = 0;
    for (int t = 0; t < n; ++t) {
        memset(&tiles[t], 0, sizeof(JpegTile));
        px_off_out[t] = px;
        Parsed P;
        const int rc = parse(bytes + off[t], off[t + 1] - off[t], P);
        if (rc < 0) return fail(PF_ERR_DECODE, "pf_jpeg_prepare: malformed JPEG tile " + std::to_string(t));
        bool ok = rc == 0 && P.w == tw[t] && P.h == th[t];
        if (ok && P.nc == 3)
            ok = P.hs[1] == 1 && P.vs[1] == 1 && P.hs[2] == 1 && P.vs[2] == 1 &&
                 ((P.hs[0] == 1 && P.vs[0] == 1) || (P.hs[0] == 2 && P.vs[0] == 2));
        for (int c = 0; ok && c < P.nc; ++c)
            ok = P.has_q[P.tq[c]] && P.td[c] < 4 && P.ta[c] < 4 && P.has_h[0][P.td[c]] && P.has_h[1][P.ta[c]];
        ok_out[t] = ok ? 0 : 1;
        if (!ok) continue;
        JpegTile& T = tiles[t];
        int hmax = 1, vmax = 1;
        for (int c = 0; c < P.nc; ++c) {
            hmax = P.hs[c] > hmax ? P.hs[c] : hmax;
            vmax = P.vs[c] > vmax ? P.vs[c] : vmax;
        }
        T.h = P.h;
        T.w = P.w;
        T.ncomp = P.nc;
        T.mcux = (P.w + 8 * hmax - 1) / (8 * hmax);
        T.mcuy = (P.h + 8 * vmax - 1) / (8 * vmax);
        T.dst = dst[t];
        // unstuff the entropy-coded segment up to the first non-stuffing marker
        T.data_off = data;
        for (int64_t i = 0; i < P.scan_len; ++i) {
            const uint8_t b = P.scan[i];
            if (b == 0xFF) {
                if (i + 1 < P.scan_len && P.scan[i + 1] == 0x00) {
                    data_out[data++] = 0xFF;
                    ++i;
                    continue;
                }
                break;
            }
            data_out[data++] = b;
        }
        T.data_len = (int32_t)(data - T.data_off);
        for (int c = 0; c < P.nc; ++c) {
            JpegComp& C = T.comp[c];
            C.hs = P.hs[c];
            C.vs = P.vs[c];
            const std::string qk(reinterpret_cast<const char*>(P.q[P.tq[c]]), 128);
            auto qi = qmap.find(qk);
            if (qi == qmap.end()) {
                memcpy(quant_out + 64 * nq, P.q[P.tq[c]], 128);
                qi = qmap.emplace(qk, (int)nq++).first;
            }
            C.q = qi->second;
            for (int tc = 0; tc < 2; ++tc) {
                const int id = tc ? P.ta[c] : P.td[c];
                std::string hk(1, (char)tc);
                hk.append(reinterpret_cast<const char*>(P.hcounts[tc][id]), 16);
                hk.append(reinterpret_cast<const char*>(P.hvals[tc][id]), P.hn[tc][id]);
                auto hi = hmap.find(hk);
                if (hi == hmap.end()) {
                    huff[nh] = make_huff(P.hcounts[tc][id], P.hvals[tc][id]);
                    hi = hmap.emplace(hk, (int)nh++).first;
                }
                (tc ? C.ac : C.dc) = hi->second;
            }
            C.bw = T.mcux * C.hs;
            C.bh = T.mcuy * C.vs;
            const int nb = C.bw * C.bh;
            C.coef_off = coef;
            C.plane_off = plane;
            coef += 64LL * nb;
            plane += 64LL * nb;
            for (int b = 0; b < nb; ++b) {
                blk_tile_out[nblk] = t;
                blk_comp_out[nblk] = c;
                blk_index_out[nblk] = b;
                ++nblk;
            }
        }
        px += (int64_t)P.h * P.w;
    }
    const int64_t counts[7] = {nh, nq, nblk, data, coef, plane, px};
    memcpy(counts_out, counts, sizeof counts);
    return PF_OK;
}
