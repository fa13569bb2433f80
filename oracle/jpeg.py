"""Baseline JPEG decode restated (TEST INFRASTRUCTURE ONLY): the checker for the GPU JPEG tile
decoder (csrc/pf_jpeg.cu), itself pinned to Pillow's decoder (tests/test_jpeg_oracle.py).

The reference decodes JPEG tiles with Pillow (decode_tile, pkg/store.py:397-416; JPEG q90 is
an ingest codec option, pkg/store.py:416-426).  Pillow links libjpeg-turbo, whose default
decompression path is restated here from the published algorithms: ITU-T T.81 baseline
Huffman decoding; the accurate integer inverse DCT of the IJG library (jidctint, "islow":
13-bit constants, two passes, PASS1_BITS = 2); "fancy" triangle-filter upsampling of 2x2
subsampled chroma (box replication when the chroma is at most 2 samples wide, as
libjpeg-turbo does); and the fixed-point YCbCr -> RGB tables (16-bit scale).
"""

from __future__ import annotations

import numpy as np

ZIGZAG = np.array([0, 1, 8, 16, 9, 2, 3, 10, 17, 24, 32, 25, 18, 11, 4, 5, 12, 19, 26, 33, 40, 48, 41, 34, 27, 20, 13, 6,
                   7, 14, 21, 28, 35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51, 58, 59, 52, 45, 38,
                   31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63])


class JpegError(ValueError):
    pass


def parse(data: bytes) -> dict:
    """Markers of a baseline JPEG: quant tables (natural order), Huffman tables, frame, scan."""
    if data[:2] != b"\xff\xd8":
        raise JpegError("no SOI")
    pos, q, huff, frame, scan = 2, {}, {}, None, None
    while pos < len(data):
        if data[pos] != 0xFF:
            raise JpegError("marker expected")
        m = data[pos + 1]
        pos += 2
        if m == 0xD9:
            break
        if m in (0x01,) or 0xD0 <= m <= 0xD7:
            continue
        ln = int.from_bytes(data[pos:pos + 2], "big")
        seg = data[pos + 2:pos + ln]
        if m == 0xDB:  # DQT
            i = 0
            while i < len(seg):
                pq, tq = seg[i] >> 4, seg[i] & 15
                n = 64 * (2 if pq else 1)
                vals = np.frombuffer(seg[i + 1:i + 1 + n], dtype=">u2" if pq else np.uint8).astype(np.int64)
                nat = np.zeros(64, np.int64)
                nat[ZIGZAG] = vals
                q[tq] = nat
                i += 1 + n
        elif m == 0xC4:  # DHT
            i = 0
            while i < len(seg):
                tc, th = seg[i] >> 4, seg[i] & 15
                counts = list(seg[i + 1:i + 17])
                n = sum(counts)
                huff[(tc, th)] = (counts, list(seg[i + 17:i + 17 + n]))
                i += 17 + n
        elif m == 0xC0:  # SOF0 baseline
            h, w, nc = int.from_bytes(seg[1:3], "big"), int.from_bytes(seg[3:5], "big"), seg[5]
            comps = [(seg[6 + 3 * k], seg[7 + 3 * k] >> 4, seg[7 + 3 * k] & 15, seg[8 + 3 * k]) for k in range(nc)]
            frame = {"h": h, "w": w, "comps": comps}
        elif m in (0xC1, 0xC2, 0xC3, 0xC5, 0xC6, 0xC7, 0xC9, 0xCA, 0xCB, 0xCD, 0xCE, 0xCF):
            raise JpegError("only baseline sequential JPEG")
        elif m == 0xDD:
            if int.from_bytes(seg[0:2], "big"):
                raise JpegError("restart intervals unsupported")
        elif m == 0xDA:  # SOS: entropy-coded data runs to the next non-RST marker
            ns = seg[0]
            sel = [(seg[1 + 2 * k], seg[2 + 2 * k] >> 4, seg[2 + 2 * k] & 15) for k in range(ns)]
            start = pos + ln
            end = start
            while end + 1 < len(data) and not (data[end] == 0xFF and data[end + 1] not in (0x00,) and not
                                                (0xD0 <= data[end + 1] <= 0xD7)):
                end += 1
            scan = {"sel": sel, "data": data[start:end]}
            pos = end
            continue
        pos += ln
    if frame is None or scan is None:
        raise JpegError("no frame / scan")
    return {"q": q, "huff": huff, "frame": frame, "scan": scan}


class _Bits:
    def __init__(self, data: bytes):
        self.d = data.replace(b"\xff\x00", b"\xff")
        self.pos = 0  # bit position

    def bit(self) -> int:
        byte = self.pos >> 3
        if byte >= len(self.d):
            return 1  # libjpeg pads with ones past the end of data
        v = (self.d[byte] >> (7 - (self.pos & 7))) & 1
        self.pos += 1
        return v

    def bits(self, n: int) -> int:
        v = 0
        for _ in range(n):
            v = (v << 1) | self.bit()
        return v


def _huff_lookup(counts, symbols):
    """code -> symbol per length (canonical codes, T.81 Annex C)."""
    table, code, k = {}, 0, 0
    for length in range(1, 17):
        for _ in range(counts[length - 1]):
            table[(length, code)] = symbols[k]
            code += 1
            k += 1
        code <<= 1
    return table


def _decode(b: _Bits, table) -> int:
    code = 0
    for length in range(1, 17):
        code = (code << 1) | b.bit()
        s = table.get((length, code))
        if s is not None:
            return s
    raise JpegError("bad Huffman code")


def _extend(v: int, s: int) -> int:
    return v - (1 << s) + 1 if s and v < (1 << (s - 1)) else v


def coefficients(j: dict):
    """Entropy-decode all blocks -> per component an int array [by, bx, 64] (natural order)."""
    fr = j["frame"]
    comps = fr["comps"]
    hmax, vmax = max(c[1] for c in comps), max(c[2] for c in comps)
    mcux, mcuy = -(-fr["w"] // (8 * hmax)), -(-fr["h"] // (8 * vmax))
    tabs = {k: _huff_lookup(*v) for k, v in j["huff"].items()}
    sel = {cid: (td, ta) for cid, td, ta in j["scan"]["sel"]}
    out = [np.zeros((mcuy * c[2], mcux * c[1], 64), np.int64) for c in comps]
    pred = [0] * len(comps)
    b = _Bits(j["scan"]["data"])
    for my in range(mcuy):
        for mx in range(mcux):
            for ci, (cid, hs, vs, tq) in enumerate(comps):
                td, ta = sel[cid]
                for v in range(vs):
                    for h in range(hs):
                        blk = np.zeros(64, np.int64)
                        s = _decode(b, tabs[(0, td)])
                        pred[ci] += _extend(b.bits(s), s)
                        blk[0] = pred[ci]
                        k = 1
                        while k < 64:
                            rs = _decode(b, tabs[(1, ta)])
                            r, s = rs >> 4, rs & 15
                            if s == 0:
                                if r == 15:
                                    k += 16
                                    continue
                                break
                            k += r
                            if k > 63:
                                raise JpegError("AC index past 63")
                            blk[ZIGZAG[k]] = _extend(b.bits(s), s)
                            k += 1
                        out[ci][my * vs + v, mx * hs + h] = blk
    return out


CONST_BITS, PASS1_BITS = 13, 2
F = {"0_298631336": 2446, "0_390180644": 3196, "0_541196100": 4433, "0_765366865": 6270, "0_899976223": 7373,
     "1_175875602": 9633, "1_501321110": 12299, "1_847759065": 15137, "1_961570560": 16069, "2_053119869": 16819,
     "2_562915447": 20995, "3_072711026": 25172}


def _descale(x, n):
    return (x + (1 << (n - 1))) >> n


def _butterfly(i0, i1, i2, i3, i4, i5, i6, i7):
    z2, z3 = i2, i6
    z1 = (z2 + z3) * F["0_541196100"]
    tmp2 = z1 + z3 * (-F["1_847759065"])
    tmp3 = z1 + z2 * F["0_765366865"]
    tmp0 = (i0 + i4) << CONST_BITS
    tmp1 = (i0 - i4) << CONST_BITS
    tmp10, tmp13, tmp11, tmp12 = tmp0 + tmp3, tmp0 - tmp3, tmp1 + tmp2, tmp1 - tmp2
    t0, t1, t2, t3 = i7, i5, i3, i1
    z1, z2, z3, z4 = t0 + t3, t1 + t2, t0 + t2, t1 + t3
    z5 = (z3 + z4) * F["1_175875602"]
    t0, t1, t2, t3 = t0 * F["0_298631336"], t1 * F["2_053119869"], t2 * F["3_072711026"], t3 * F["1_501321110"]
    z1, z2 = z1 * (-F["0_899976223"]), z2 * (-F["2_562915447"])
    z3, z4 = z3 * (-F["1_961570560"]) + z5, z4 * (-F["0_390180644"]) + z5
    t0, t1, t2, t3 = t0 + z1 + z3, t1 + z2 + z4, t2 + z2 + z3, t3 + z1 + z4
    return (tmp10 + t3, tmp11 + t2, tmp12 + t1, tmp13 + t0, tmp13 - t0, tmp12 - t1, tmp11 - t2, tmp10 - t3)


def idct_islow(coef: np.ndarray, q: np.ndarray) -> np.ndarray:
    """[..., 64] natural-order coefficients x quant -> [..., 8, 8] uint8 (vectorised over blocks)."""
    d = (coef * q).reshape(coef.shape[:-1] + (8, 8))  # [.., row(v), col(u)]
    cols = _butterfly(*[d[..., k, :] for k in range(8)])  # pass 1 down the columns
    ws = np.stack([_descale(c, CONST_BITS - PASS1_BITS) for c in cols], -2)  # [.., 8 rows, 8 cols]
    rows = _butterfly(*[ws[..., :, k] for k in range(8)])  # pass 2 along the rows
    out = np.stack([_descale(r, CONST_BITS + PASS1_BITS + 3) for r in rows], -1) + 128
    return np.clip(out, 0, 255).astype(np.uint8)


def _plane(blocks: np.ndarray, q: np.ndarray) -> np.ndarray:
    by, bx = blocks.shape[:2]
    px = idct_islow(blocks, q)  # [by, bx, 8, 8]
    return px.transpose(0, 2, 1, 3).reshape(by * 8, bx * 8)


def fancy_h2v2(c: np.ndarray, h: int, w: int) -> np.ndarray:
    """2x2 triangle-filter upsampling of a chroma plane covering (ceil(h/2), ceil(w/2)) samples."""
    cw, ch = -(-w // 2), -(-h // 2)
    a = c[:ch, :cw].astype(np.int64)
    if cw <= 2:  # libjpeg-turbo skips fancy upsampling for chroma at most 2 samples wide: replicate
        return np.repeat(np.repeat(a, 2, 0), 2, 1)[:h, :w]
    up = np.vstack([a[:1], a[:-1]])  # row above (replicated at the top)
    dn = np.vstack([a[1:], a[-1:]])  # row below (replicated at the bottom)
    out = np.zeros((2 * ch, 2 * cw), np.int64)
    for half, nb in ((0, up), (1, dn)):
        col = a * 3 + nb  # vertical pass: 3 * nearer + farther
        left = np.hstack([col[:, :1], col[:, :-1]])
        right = np.hstack([col[:, 1:], col[:, -1:]])
        ev = (col * 3 + left + 8) >> 4
        od = (col * 3 + right + 7) >> 4
        ev[:, 0] = (col[:, 0] * 4 + 8) >> 4
        od[:, -1] = (col[:, -1] * 4 + 7) >> 4
        out[half::2, 0::2] = ev
        out[half::2, 1::2] = od
    return out[:h, :w]


def ycc_to_rgb(y, cb, cr) -> np.ndarray:
    scale, half = 16, 1 << 15

    def fix(x):
        return int(x * (1 << scale) + 0.5)

    cb = cb.astype(np.int64) - 128
    cr = cr.astype(np.int64) - 128
    r = y + ((fix(1.40200) * cr + half) >> scale)
    b = y + ((fix(1.77200) * cb + half) >> scale)
    g = y + ((-fix(0.34414) * cb + half - fix(0.71414) * cr) >> scale)
    return np.clip(np.stack([r, g, b], -1), 0, 255).astype(np.uint8)


def decode(data: bytes) -> np.ndarray:
    """Baseline JPEG (grayscale or YCbCr with 1x1 / 2x1 / 2x2 luma sampling) -> (h, w, 3) uint8."""
    j = parse(data)
    fr = j["frame"]
    h, w, comps = fr["h"], fr["w"], fr["comps"]
    blocks = coefficients(j)
    planes = [_plane(b, j["q"][c[3]]) for b, c in zip(blocks, comps)]
    if len(comps) == 1:
        y = planes[0][:h, :w]
        return np.repeat(y[..., None], 3, -1)
    (_, hy, vy, _), (_, hc, vc, _) = comps[0], comps[1]
    y = planes[0][:h, :w].astype(np.int64)
    if (hy, vy) == (hc, vc):
        cb, cr = planes[1][:h, :w], planes[2][:h, :w]
    elif (hy // hc, vy // vc) == (2, 2):
        cb, cr = fancy_h2v2(planes[1], h, w), fancy_h2v2(planes[2], h, w)
    else:
        raise JpegError(f"unsupported sampling {hy}x{vy}/{hc}x{vc}")
    return ycc_to_rgb(y, cb, cr)
