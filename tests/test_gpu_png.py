"""GPU PNG tile decode (pf_png_inflate / pf_png_unfilter) against the image that was encoded:
every PNG row filter, stored / fixed / dynamic DEFLATE blocks (zlib levels 0, 1, 6, 9 and
Pillow's own writer), edge-sized tiles, and corrupt streams."""

import io
import struct
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _paeth(a, b, c):
    p = a + b - c
    pa, pb, pc = abs(p - a), abs(p - b), abs(p - c)
    return a if (pa <= pb and pa <= pc) else (b if pb <= pc else c)


def _filter_rows(img, filters):
    """PNG scanlines of an RGB image with the given per-row filter types."""
    h, w, _ = img.shape
    a = img.astype(np.int64).reshape(h, w * 3)
    out = bytearray()
    for r in range(h):
        ft = int(filters[r])
        prev = a[r - 1] if r else np.zeros(w * 3, np.int64)
        cur = a[r]
        left = np.concatenate([np.zeros(3, np.int64), cur[:-3]])
        ul = np.concatenate([np.zeros(3, np.int64), prev[:-3]])
        if ft == 0:
            f = cur
        elif ft == 1:
            f = cur - left
        elif ft == 2:
            f = cur - prev
        elif ft == 3:
            f = cur - (left + prev) // 2
        else:
            f = cur - np.array([_paeth(x, y, z) for x, y, z in zip(left, prev, ul)])
        out.append(ft)
        out += bytes((f & 255).astype(np.uint8))
    return bytes(out)


def _png(img, filters, level):
    h, w, _ = img.shape

    def chunk(t, b):
        return struct.pack(">I", len(b)) + t + b + struct.pack(">I", zlib.crc32(t + b))

    return (b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, 2, 0, 0, 0))
            + chunk(b"IDAT", zlib.compress(_filter_rows(img, filters), level)) + chunk(b"IEND", b""))


def _decode(tiles, T):
    """tiles: list of (png bytes, w, h) -> decoded [n, T, T, 3] via the store's GPU path."""
    import torch

    from paper_2404_15217_b200 import store

    level = torch.zeros((1, len(tiles), T, T, 3), dtype=torch.uint8, device="cuda")
    part = [(i, 0, w, h, store._png_zlib_stream(b, w, h)) for i, (b, w, h) in enumerate(tiles)]
    store._decode_png_tiles(level, T, part)
    return level[0].cpu().numpy()


def _image(rs, h, w, smooth):
    if smooth:
        yy, xx = np.mgrid[0:h, 0:w]
        base = np.stack([(xx * 3 + yy) % 256, (yy * 5) % 256, (xx ^ yy) % 256], -1)
        return np.clip(base + rs.integers(-3, 4, (h, w, 3)), 0, 255).astype(np.uint8)
    return rs.integers(0, 256, (h, w, 3), dtype=np.uint8)


def test_all_filters_and_block_types(cuda):
    rs = np.random.default_rng(0)
    T = 64
    tiles, want = [], []
    for level in (0, 1, 6, 9):
        for smooth in (True, False):
            for (h, w) in ((64, 64), (17, 64), (64, 5), (1, 1), (33, 47)):
                img = _image(rs, h, w, smooth)
                tiles.append((_png(img, rs.integers(0, 5, h), level), w, h))
                want.append(img)
    got = _decode(tiles, T)
    for k, img in enumerate(want):
        h, w, _ = img.shape
        assert np.array_equal(got[k, :h, :w], img), k


def test_pillow_written_tiles(cuda):
    from PIL import Image

    rs = np.random.default_rng(1)
    tiles, want = [], []
    for smooth in (True, False):
        for size in ((256, 256), (256, 100), (31, 256)):
            img = _image(rs, size[0], size[1], smooth)
            buf = io.BytesIO()
            Image.fromarray(img).save(buf, format="PNG")
            tiles.append((buf.getvalue(), size[1], size[0]))
            want.append(img)
    got = _decode(tiles, 256)
    for k, img in enumerate(want):
        assert np.array_equal(got[k, :img.shape[0], :img.shape[1]], img), k


def test_corrupt_streams_raise(cuda):
    from paper_2404_15217_b200 import store
    from paper_2404_15217_b200.errors import DecodeError

    rs = np.random.default_rng(2)
    img = _image(rs, 32, 32, True)
    good = _png(img, rs.integers(0, 5, 32), 6)
    with pytest.raises(DecodeError):  # flipped IDAT byte: the chunk CRC catches it on the host
        bad = bytearray(good)
        bad[60] ^= 0xFF
        store._png_zlib_stream(bytes(bad), 32, 32)
    # a valid-CRC stream whose deflate data is truncated: the GPU inflater reports it
    ihdr = good[8:33]
    z = zlib.compress(_filter_rows(img, np.zeros(32, int)), 6)[:-20]
    trunc = b"\x89PNG\r\n\x1a\n" + ihdr + struct.pack(">I", len(z)) + b"IDAT" + z + struct.pack(
        ">I", zlib.crc32(b"IDAT" + z)) + good[-12:]
    with pytest.raises(DecodeError):
        _decode([(trunc, 32, 32)], 32)
    assert store._png_zlib_stream(good.replace(struct.pack(">IIBBBBB", 32, 32, 8, 2, 0, 0, 0),
                                               struct.pack(">IIBBBBB", 32, 32, 8, 2, 0, 0, 0)), 32, 32) is not None
