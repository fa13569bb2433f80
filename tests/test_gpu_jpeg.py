"""GPU baseline JPEG tile decode (pf_jpeg_decode) bit-exact with Pillow's decoder and the
restatement in oracle/jpeg.py, through the store's load path."""

import io

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
Image = pytest.importorskip("PIL.Image")


def _img(rs, h, w, smooth):
    if smooth:
        yy, xx = np.mgrid[0:h, 0:w]
        base = np.stack([(xx * 7 + yy) % 256, (yy * 3) % 256, (xx * yy) % 256], -1)
        return np.clip(base + rs.integers(-5, 6, (h, w, 3)), 0, 255).astype(np.uint8)
    return rs.integers(0, 256, (h, w, 3), dtype=np.uint8)


def test_tiles_match_pillow(cuda):
    import torch

    from paper_2404_15217_b200 import store

    rs = np.random.default_rng(0)
    T = 256
    cases = [(h, w, sm, q) for h, w in ((256, 256), (256, 100), (31, 256), (17, 33), (8, 8), (3, 5), (1, 1), (2, 3))
             for sm in (True, False) for q in (90, 75)]
    level = torch.zeros((1, len(cases), T, T, 3), dtype=torch.uint8, device="cuda")
    tiles, want = [], []
    for k, (h, w, sm, q) in enumerate(cases):
        a = _img(rs, h, w, sm)
        buf = io.BytesIO()
        Image.fromarray(a).save(buf, format="JPEG", quality=q)
        want.append(np.asarray(Image.open(io.BytesIO(buf.getvalue())).convert("RGB")))
        tiles.append((k, 0, w, h, buf.getvalue()))
    assert store._decode_jpeg_tiles(level, T, tiles) == []
    got = level[0].cpu().numpy()
    for k, (h, w, sm, q) in enumerate(cases):
        assert np.array_equal(got[k, :h, :w], want[k]), cases[k]


def test_jpeg_store_loads_on_gpu(cuda, golden_arrays, tmp_path):
    """A reference-format JPEG store (ingest_image codec="jpeg") loads to the pixels Pillow
    decodes from the same files."""
    import paper_2404_15217_b200 as pf
    from paper_2404_15217_b200 import store

    img = golden_arrays["synthetic_700x500"]
    rec = pf.store.ingest_image(img, "s0", 0.25, tmp_path, tile_size=128, downsample_factor=2, codec="jpeg")
    gpu = pf.GpuSlide.from_store(tmp_path, "s0")
    host = pf.GpuSlide.from_store(tmp_path, "s0", gpu_png=False)
    for li in range(len(rec.levels)):
        assert cuda.equal(gpu.level_array(li), host.level_array(li)), li
    # a progressive tile is left to the host decoder; a truncated header is a DecodeError
    rs = np.random.default_rng(3)
    a = _img(rs, 16, 16, True)
    buf = io.BytesIO()
    Image.fromarray(a).save(buf, format="JPEG", quality=90, progressive=True)
    lv = cuda.zeros((1, 1, 16, 16, 3), dtype=cuda.uint8, device="cuda")
    assert store._decode_jpeg_tiles(lv, 16, [(0, 0, 16, 16, buf.getvalue())]) == [0]
    with pytest.raises(pf.errors.DecodeError):
        store._decode_jpeg_tiles(lv, 16, [(0, 0, 16, 16, buf.getvalue()[:30])])
