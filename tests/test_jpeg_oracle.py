"""The JPEG restatement (oracle/jpeg.py) against Pillow's decoder (libjpeg-turbo): baseline
files Pillow writes at several qualities, sizes (1 px .. 256 px, odd edges) and contents."""

import io

import numpy as np
import pytest

from oracle import jpeg as J

Image = pytest.importorskip("PIL.Image")


def _img(rs, h, w, smooth):
    if smooth:
        yy, xx = np.mgrid[0:h, 0:w]
        base = np.stack([(xx * 7 + yy) % 256, (yy * 3) % 256, (xx * yy) % 256], -1)
        return np.clip(base + rs.integers(-5, 6, (h, w, 3)), 0, 255).astype(np.uint8)
    return rs.integers(0, 256, (h, w, 3), dtype=np.uint8)


@pytest.mark.parametrize("quality", [90, 75])
def test_restatement_matches_pillow(quality):
    rs = np.random.default_rng(quality)
    for h in (1, 2, 3, 8, 17, 60, 256):
        for w in (1, 2, 3, 5, 9, 33, 100, 256):
            for smooth in (True, False):
                a = _img(rs, h, w, smooth)
                buf = io.BytesIO()
                Image.fromarray(a).save(buf, format="JPEG", quality=quality)
                want = np.asarray(Image.open(io.BytesIO(buf.getvalue())).convert("RGB"))
                assert np.array_equal(J.decode(buf.getvalue()), want), (h, w, smooth)
