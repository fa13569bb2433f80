"""Pin the float32 restatement of torchvision's uint8 colour ops (oracle/augment.py) that the CUDA
multi-crop kernel implements, against torchvision itself (CPU)."""

import numpy as np
import pytest

from oracle import augment as A
from oracle import port

torch = pytest.importorskip("torch")
TF = pytest.importorskip("torchvision.transforms.v2.functional")


def _img(seed, h=53, w=61):
    rs = np.random.default_rng(seed)
    a = rs.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
    a[rs.random((h, w)) < 0.1] = rs.integers(0, 256, size=3)  # some equal-channel pixels
    a[rs.random((h, w)) < 0.05] = 255
    return a


def _tv(fn, img, *args, **kw):
    x = torch.from_numpy(img).permute(2, 0, 1).contiguous()
    return fn(x, *args, **kw).permute(1, 2, 0).numpy()


@pytest.mark.parametrize("seed", range(6))
def test_pointwise_ops_exact(seed):
    img = _img(seed)
    rs = np.random.default_rng(100 + seed)
    for _ in range(4):
        f = float(np.float32(rs.uniform(0.6, 1.4)))
        assert np.array_equal(A.brightness(img, f), _tv(TF.adjust_brightness, img, f))
        assert np.array_equal(A.contrast(img, f), _tv(TF.adjust_contrast, img, f))
        s = float(np.float32(rs.uniform(0.8, 1.2)))
        assert np.array_equal(A.saturation(img, s), _tv(TF.adjust_saturation, img, s))
        h = float(np.float32(rs.uniform(-0.1, 0.1)))
        assert np.array_equal(A.hue(img, h), _tv(TF.adjust_hue, img, h))
    assert np.array_equal(A.grayscale3(img), _tv(TF.rgb_to_grayscale, img, num_output_channels=3))
    assert np.array_equal(A.solarize(img, 128), _tv(TF.solarize, img, 128.0))


@pytest.mark.parametrize("seed", range(4))
def test_blur_within_one_lsb(seed):
    img = _img(seed, 96, 96)
    rs = np.random.default_rng(seed)
    for sigma in (0.1, float(np.float32(rs.uniform(0.1, 2.0))), 2.0):
        got = A.blur(img, sigma)
        want = _tv(TF.gaussian_blur, img, [9, 9], [sigma, sigma])
        d = np.abs(got.astype(int) - want.astype(int))
        assert d.max() <= 1 and (d > 0).mean() < 1e-3


def test_resized_crop_is_torch_aa():
    from torchvision.transforms import InterpolationMode

    rs = np.random.default_rng(5)
    src = rs.integers(0, 256, size=(224, 224, 3), dtype=np.uint8)
    for _ in range(12):
        h, w = int(rs.integers(10, 225)), int(rs.integers(10, 225))
        top, left = int(rs.integers(0, 225 - h)), int(rs.integers(0, 225 - w))
        o = int(rs.choice([96, 224]))
        want = _tv(TF.resized_crop, src, top, left, h, w, [o, o], interpolation=InterpolationMode.BILINEAR, antialias=True)
        got = port.aa_resize_hwc(src[top:top + h, left:left + w], o, o, "torch")
        assert np.array_equal(got, want)
