"""Multi-crop augmentation oracle (TEST INFRASTRUCTURE ONLY).

The reference has no augmentation stage; BASELINE.json
config 2 asks for the DINOv2 multi-crop.  The oracle is torchvision 0.26
``transforms.v2.functional`` on uint8 CHW tensors, driven by the explicit
per-crop parameter records the GPU parameter generator exports
(pf_crop_param) — parity with the reference is therefore "unpinned"; parity
with torchvision is what the tests check.

``restated`` below re-derives each torchvision uint8 op as explicit float32
arithmetic (one IEEE rounding per torch op; ``fma`` where ATen's vectorised
``add(…, alpha)`` fuses).  tests/test_aug_semantics.py pins it against
torchvision on the CPU; the CUDA kernel (csrc/pf_multicrop.cu) evaluates the
same expressions.
"""

from __future__ import annotations

import math

import numpy as np

F32 = np.float32
AUG_FLIP, AUG_JITTER, AUG_GRAY, AUG_BLUR, AUG_SOLARIZE = 1, 2, 4, 8, 16


def torchvision_crop(src_hwc: np.ndarray, p) -> np.ndarray:
    """One crop of one patch through torchvision v2 functional ops -> (O, O, 3) uint8."""
    import torch
    from torchvision.transforms import InterpolationMode
    from torchvision.transforms.v2 import functional as TF

    x = torch.from_numpy(np.ascontiguousarray(src_hwc)).permute(2, 0, 1).contiguous()
    o = int(p["out_size"])
    x = TF.resized_crop(x, int(p["top"]), int(p["left"]), int(p["height"]), int(p["width"]), [o, o],
                        interpolation=InterpolationMode.BILINEAR, antialias=True)
    flags = int(p["flags"])
    if flags & AUG_FLIP:
        x = TF.horizontal_flip(x)
    if flags & AUG_JITTER:
        for op in p["order"]:
            if op == 0:
                x = TF.adjust_brightness(x, float(p["brightness"]))
            elif op == 1:
                x = TF.adjust_contrast(x, float(p["contrast"]))
            elif op == 2:
                x = TF.adjust_saturation(x, float(p["saturation"]))
            else:
                x = TF.adjust_hue(x, float(p["hue"]))
    if flags & AUG_GRAY:
        x = TF.rgb_to_grayscale(x, num_output_channels=3)
    if flags & AUG_BLUR:
        s = float(p["sigma"])
        x = TF.gaussian_blur(x, [9, 9], [s, s])
    if flags & AUG_SOLARIZE:
        x = TF.solarize(x, float(p["solarize_threshold"]))
    return x.permute(1, 2, 0).contiguous().numpy()


def normalize(u8: np.ndarray, mean, std) -> np.ndarray:
    """ToTensor (v/255) + Normalize ((x - mean)/std), float32, HWC."""
    return (u8.astype(np.float32) / F32(255.0) - np.asarray(mean, F32)) / np.asarray(std, F32)


# ---------------------------------------------------------------------------
# explicit float32 restatement of the torchvision uint8 ops


def fma32(a, b, c):
    """fma in float32: the product of two floats is exact in float64, the sum is exact here
    (small magnitudes), so one rounding to float32 gives the fused result."""
    return (np.asarray(a, np.float64) * np.asarray(b, np.float64) + np.asarray(c, np.float64)).astype(F32)


def _trunc_u8(x):
    return np.clip(x, F32(0), F32(255)).astype(np.uint8)


def gray_f32(img):  # r.mul(0.2989).add_(g, alpha=0.587).add_(b, alpha=0.114)
    r, g, b = (img[..., i].astype(F32) for i in range(3))
    return fma32(b, F32(0.114), fma32(g, F32(0.587), r * F32(0.2989)))


def brightness(img, f):
    return _trunc_u8(img.astype(F32) * F32(f))


def blend(img, other, f):
    f = F32(f)
    alpha = F32(1.0 - float(f))
    return _trunc_u8(fma32(other, alpha, img.astype(F32) * f))


def contrast(img, f):
    g = np.floor(gray_f32(img))
    mean = F32(F32(g.sum(dtype=np.float64)) / F32(g.size))
    return blend(img, mean, f)


def saturation(img, f):
    return blend(img, np.floor(gray_f32(img))[..., None], f)


def hue(img, hf):
    x = img.astype(F32) * F32(1.0 / 255.0)
    r, g, b = x[..., 0], x[..., 1], x[..., 2]
    maxc, minc = x.max(axis=-1), x.min(axis=-1)
    eqc = maxc == minc
    cr = maxc - minc
    s = cr / np.where(eqc, F32(1), maxc)
    crd = np.where(eqc, F32(1), cr)
    rc, gc, bc = (maxc - r) / crd, (maxc - g) / crd, (maxc - b) / crd
    neq_r, eq_g = maxc != r, maxc == g
    hr = np.where(~neq_r, bc - gc, F32(0))
    hg = np.where(eq_g & neq_r, (rc + F32(2)) - bc, F32(0))
    hb = np.where(neq_r & ~eq_g, (gc + F32(4)) - rc, F32(0))
    h = (hr + hg) + hb
    h = np.fmod(h * F32(1.0 / 6.0) + F32(1.0), F32(1.0))
    h = h + F32(hf)
    h = np.fmod(h, F32(1.0))
    h = np.where(h < 0, h + F32(1.0), h)
    h6 = h * F32(6)
    i = np.floor(h6)
    fr = h6 - i
    i = np.mod(i.astype(np.int32), 6)
    v = maxc
    sxf = s * fr
    oms = F32(1.0) - s
    q = np.clip((F32(1.0) - sxf) * v, F32(0), F32(1))
    t = np.clip((sxf + oms) * v, F32(0), F32(1))
    p = np.clip(oms * v, F32(0), F32(1))
    tab = np.stack([v, p, q, t], -1)
    sel = np.array([[0, 2, 1, 1, 3, 0], [3, 0, 0, 2, 1, 1], [1, 1, 3, 0, 0, 2]])
    out = np.stack([np.take_along_axis(tab, sel[c][i][..., None], -1)[..., 0] for c in range(3)], -1)
    return (out * F32(255.999)).astype(np.uint8)


def grayscale3(img):
    g = gray_f32(img).astype(np.uint8)
    return np.repeat(g[..., None], 3, axis=-1)


def gaussian_kernel1d(sigma: float) -> np.ndarray:
    """torchvision _get_gaussian_kernel1d(9, sigma) in float32 (linspace, softmax)."""
    lim = (9 - 1) / (2.0 * math.sqrt(2.0))
    import torch

    x = torch.linspace(-lim, lim, steps=9, dtype=torch.float32)
    return torch.softmax(x.div(float(F32(sigma))).pow(2).neg(), dim=0).numpy()


def blur(img, sigma):
    """Separable reflect-padded blur, float32, round half to even."""
    k = gaussian_kernel1d(sigma)
    a = img.astype(F32)
    pad = np.pad(a, ((4, 4), (4, 4), (0, 0)), mode="reflect")
    h = np.zeros((pad.shape[0], a.shape[1], 3), F32)
    for j in range(9):
        h = fma32(pad[:, j:j + a.shape[1]], k[j], h)
    v = np.zeros(a.shape, F32)
    for j in range(9):
        v = fma32(h[j:j + a.shape[0]], k[j], v)
    return np.clip(np.rint(v), 0, 255).astype(np.uint8)


def solarize(img, thr):
    return np.where(img >= thr, 255 - img, img).astype(np.uint8)
