"""Synthetic H&E-like slides for the BASELINE configs (stand-ins for TCGA WSIs).

BASELINE.json: near-white background (230-250 per channel + N(0, 4) noise);
tissue = smooth random blobs from thresholded Gaussian-filtered noise,
~40 % coverage, pink/purple (R 150-220, G 60-140, B 140-210).  The smooth
field is tiny (one value per 64 level-0 px) and made on the host with a seeded
numpy generator; level 0 is rendered straight into HBM by pf_synth_level0 and
the pyramid is box-filtered on device.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native as N
from .store import GpuSlide

FIELD_CELL = 64


def _gaussian_blur(a: np.ndarray, sigma: float) -> np.ndarray:
    r = max(1, int(math.ceil(3 * sigma)))
    x = np.arange(-r, r + 1, dtype=np.float64)
    k = np.exp(-0.5 * (x / sigma) ** 2)
    k /= k.sum()
    p = np.pad(a, r, mode="wrap")
    p = np.apply_along_axis(lambda v: np.convolve(v, k, mode="valid"), 1, p)
    p = np.apply_along_axis(lambda v: np.convolve(v, k, mode="valid"), 0, p)
    return p


def tissue_field(width: int, height: int, seed: int, coverage: float = 0.40, blob_px: float = 2048.0,
                 cell: int = FIELD_CELL):
    """Smooth field on a (ceil(H/cell)+1, ceil(W/cell)+1) grid and the threshold giving `coverage`."""
    fw, fh = -(-width // cell) + 1, -(-height // cell) + 1
    rs = np.random.default_rng(seed)
    noise = rs.standard_normal((fh, fw))
    f = _gaussian_blur(noise, max(blob_px / cell / 2.0, 0.75))
    f = (f - f.min()) / max(f.max() - f.min(), 1e-12)
    thr = float(np.quantile(f, 1.0 - coverage))
    # C order: apply_along_axis leaves the blurred field Fortran-ordered, and the renderer
    # indexes the raw buffer row-major
    return np.ascontiguousarray(f, dtype=np.float32), thr


def synthetic_slide(slide_id: str, width: int, height: int, *, seed: int = 0, base_mpp: float = 0.25,
                    tile_size: int = 256, downsample_factor: int = 4, coverage: float = 0.40,
                    blob_px: float = 2048.0, stream=None) -> GpuSlide:
    """Allocate a pyramid in HBM and render a synthetic slide into it."""
    torch = N.require_cuda()
    slide = GpuSlide.allocate(slide_id, width, height, base_mpp, tile_size, downsample_factor)
    field, thr = tissue_field(width, height, seed, coverage, blob_px)
    fdev = torch.from_numpy(np.ascontiguousarray(field)).cuda().contiguous()
    N.check(N.lib().pf_synth_level0(slide.desc, fdev.data_ptr(), field.shape[0], field.shape[1], FIELD_CELL,
                                    float(thr), int(seed) & ((1 << 64) - 1), N.stream_ptr(stream)),
            "pf_synth_level0")
    slide.build_pyramid(stream)
    torch.cuda.current_stream().synchronize() if stream is None else stream.synchronize()
    del fdev
    return slide
