"""HBM tile residency planned from the tissue mask.

The reference keeps decoded tiles in a 64 MiB LRU (``TileCache``) and
fetches chunks on demand (``Slide.fetch_chunk``, pkg/store.py:270-319,
611-649).  On a B200 the sampler's working set is known before the first
read: ``sample_patch`` (pkg/sampler.py:140-184) only accepts windows whose
overlap with the foreground polygon reaches ``min_foreground`` > 0, every
accepted window therefore intersects the polygon, and the polygon
(marching squares at level 0.5 of the padded thumbnail mask,
pkg/foreground.py:169-220) lies within half a mask pixel of the mask's
foreground pixels.  So no admissible read ever touches a tile farther than
``footprint + margin`` level-0 pixels from a foreground mask pixel, and
those tiles need never enter HBM.  Slides whose full pyramids exceed the
180 GB of one GPU (BASELINE config 4) keep only their reachable tiles
resident; the rest map to an all-zero hole slot (``pf_slide_desc.tile_map``).
"""

from __future__ import annotations

import math

import numpy as np


def reachable_tiles(record, mask_bits: np.ndarray, mask_scale: float, footprint_l0: float,
                    margin_mask_px: int = 2) -> list:
    """Per level, a bool [tiles_y, tiles_x] grid of tiles an admissible read can touch.

    mask_bits: (h, w) foreground grid at ``mask_scale`` mask px per level-0 px.
    footprint_l0: the largest level-0 window side the sampler can emit
    (``footprint_px`` over the configured target mpps, pkg/sampler.py:118-127).
    margin_mask_px covers the polygon's half-pixel contour offset plus the
    +-1 level-L pixel of ``read_region``'s window rounding (pkg/store.py:679-681).
    """
    bits = np.asarray(mask_bits, dtype=bool)
    if bits.ndim != 2:
        raise ValueError("mask must be 2D")
    if not (0 < mask_scale <= 1):
        raise ValueError("mask_scale must be in (0, 1]")
    h, w = bits.shape
    sat = np.zeros((h + 1, w + 1), dtype=np.int64)  # summed-area table
    sat[1:, 1:] = bits.astype(np.int64).cumsum(0).cumsum(1)
    out = []
    T = record.tile_size
    for li, lv in enumerate(record.levels):
        ds = lv.downsample
        nx, ny = record.tile_grid(li)
        reach = footprint_l0 + 2.0 * ds  # level-0 px a read may extend past its window's tile
        # tile t covers level-0 [t*T*ds, (t+1)*T*ds); dilate by reach, convert to mask px
        def span(n):
            t = np.arange(n, dtype=np.float64)
            lo = np.floor((t * T * ds - reach) * mask_scale).astype(np.int64) - margin_mask_px
            hi = np.ceil(((t + 1) * T * ds + reach) * mask_scale).astype(np.int64) + margin_mask_px
            return lo, hi
        xlo, xhi = span(nx)
        ylo, yhi = span(ny)
        xlo, xhi = np.clip(xlo, 0, w), np.clip(xhi, 0, w)
        ylo, yhi = np.clip(ylo, 0, h), np.clip(yhi, 0, h)
        cnt = (sat[yhi[:, None], xhi[None, :]] - sat[ylo[:, None], xhi[None, :]]
               - sat[yhi[:, None], xlo[None, :]] + sat[ylo[:, None], xlo[None, :]])
        out.append(cnt > 0)
    return out


def max_footprint(record, patch_size: int, target_mpps) -> float:
    """Largest level-0 window side over the sampler's target mpps (footprint_px)."""
    from .store import round_half_away

    return float(max(max(1, round_half_away(patch_size * float(m) / record.base_mpp)) for m, _ in target_mpps))


def resident_bytes(record, plan) -> int:
    """HBM bytes of a compacted pyramid (resident tiles + one hole slot per level)."""
    tb = record.tile_size * record.tile_size * 3
    return int(sum((int(p.sum()) + 1) * tb for p in plan))


def dense_bytes(record) -> int:
    tb = record.tile_size * record.tile_size * 3
    return int(sum(math.prod(record.tile_grid(li)) * tb for li in range(len(record.levels))))
