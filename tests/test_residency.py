"""Residency planner (residency.reachable_tiles): every tile that a window intersecting the
foreground polygon can read -- at any pyramid level, with read_region's window rounding -- is
planned resident.  Host-only (numpy oracle for the polygon and the even-odd test)."""

import numpy as np

from oracle import port
from paper_2404_15217_b200 import residency as R
from paper_2404_15217_b200.store import make_record


def _blob_mask(seed, h=60, w=80):
    rs = np.random.default_rng(seed)
    m = np.zeros((h, w), bool)
    for _ in range(5):
        cy, cx, r = rs.integers(0, h), rs.integers(0, w), rs.integers(3, 12)
        yy, xx = np.mgrid[0:h, 0:w]
        m |= (yy - cy) ** 2 + (xx - cx) ** 2 < r * r
    return m


def _tiles_read(rec, x, y, fp, mpp):
    """Tiles of level select_level(mpp) that read_region(x, y, fp, fp) touches (store.py:667-724)."""
    li = port.select_level([lv.mpp for lv in rec.levels], mpp)
    lv = rec.levels[li]
    T = rec.tile_size
    side = max(1, port.round_half_away(fp * rec.base_mpp / lv.mpp))
    sx, sy = port.round_half_away(x / lv.downsample), port.round_half_away(y / lv.downsample)
    x0, y0 = min(max(sx, 0), lv.width - 1), min(max(sy, 0), lv.height - 1)
    x1, y1 = min(max(sx + side - 1, 0), lv.width - 1), min(max(sy + side - 1, 0), lv.height - 1)
    return li, [(tx, ty) for ty in range(y0 // T, y1 // T + 1) for tx in range(x0 // T, x1 // T + 1)]


def test_windows_touching_foreground_only_read_planned_tiles():
    scale = 1 / 32
    for seed in range(3):
        bits = _blob_mask(seed)
        rec = make_record("r", 80 * 32, 60 * 32, 0.25, tile_size=64, downsample_factor=2)
        rings = port.polygon_from_mask(bits, scale, 64.0)
        for mpp, fp in ((0.25, 224), (0.5, 448)):
            plan = R.reachable_tiles(rec, bits, scale, fp)
            assert 0 < sum(int(p.sum()) for p in plan) < sum(p.size for p in plan)  # sparse, non-empty
            rs = np.random.default_rng(100 + seed)
            hits = 0
            for _ in range(400):
                x, y = int(rs.integers(-fp // 2, rec.levels[0].width)), int(rs.integers(-fp // 2, rec.levels[0].height))
                g = np.linspace(0.0, fp, 17)
                pts = np.stack(np.meshgrid(x + g, y + g), -1).reshape(-1, 2)
                if not port.points_in_polygon(pts, rings).any():
                    continue  # overlap 0 < min_foreground: never sampled
                hits += 1
                li, tiles = _tiles_read(rec, max(x, 0), max(y, 0), fp, mpp)
                for tx, ty in tiles:
                    assert plan[li][ty, tx], (seed, mpp, x, y, li, tx, ty)
            assert hits > 50


def test_resident_and_dense_bytes():
    rec = make_record("r", 1000, 700, 0.25, tile_size=128, downsample_factor=4)
    plan = [np.ones(rec.tile_grid(li)[::-1], bool) for li in range(len(rec.levels))]
    tb = 128 * 128 * 3
    assert R.dense_bytes(rec) == sum(int(np.prod(rec.tile_grid(li))) for li in range(len(rec.levels))) * tb
    assert R.resident_bytes(rec, plan) == R.dense_bytes(rec) + len(rec.levels) * tb
    assert R.max_footprint(rec, 224, [(0.25, 1.0), (0.5, 1.0)]) == 448.0
