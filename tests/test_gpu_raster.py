"""GPU: the polygon classification raster (csrc/pf_raster.cu) in front of the sampler's overlap
test.  Its claim -- every point of a clean cell, grown by 1 px, has the cell's even-odd parity
-- is checked point-wise with the exact device test (pf_overlap_fraction on tiny windows, so
every lattice point is a probe), window decisions are checked against overlap_fraction, and
the sampler's spec stream is the same with and without rasters."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def polys(cuda):
    import paper_2404_15217_b200 as pf

    z = np.load(GOLDEN / "c2_polygons.npz")
    out = []
    for g in range(2):
        rings = [z[f"s{g}_ring{r}"] for r in range(int(z[f"s{g}_nrings"][0]))]
        out.append(pf.ForegroundPolygon(rings=rings, slide_id=f"c2_{g}"))
    return pf, out


def _decode(raster, level=0):
    raw = raster.cpu().numpy()
    for _ in range(level):  # header.coarse: byte offset of the next level
        raw = raw[int(raw[48:56].view(np.int64)[0]):]
    ox, oy, cell, inv = raw[:32].view(np.float64)
    nx, ny, pitch, magic = raw[32:48].view(np.int32)
    assert magic == 0x50465231
    words = raw[64:64 + 4 * ny * pitch].view(np.uint32).reshape(ny, pitch)
    codes = np.zeros((ny, pitch * 16), dtype=np.uint8)
    for k in range(16):
        codes[:, k::16] = (words >> (2 * k)) & 3
    return ox, oy, cell, codes[:, :nx]


def _fractions(pf, poly, rects, grid=32):
    import torch

    r = torch.from_numpy(np.ascontiguousarray(rects, dtype=np.float64)).cuda()
    out = torch.empty(len(rects), dtype=torch.float64, device="cuda")
    pf._native.check(pf._native.lib().pf_overlap_fraction(poly.device_blob().data_ptr(), r.data_ptr(), len(rects),
                                                          grid, out.data_ptr(), None), "pf_overlap_fraction")
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("level", [0, 1])
def test_clean_cells_have_one_parity(polys, level):
    pf, ps = polys
    rs = np.random.default_rng(level)
    for poly in ps:
        ox, oy, cell, codes = _decode(poly.device_raster(), level)
        ny, nx = codes.shape
        clean = np.argwhere(codes < 2)
        assert len(clean) > 0.5 * codes.size and (codes == 1).sum() > 0 and (codes == 2).sum() > 0
        pick = clean[rs.choice(len(clean), size=min(6000, len(clean)), replace=False)]
        # a tiny window anywhere in the grown cell: its 33x33 lattice points all probe the parity
        gx = ox + pick[:, 1] * cell - 1.0 + rs.random(len(pick)) * (cell + 2.0 - 0.5)
        gy = oy + pick[:, 0] * cell - 1.0 + rs.random(len(pick)) * (cell + 2.0 - 0.5)
        rects = np.stack([gx, gy, np.full(len(pick), 0.5), np.full(len(pick), 0.5)], axis=1)
        f = _fractions(pf, poly, rects)
        want = np.where(codes[pick[:, 0], pick[:, 1]] == 1, 1.0, 0.0)
        assert np.array_equal(f, want)


def _decide(ox, oy, cell, codes, x, y, w):
    ny, nx = codes.shape
    a0, a1 = int(np.floor((x - ox) / cell)), int(np.floor((x + w - ox) / cell))
    b0, b1 = int(np.floor((y - oy) / cell)), int(np.floor((y + w - oy) / cell))
    partial = a0 < 0 or b0 < 0 or a1 >= nx or b1 >= ny
    sub = codes[max(b0, 0):min(b1, ny - 1) + 1, max(a0, 0):min(a1, nx - 1) + 1]
    if not partial and sub.size and (sub == 1).all():
        return 1
    if (sub == 0).all():
        return 0
    return -1


def test_window_decisions_match_overlap_fraction(polys):
    pf, ps = polys
    rs = np.random.default_rng(1)
    for poly in ps:
        ox, oy, cell, codes = _decode(poly.device_raster())
        bx0, by0, bx1, by1 = poly.bounding_box()
        n = 4000
        w = rs.choice([224.0, 448.0, 896.0, 1792.0], size=n)
        x = np.floor(bx0 - 300 + rs.random(n) * (bx1 - bx0 + 600))
        y = np.floor(by0 - 300 + rs.random(n) * (by1 - by0 + 600))
        d = np.array([_decide(ox, oy, cell, codes, x[i], y[i], w[i]) for i in range(n)])
        assert (d == 1).sum() > 0.2 * n and (d == 0).sum() > 0.1 * n
        f = _fractions(pf, poly, np.stack([x, y, w, w], axis=1), grid=128)
        assert np.all(f[d == 1] == 1.0) and np.all(f[d == 0] == 0.0)


def test_sampler_stream_same_without_raster(polys):
    pf, ps = polys
    import torch
    from paper_2404_15217_b200.store import LevelInfo, SlideRecord

    # metadata-only records of the C2 slides (40000 x 30000, levels 1/4/16): the sampler reads
    # no pixels
    recs = [SlideRecord(f"c2_{g}", 0.25, 256, [LevelInfo(40000, 30000, 0.25, 1), LevelInfo(10000, 7500, 1.0, 4),
                                               LevelInfo(2500, 1875, 4.0, 16)]) for g in range(2)]
    cfg = pf.SamplerConfig(patch_size=224, seed=3, target_mpps=[(0.25, 1.0), (0.5, 1.0), (1.0, 1.0), (2.0, 1.0)])
    a = pf.GpuSampler(cfg, list(zip(recs, ps)))
    b = pf.GpuSampler(cfg, list(zip(recs, ps)), raster=False)
    for k in (1024, 517, 2048):
        oa, ob = a.next_batch(k), b.next_batch(k)
        torch.cuda.synchronize()
        assert torch.equal(oa, ob)
    a.check()


def _bounds(ox, oy, cell, codes, x, y, w, grid):
    """Python mirror of raster_bounds_thread (pf_poly.cuh)."""
    ny, nx = codes.shape
    inv = grid / w

    def span(origin, p0, c):  # noqa: E306
        c0 = origin + c * cell
        k0 = max(0, int(np.ceil((c0 - p0) * inv)))
        k1 = min(grid - 1, int(np.floor((c0 + cell - p0) * inv)) - 1)
        return max(0, k1 - k0 + 1)

    a0, a1 = int(np.floor((x - ox) / cell)), int(np.floor((x + w - ox) / cell))
    b0, b1 = int(np.floor((y - oy) / cell)), int(np.floor((y + w - oy) / cell))
    lo = out = 0
    for r in range(b0, b1 + 1):
        bh = span(oy, y, r)
        for c in range(a0, a1 + 1):
            aw = span(ox, x, c)
            code = codes[r, c] if 0 <= r < ny and 0 <= c < nx else 0
            if code == 1:
                lo += aw * bh
            elif code == 0:
                out += aw * bh
    return lo, grid * grid - out


def test_count_bounds_hold(polys):
    """The classification pass's covered-cell bounds bracket overlap_fraction's exact count, and
    are tight enough to settle most boundary windows at the sampler's threshold (windows 16 or
    more fine cells wide read the coarse level, as raster_bounds_thread does)."""
    pf, ps = polys
    rs = np.random.default_rng(2)
    grid = 128
    need = 0.4 * grid * grid
    for poly in ps:
        levels = [_decode(poly.device_raster(), lv) for lv in (0, 1)]
        bx0, by0, bx1, by1 = poly.bounding_box()
        n = 3000
        w = rs.choice([224.0, 448.0, 896.0, 1792.0], size=n)
        x = np.floor(bx0 + rs.random(n) * (bx1 - bx0))
        y = np.floor(by0 + rs.random(n) * (by1 - by0))

        def bounds(i):
            ox, oy, cell, codes = levels[0]
            if int(np.floor((x[i] + w[i] - ox) / cell)) - int(np.floor((x[i] - ox) / cell)) >= 16:
                ox, oy, cell, codes = levels[1]
            return _bounds(ox, oy, cell, codes, x[i], y[i], w[i], grid)

        b = np.array([bounds(i) for i in range(n)])
        count = np.rint(_fractions(pf, poly, np.stack([x, y, w, w], axis=1), grid=grid) * grid * grid)
        assert np.all(b[:, 0] <= count) and np.all(count <= b[:, 1])
        boundary = (count > 0) & (count < grid * grid)
        settled = boundary & ((b[:, 0] >= need) | (b[:, 1] < need))
        assert boundary.sum() > 50 and settled.sum() > 0.3 * boundary.sum()


def test_large_batches_and_windows_keep_the_stream(polys):
    """Batches of thousands of specs: split into sub-batches whose window keeps the walk's table
    (entries below the 0x4000 mark), or walked over the bitmaps when a forced window is larger,
    or sampled 1000 at a time -- the same stream."""
    pf, ps = polys
    import torch
    from paper_2404_15217_b200.store import LevelInfo, SlideRecord

    recs = [SlideRecord(f"c2_{g}", 0.25, 256, [LevelInfo(40000, 30000, 0.25, 1), LevelInfo(10000, 7500, 1.0, 4),
                                               LevelInfo(2500, 1875, 4.0, 16)]) for g in range(2)]
    cfg = pf.SamplerConfig(patch_size=224, seed=11, max_attempts_per_slide=8)
    pairs = list(zip(recs, ps))
    a = pf.GpuSampler(cfg, pairs, rounds=1)
    b = pf.GpuSampler(cfg, pairs, rounds=1, window=20000)
    c = pf.GpuSampler(cfg, pairs, rounds=2)
    oa = a.next_batch(9000)
    ob = b.next_batch(9000)
    oc = torch.cat([c.next_batch(1000) for _ in range(9)])
    torch.cuda.synchronize()
    assert torch.equal(oa, ob) and torch.equal(oa, oc)
    for s in (a, b, c):
        s.check()
