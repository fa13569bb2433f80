"""GPU parity: tissue masks and overlap_fraction (bit-exact FP64 even-odd test)."""

import hashlib

import numpy as np
import pytest

from oracle import port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf(cuda):
    import paper_2404_15217_b200 as pf

    return pf


def test_luminance_mask_all_colours(pf, goldens, golden_arrays):
    allc = np.arange(1 << 24, dtype=np.uint32)
    rgb = np.stack([(allc >> 16) & 255, (allc >> 8) & 255, allc & 255], axis=1).astype(np.uint8).reshape(4096, 4096, 3)
    for thr in (0.9, 0.5, 0.25):
        bits = pf.mask_from_rgb(rgb, thr).bits
        assert hashlib.sha256(np.packbits(bits).tobytes()).hexdigest() == goldens[f"allcolors_lum_{thr}_sha256"], thr
    m = pf.mask_from_rgb(golden_arrays["blob_thumb8"], 0.9, scale=1 / 8)
    assert np.array_equal(m.bits, golden_arrays["blob_mask_lum"]) and m.scale == 1 / 8
    with pytest.raises(ValueError):
        pf.mask_from_rgb(rgb, 1.0)


def test_saturation_mask_vs_scipy(pf):
    rs = np.random.default_rng(4)
    for radius in (0, 1, 2):
        img = rs.integers(0, 256, size=(97, 131, 3), dtype=np.uint8)
        img[rs.random((97, 131)) < 0.5] = 240  # gray pixels -> saturation 0
        got = pf.mask_from_saturation(img, 0.07, morph_radius=radius).bits
        assert np.array_equal(got, port.mask_saturation(img, 0.07, radius)), radius


def test_overlap_fraction_goldens(pf, goldens):
    poly = pf.ForegroundPolygon.from_json_dict(goldens["blob_poly"])
    rects = np.array([r[:4] for r in goldens["blob_overlap"]])
    got = pf.overlap_fractions(poly, rects).cpu().numpy()
    assert got.tolist() == [r[4] for r in goldens["blob_overlap"]]
    hpoly = pf.ForegroundPolygon.from_json_dict(goldens["hand_poly"])
    got = pf.overlap_fractions(hpoly, np.array([r[:4] for r in goldens["hand_overlap_grid64"]]), grid=64).cpu().numpy()
    assert got.tolist() == [r[4] for r in goldens["hand_overlap_grid64"]]
    rp = pf.rect_polygon(0, 0, 100, 100)
    assert [pf.overlap_fraction(rp, r) for r in ((10, 10, 20, 20), (200, 200, 20, 20), (90, 10, 20, 20))] == goldens["rect_kats"]


def test_overlap_fraction_random_vs_oracle(pf, goldens):
    rs = np.random.default_rng(9)
    for key in ("blob_poly", "sampler_poly_b1", "sampler_poly_b2"):
        poly = pf.ForegroundPolygon.from_json_dict(goldens[key])
        bx0, by0, bx1, by1 = poly.bounding_box()
        n = 60
        w = rs.choice([1.0, 5.0, 16.0, 33.0, 64.0, 224.0], size=n)
        rects = np.stack([rs.uniform(bx0 - 50, bx1, n), rs.uniform(by0 - 50, by1, n), w, w * rs.choice([1.0, 0.5], n)], 1)
        rects[::7, :2] = np.round(rects[::7, :2])  # integer corners land exactly on polygon edges
        for grid in (128, 32, 200):
            got = pf.overlap_fractions(poly, rects, grid=grid).cpu().numpy()
            want = [port.overlap_fraction(poly.rings, tuple(r), grid) for r in rects]
            assert got.tolist() == want, (key, grid)


def test_polygon_from_device_mask_pipeline(pf, goldens, golden_arrays):
    # thumbnail -> mask -> polygon with all device steps, equal to the reference's polygon
    m = pf.mask_from_rgb(golden_arrays["blob_thumb8"], 0.9, scale=1 / 8)
    poly = pf.polygon_from_mask(m, slide_id="blob")
    for a, b in zip(poly.rings, goldens["blob_poly"]["rings"]):
        assert np.array_equal(a, np.asarray(b))


def test_overlap_uniform_window_shortcut_vs_oracle(pf, goldens):
    """Windows deep inside / outside / straddling horizontal and vertical edges, on polygons with
    holes and axis-aligned edges: the device's whole-window shortcut (no edge near the lattice)
    must equal the row-by-row even-odd count of the reference."""
    rs = np.random.default_rng(21)
    ring = lambda x0, y0, x1, y1: np.array([[x0, y0], [x1, y0], [x1, y1], [x0, y1]], float)
    polys = [
        pf.rect_polygon(100, 100, 400, 300),
        pf.ForegroundPolygon([ring(0, 0, 600, 600), ring(200, 200, 400, 400)[::-1]]),  # hole
        pf.ForegroundPolygon.from_json_dict(goldens["blob_poly"]),
    ]
    for poly in polys:
        bx0, by0, bx1, by1 = poly.bounding_box()
        n = 120
        w = rs.choice([16.0, 64.0, 100.0, 224.0], size=n)
        x = rs.uniform(bx0 - 120, bx1 + 20, n)
        y = rs.uniform(by0 - 120, by1 + 20, n)
        k = rs.random(n) < 0.4  # snap onto the 100-px lattice: windows touching edges exactly
        x[k], y[k] = np.round(x[k] / 100) * 100, np.round(y[k] / 100) * 100
        rects = np.stack([x, y, w, w], 1)
        for grid in (128, 64):
            got = pf.overlap_fractions(poly, rects, grid=grid).cpu().numpy()
            want = [port.overlap_fraction(poly.rings, tuple(r), grid) for r in rects]
            assert got.tolist() == want, grid
            assert 0.0 < np.mean(np.asarray(want) == 1.0) < 1.0  # both shortcut outcomes exercised
