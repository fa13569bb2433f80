"""polygon_from_mask (pkg/foreground.py:169-220) tracing pins that do not depend on the
builder's own find_contours restatement (scikit-image is not installed, so the goldens'
tracer is the oracle's restatement):

* the SPEC.md:149-153 examples: a filled 10x10 rectangle in a 100x100 mask gives one ring of
  area 100 +- 2; an empty mask raises EmptyForegroundError; a full mask gives one ring covering
  the extent with area W*H up to the perimeter error;
* marching-squares invariants of find_contours(padded, 0.5) on a binary image, whatever the
  implementation: the ring vertices are exactly the midpoints of the 4-neighbour pixel pairs
  with different values (each once), consecutive vertices share a 2x2 cell, and the oriented
  rings' signed areas sum to the per-cell case areas with saddles resolved as
  fully_connected='low' (1/8, 1/2, 1/4 for a saddle, 7/8, 1).

Run on the native tracer (host C++ in libpfb200.so, no device) and on the oracle.
"""

import numpy as np
import pytest

from oracle import port


def _native(bits, scale=1.0, mrp=64.0):
    from paper_2404_15217_b200.foreground import BinaryMask, polygon_from_mask

    return [np.asarray(r) for r in polygon_from_mask(BinaryMask(bits, scale), min_region_px=mrp).rings]


def _oracle(bits, scale=1.0, mrp=64.0):
    return [np.asarray(r) for r in port.polygon_from_mask(bits, scale, mrp)]


TRACERS = {"native": _native, "oracle": _oracle}


def _area(ring):
    return port.shoelace(np.asarray(ring))


@pytest.mark.parametrize("tracer", TRACERS)
def test_spec_filled_rectangle(tracer):
    m = np.zeros((100, 100), bool)
    m[30:40, 50:60] = True
    rings = TRACERS[tracer](m)
    assert len(rings) == 1
    assert abs(abs(_area(rings[0])) - 100.0) <= 2.0
    assert _area(rings[0]) > 0  # an outer boundary is positive (nesting depth 0)


@pytest.mark.parametrize("tracer", TRACERS)
def test_spec_empty_mask(tracer):
    from paper_2404_15217_b200.errors import EmptyForegroundError

    m = np.zeros((20, 30), bool)
    with pytest.raises((EmptyForegroundError, ValueError)):
        TRACERS[tracer](m)


@pytest.mark.parametrize("tracer", TRACERS)
@pytest.mark.parametrize("shape", [(64, 64), (37, 91)])
def test_spec_full_mask(tracer, shape):
    h, w = shape
    rings = TRACERS[tracer](np.ones(shape, bool))
    assert len(rings) == 1
    r = rings[0]
    assert np.isclose(r[:, 0].min(), -0.5) and np.isclose(r[:, 0].max(), w - 0.5)
    assert np.isclose(r[:, 1].min(), -0.5) and np.isclose(r[:, 1].max(), h - 0.5)
    assert abs(_area(r) - w * h) <= (w + h)  # perimeter error: the chamfered corners, 4 x 1/8 here


def _crossing_midpoints(bits):
    """Midpoints of 4-neighbour pixel pairs with different values (outside = background)."""
    p = np.pad(bits.astype(bool), 1)
    pts = set()
    ys, xs = np.nonzero(p[:, :-1] != p[:, 1:])
    for y, x in zip(ys, xs):  # pixels (y-1, x-1) and (y-1, x) in unpadded coordinates
        pts.add((x - 1 + 0.5, float(y - 1)))
    ys, xs = np.nonzero(p[:-1, :] != p[1:, :])
    for y, x in zip(ys, xs):
        pts.add((float(x - 1), y - 1 + 0.5))
    return pts


def _case_area(bits):
    """Sum over 2x2 cells of the foreground area inside the cell, saddles 'low'-connected."""
    p = np.pad(bits.astype(np.int64), 1)
    a, b, c, d = p[:-1, :-1], p[:-1, 1:], p[1:, :-1], p[1:, 1:]
    k = a + b + c + d
    saddle = (k == 2) & (a == d)
    area = np.select([k == 1, (k == 2) & ~saddle, saddle, k == 3, k == 4], [1 / 8, 1 / 2, 1 / 4, 7 / 8, 1.0], 0.0)
    return float(area.sum())


def _random_masks():
    rs = np.random.default_rng(7)
    out = []
    for h, w, p in [(12, 17, 0.5), (40, 33, 0.35), (64, 64, 0.6), (25, 80, 0.2)]:
        out.append(rs.random((h, w)) < p)
    # smooth blobs with holes
    yy, xx = np.mgrid[0:90, 0:120]
    out.append(((np.sin(xx / 9.0) + np.cos(yy / 7.0)) > 0.4))
    ck = np.indices((16, 16)).sum(axis=0) % 2 == 0  # every cell a saddle
    out.append(ck)
    return out


@pytest.mark.parametrize("tracer", TRACERS)
@pytest.mark.parametrize("k", range(6))
def test_marching_squares_invariants(tracer, k):
    bits = _random_masks()[k]
    rings = TRACERS[tracer](bits, 1.0, 1e-9)  # keep every non-degenerate ring
    verts = [tuple(map(float, v)) for r in rings for v in r]
    assert len(verts) == len(set(verts)), "a crossing edge visited twice"
    assert set(verts) == _crossing_midpoints(bits)
    for r in rings:  # consecutive vertices lie on the boundary of one 2x2 cell
        d = np.abs(r - np.roll(r, -1, axis=0))
        assert np.all((d[:, 0] <= 1.0) & (d[:, 1] <= 1.0) & (d.sum(axis=1) > 0))
    assert sum(_area(r) for r in rings) == pytest.approx(_case_area(bits), abs=1e-9)


@pytest.mark.parametrize("tracer", TRACERS)
def test_invariants_on_c2_masks(tracer):
    """The saturation masks of the two 40000 x 30000 C2 test slides (1250 x 938)."""
    from pathlib import Path

    z = np.load(Path(__file__).resolve().parent / "golden" / "c2_polygons.npz")
    for g in range(2):
        shape = tuple(z[f"s{g}_mask_shape"])
        bits = np.unpackbits(z[f"s{g}_mask"])[: shape[0] * shape[1]].reshape(shape).astype(bool)
        rings = TRACERS[tracer](bits, 1.0, 1e-9)
        verts = [tuple(map(float, v)) for r in rings for v in r]
        assert len(verts) == len(set(verts))
        assert set(verts) == _crossing_midpoints(bits)
        assert sum(_area(r) for r in rings) == pytest.approx(_case_area(bits), abs=1e-6)
        if tracer == "native":  # default filter + scale: the committed product rings
            got = _native(bits, float(z[f"s{g}_scale"][0]))
            want = [z[f"s{g}_ring{r}"] for r in range(int(z[f"s{g}_nrings"][0]))]
            assert len(got) == len(want) and all(np.array_equal(a, b) for a, b in zip(got, want))
