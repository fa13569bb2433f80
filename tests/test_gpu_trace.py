"""On-GPU polygon tracing (pf_polygon_trace_device) against the host tracer
(pinned to the reference goldens in test_abi.py / test_oracle.py and to the implementation-free
marching-squares invariants in test_tracing_kats.py): same rings, same order, same start vertex
and orientation, bit-identical float64 vertices."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _masks(golden_arrays):
    rs = np.random.default_rng(11)
    out = [("blob_lum", golden_arrays["blob_mask_lum"], 1 / 8, 64.0), ("hand", golden_arrays["hand_mask"], 0.5, 4.0)]
    for k, (h, w, p) in enumerate([(12, 17, 0.5), (40, 33, 0.35), (64, 64, 0.6), (25, 80, 0.2), (200, 150, 0.45)]):
        out.append((f"rand{k}", rs.random((h, w)) < p, 1.0, 1e-9))
    yy, xx = np.mgrid[0:90, 0:120]
    out.append(("waves", (np.sin(xx / 9.0) + np.cos(yy / 7.0)) > 0.4, 0.25, 2.0))
    out.append(("checker", np.indices((16, 16)).sum(axis=0) % 2 == 0, 1.0, 0.0))
    out.append(("full", np.ones((37, 91), bool), 0.5, 64.0))
    z = np.load(Path(__file__).resolve().parent / "golden" / "c2_polygons.npz")
    for g in range(2):
        shape = tuple(z[f"s{g}_mask_shape"])
        bits = np.unpackbits(z[f"s{g}_mask"])[: shape[0] * shape[1]].reshape(shape).astype(bool)
        out.append((f"c2_s{g}", bits, float(z[f"s{g}_scale"][0]), 64.0))
    return out


def test_device_tracer_equals_host_tracer(cuda, golden_arrays):
    import paper_2404_15217_b200 as pf

    torch = cuda
    for name, bits, scale, mrp in _masks(golden_arrays):
        want = pf.polygon_from_mask(pf.BinaryMask(bits, scale), min_region_px=mrp)
        got = pf.polygon_from_mask_device(torch.from_numpy(bits.astype(np.uint8)).cuda(), scale, mrp)
        assert len(got.rings) == len(want.rings), name
        for i, (a, b) in enumerate(zip(got.rings, want.rings)):
            assert a.shape == b.shape and np.array_equal(a, b), (name, i)


def test_device_tracer_c2_matches_committed_rings(cuda):
    import paper_2404_15217_b200 as pf

    z = np.load(Path(__file__).resolve().parent / "golden" / "c2_polygons.npz")
    for g in range(2):
        shape = tuple(z[f"s{g}_mask_shape"])
        bits = np.unpackbits(z[f"s{g}_mask"])[: shape[0] * shape[1]].reshape(shape)
        got = pf.polygon_from_mask_device(cuda.from_numpy(bits).cuda(), float(z[f"s{g}_scale"][0]))
        want = [z[f"s{g}_ring{r}"] for r in range(int(z[f"s{g}_nrings"][0]))]
        assert len(got.rings) == len(want) and all(np.array_equal(a, b) for a, b in zip(got.rings, want))


def test_device_tracer_empty_masks(cuda):
    import paper_2404_15217_b200 as pf

    with pytest.raises(pf.EmptyForegroundError):
        pf.polygon_from_mask_device(cuda.zeros((20, 30), dtype=cuda.uint8, device="cuda"), 1.0)
    tiny = np.zeros((20, 30), np.uint8)
    tiny[5, 5] = 1  # one pixel: area 0.5 < 64
    with pytest.raises(pf.EmptyForegroundError):
        pf.polygon_from_mask_device(cuda.from_numpy(tiny).cuda(), 1.0)
