"""GPU: randomized differential test of the device sampler against the CPU oracle's
epoch_stream (oracle/port.py, pinned to the reference by tests/test_oracle.py).

Each case draws a sampler configuration (patch size, min_foreground, target mpps, uniform or
weighted slides, max_attempts from 1 to 100) and a device schedule (speculation window and
rounds, raster on or off, the stream cut into random batch sizes), on the reference golden
slides, with a 32x32 overlap lattice on both sides (the oracle's numpy lattice at the
reference's 128 costs ~1 min per case; the walk logic under test does not depend on it).
The specs -- or the NoSamplableSlideError -- must be the oracle's."""

import os

import numpy as np
import pytest

from oracle import port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf(cuda):
    import paper_2404_15217_b200 as pf

    return pf


def _slides(pf, goldens):
    out = []
    for i in range(3):
        w, h = goldens[f"sampler_dims_b{i}"]
        rec = pf.store.make_record(f"b{i}", w, h, 0.25, tile_size=128, downsample_factor=2)
        out.append((rec, pf.ForegroundPolygon.from_json_dict(goldens[f"sampler_poly_b{i}"])))
    return out


@pytest.mark.parametrize("case", range(int(os.environ.get("PF_FUZZ_CASES", "12"))))
def test_random_schedule_matches_oracle(pf, goldens, case):
    rs = np.random.default_rng(1000 + case)
    slides = _slides(pf, goldens)
    patch = int(rs.choice([24, 32, 48]))
    min_fg = float(rs.choice([0.2, 0.4, 0.7, 0.9]))
    pool = [(0.25, 1.0), (0.5, 1.0), (1.0, 2.0)]
    mpps = [pool[i] for i in sorted(rs.choice(3, size=int(rs.integers(1, 4)), replace=False))]
    max_att = int(rs.choice([1, 2, 3, 8, 100]))
    weighted = bool(rs.integers(0, 2))
    weights = {f"b{i}": float(rs.choice([0.0, 1.0, 2.5])) for i in range(3)} if weighted else None
    if weighted and sum(weights.values()) == 0:
        weights["b1"] = 1.0
    n_total = 150
    seed = int(rs.integers(0, 1 << 30))
    cfg = pf.SamplerConfig(patch_size=patch, min_foreground=min_fg, target_mpps=mpps, seed=seed,
                           max_attempts_per_slide=max_att, slide_strategy="weighted" if weighted else "uniform",
                           slide_weights=weights)
    orc = [{"id": r.slide_id, "width": r.width, "height": r.height, "base_mpp": 0.25, "rings": p.rings}
           for r, p in slides]
    try:
        want, _ = port.epoch_stream(orc, patch_size=patch, min_fg=min_fg, mpps=mpps, seed=seed, epoch_size=n_total,
                                    max_attempts=max_att, strategy="weighted" if weighted else "uniform",
                                    weights=weights, grid=32)
        raises = False
    except RuntimeError:
        raises = True
    window = None if rs.integers(0, 2) else int(rs.integers(1, 64)) * 32
    rounds = int(rs.choice([0, 1, 2, 3]))
    smp = pf.GpuSampler(cfg, slides, window=window, rounds=rounds, raster=bool(rs.integers(0, 2)), grid=32)
    sizes = []
    while sum(sizes) < n_total:
        sizes.append(int(min(n_total - sum(sizes), rs.integers(1, 80))))
    got = []
    if raises:
        with pytest.raises(pf.NoSamplableSlideError):
            for k in sizes:
                got += smp.to_patch_specs(smp.next_batch(k))
                smp.check()
        return
    for k in sizes:
        got += smp.to_patch_specs(smp.next_batch(k))
    smp.check()
    assert [(s.slide_id, s.x, s.y, s.width, s.target_mpp, s.seq) for s in got] == \
        [(orc[si]["id"], x, y, fp, m, q) for si, x, y, fp, m, q in want], \
        dict(patch=patch, min_fg=min_fg, mpps=mpps, max_att=max_att, weights=weights, window=window, rounds=rounds)
