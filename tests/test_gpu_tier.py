"""GPU: host-backed tile tier (csrc/pf_tier.cu).  A level-0 slot pool far
smaller than the reachable tile set, refilled a batch ahead from a pinned host store: crops and
regions byte-identical to a dense slide over many batches with evictions, the fault word clean,
and a pool smaller than one batch's tiles reported as a capacity fault."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf(cuda):
    import paper_2404_15217_b200 as pf
    from paper_2404_15217_b200 import multicrop as mc
    from paper_2404_15217_b200 import residency as R
    from paper_2404_15217_b200 import tier as TR

    pf.mc, pf.R, pf.TR = mc, R, TR
    return pf


def _slide_and_poly(pf, seed, sid=None):
    from paper_2404_15217_b200.synthetic import synthetic_slide

    s = synthetic_slide(sid or f"t{seed}", 12000, 9000, seed=seed, blob_px=1500, coverage=0.35, downsample_factor=4)
    thumb, scale = s.thumbnail(32)
    bm = pf.mask_from_saturation(thumb, 0.07, 1, scale=scale)
    return s, bm, pf.polygon_from_mask(bm, slide_id=s.record.slide_id)


def _tiered(pf, seed, frac):
    s, bm, poly = _slide_and_poly(pf, seed)
    plan = pf.R.reachable_tiles(s.record, bm.bits, bm.scale, pf.R.max_footprint(s.record, 224, [(0.25, 1.0), (0.5, 1.0)]))
    n0 = int(plan[0].sum())
    st = pf.TR.tier_level(s, 0, plan[0], hbm_slots=max(1, int(frac * n0)))
    return s, poly, st, n0


def test_tiered_crops_match_dense_with_evictions(pf, cuda):
    torch = cuda
    dense, tiered, states = [], [], []
    for seed in (11, 12):
        d, _, poly = _slide_and_poly(pf, seed)
        t, poly_t, st, n0 = _tiered(pf, seed, 0.3)
        assert st.n_slots < n0
        dense.append((d, poly))
        tiered.append((t, poly_t))
        states.append(st)
    cfg = pf.SamplerConfig(patch_size=224, seed=9, target_mpps=[(0.25, 1.0), (0.5, 1.0)])
    a = pf.mc.MultiCropLoader(dense, cfg, batch_size=48, dtype="u8")
    b = pf.mc.MultiCropLoader(tiered, cfg, batch_size=48, dtype="u8")
    assert b.tiers is not None and a.tiers is None
    for _ in range(16):
        oa, ob = a.next_batch(), b.next_batch()
        torch.cuda.synchronize()
        b.check()  # no capacity fault (pool >= two batches' tiles), no hole read
        assert torch.equal(oa["specs"], ob["specs"])
        assert torch.equal(oa["global_crops"], ob["global_crops"]) and torch.equal(oa["local_crops"], ob["local_crops"])
    b.check()  # no hole read, no capacity fault
    assert sum(s.tiles_filled() for s in states) > 0  # misses were filled from the host store
    # the host drop-in read_region brings its window in first
    rs = np.random.default_rng(3)
    for _ in range(20):
        sp = oa["specs"].cpu().numpy().view(pf._native.SPEC_DTYPE).reshape(-1)[int(rs.integers(0, 48))]
        si = int(sp["slide"])
        rect = (int(sp["x"]), int(sp["y"]), int(sp["width"]), int(sp["height"]))
        assert np.array_equal(tiered[si][0].read_region(rect, float(sp["target_mpp"]), 224),
                              dense[si][0].read_region(rect, float(sp["target_mpp"]), 224))


def test_pool_smaller_than_a_batch_faults(pf, cuda):
    t, poly, st, n0 = _tiered(pf, 13, 0.0)  # a single slot
    cfg = pf.SamplerConfig(patch_size=224, seed=1)
    ld = pf.mc.MultiCropLoader([(t, poly)], cfg, batch_size=64, dtype="u8")
    ld.next_batch()
    with pytest.raises(pf.errors.CapacityError):
        ld.check()


def test_resize_pool_under_a_live_loader(pf, cuda):
    """resize_pool after a loader was built: the loader's tier records follow the new pool."""
    torch = cuda
    d, _, poly = _slide_and_poly(pf, 14)
    t, poly_t, st, n0 = _tiered(pf, 14, 0.3)
    cfg = pf.SamplerConfig(patch_size=224, seed=5, target_mpps=[(0.25, 1.0), (0.5, 1.0)])
    a = pf.mc.MultiCropLoader([(d, poly)], cfg, batch_size=32, dtype="u8")
    b = pf.mc.MultiCropLoader([(t, poly_t)], cfg, batch_size=32, dtype="u8")
    for step in range(8):
        if step == 3:
            pf.TR.resize_pool(t, int(0.5 * n0))
            assert st.n_slots == int(0.5 * n0)
        oa, ob = a.next_batch(), b.next_batch()
        torch.cuda.synchronize()
        b.check()
        assert torch.equal(oa["global_crops"], ob["global_crops"]) and torch.equal(oa["local_crops"], ob["local_crops"])


@pytest.mark.parametrize("case", range(3))
def test_random_pools_and_batches_match_dense(pf, cuda, case):
    """Random pool fractions, batch sizes and sampler seeds over many batches (evictions every
    step): crops byte-identical to the dense slides and no fault."""
    torch = cuda
    rs = np.random.default_rng(40 + case)
    seed = int(rs.integers(20, 1000))
    d, _, poly = _slide_and_poly(pf, seed, sid=f"d{seed}")
    t, poly_t, st, n0 = _tiered(pf, seed, float(rs.uniform(0.3, 0.6)))
    batch = int(rs.choice([16, 32, 48]))
    cfg = pf.SamplerConfig(patch_size=224, seed=int(rs.integers(0, 1 << 20)), target_mpps=[(0.25, 1.0), (0.5, 1.0)])
    a = pf.mc.MultiCropLoader([(d, poly)], cfg, batch_size=batch, dtype="u8")
    b = pf.mc.MultiCropLoader([(t, poly_t)], cfg, batch_size=batch, dtype="u8")
    for _ in range(10):
        oa, ob = a.next_batch(), b.next_batch()
        torch.cuda.synchronize()
        assert torch.equal(oa["global_crops"], ob["global_crops"]) and torch.equal(oa["local_crops"], ob["local_crops"])
    b.check()
    assert st.tiles_filled() > 0
