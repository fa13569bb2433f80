"""GPU: slides compacted to their reachable tiles (pf_slide_desc.tile_map) serve the sampler's
windows with exactly the bytes of the dense pyramid (multi-crop, read_region at two mpps), and
non-resident tiles read as the zero hole."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf(cuda):
    import paper_2404_15217_b200 as pf
    from paper_2404_15217_b200 import multicrop as mc
    from paper_2404_15217_b200 import residency as R

    pf.mc, pf.R = mc, R
    return pf


def _slide_and_poly(pf, seed):
    from paper_2404_15217_b200.synthetic import synthetic_slide

    s = synthetic_slide(f"r{seed}", 9000, 6400, seed=seed, blob_px=1500, coverage=0.2, downsample_factor=4)
    thumb, scale = s.thumbnail(32)
    bm = pf.mask_from_saturation(thumb, 0.07, 1, scale=scale)
    return s, bm, pf.polygon_from_mask(bm, slide_id=s.record.slide_id)


def test_compacted_slides_match_dense(pf):
    torch = pytest.importorskip("torch")
    dense, compact = [], []
    for seed in (3, 4):
        s, bm, poly = _slide_and_poly(pf, seed)
        c, _, _ = _slide_and_poly(pf, seed)
        plan = pf.R.reachable_tiles(c.record, bm.bits, bm.scale, pf.R.max_footprint(c.record, 224, [(0.25, 1.0), (0.5, 1.0)]))
        frac = sum(int(p.sum()) for p in plan) / sum(p.size for p in plan)
        assert 0.1 < frac < 0.97, frac
        c.compact(plan)
        assert c.compacted and c.desc.tile_map[0] != 0
        dense.append((s, poly))
        compact.append((c, poly))
    cfg = pf.SamplerConfig(patch_size=224, seed=5, target_mpps=[(0.25, 1.0), (0.5, 1.0)])
    a = pf.mc.MultiCropLoader(dense, cfg, batch_size=96, dtype="u8")
    b = pf.mc.MultiCropLoader(compact, cfg, batch_size=96, dtype="u8")
    for _ in range(3):
        oa, ob = a.next_batch(), b.next_batch()
        torch.cuda.synchronize()
        assert torch.equal(oa["specs"], ob["specs"])
        assert torch.equal(oa["global_crops"], ob["global_crops"]) and torch.equal(oa["local_crops"], ob["local_crops"])
        ra = a.slide_set.read_regions(oa["specs"], 224)
        rb = b.slide_set.read_regions(ob["specs"], 224)
        assert torch.equal(ra, rb)


def test_non_resident_tiles_read_as_hole(pf):
    s, bm, _ = _slide_and_poly(pf, 3)
    plan = pf.R.reachable_tiles(s.record, bm.bits, bm.scale, 224.0)
    T = s.record.tile_size
    ty, tx = np.argwhere(~plan[0])[0]
    s.compact(plan)
    with pytest.raises(pf.StoreError):  # the host drop-in refuses non-resident windows
        s.read_region((int(tx) * T + 8, int(ty) * T + 8, 64, 64), 0.25, 64)
    specs = pf.store.plan_specs([(0, (int(tx) * T + 8, int(ty) * T + 8, 64, 64), 0.25, 64)], [s.record])
    px = pf.SlideSet([s]).read_regions(specs, 64)  # the batched device path reads the zero hole
    assert px.shape == (1, 64, 64, 3) and not px.any()
    with pytest.raises(ValueError):
        s.level_array(0)
