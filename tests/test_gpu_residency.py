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
    ss = pf.SlideSet([s])
    ss.check_status()  # clean so far
    px = ss.read_regions(specs, 64)  # the batched device path reads the zero hole ...
    assert px.shape == (1, 64, 64, 3) and not px.any()
    with pytest.raises(pf.OutOfBoundsError):  # ... and the fault word reports it (pf_slide_status)
        ss.check_status()
    ss.check_status()  # cleared by the check
    with pytest.raises(ValueError):
        s.level_array(0)


def test_multicrop_hole_read_fails_loudly(pf):
    """A multi-crop over specs whose windows reach non-resident tiles raises at check()."""
    torch = pytest.importorskip("torch")
    s, bm, poly = _slide_and_poly(pf, 4)
    plan = pf.R.reachable_tiles(s.record, bm.bits, bm.scale, 224.0)
    cfg = pf.SamplerConfig(patch_size=224, seed=1)
    loader = pf.mc.MultiCropLoader([(s, poly)], cfg, batch_size=32, dtype="u8")
    loader.next_batch()
    loader.check()  # dense slide: no fault
    # shrink the plan to one level-0 tile: every sampled window now reads holes
    keep = [np.zeros_like(p) for p in plan]
    keep[0][np.argwhere(plan[0])[0][0], np.argwhere(plan[0])[0][1]] = True
    for li in range(1, len(keep)):
        keep[li] = plan[li]
    s.compact(keep)  # refreshes the loader's descriptors (SlideSet built before compact)
    loader.next_batch()
    torch.cuda.synchronize()
    with pytest.raises(pf.OutOfBoundsError):
        loader.check()


def test_compact_refreshes_earlier_slide_sets(pf):
    """SlideSets (and the samplers sharing their descriptor tensor) built before compact() read
    the compacted slots, never the freed dense level."""
    torch = pytest.importorskip("torch")
    s, bm, poly = _slide_and_poly(pf, 3)
    ref, _, _ = _slide_and_poly(pf, 3)
    early = pf.SlideSet([s])
    plan = pf.R.reachable_tiles(s.record, bm.bits, bm.scale, 224.0)
    smp = pf.GpuSampler(pf.SamplerConfig(patch_size=224, seed=2), [(ref, poly)])
    specs = smp.next_batch(64)
    s.compact(plan)
    torch.cuda.empty_cache()
    junk = torch.full((1 << 28,), 77, dtype=torch.uint8, device="cuda")  # reuse the freed blocks
    got = early.read_regions(specs, 224)
    want = pf.SlideSet([ref]).read_regions(specs, 224)
    del junk
    assert torch.equal(got, want)
    early.check_status()


def test_library_owned_slide_handle(pf, golden_arrays):
    """pf_slide_create / upload_level0 / get_desc / destroy: a torch-free caller's slide reads
    exactly what GpuSlide.from_array reads (levels box-filtered on device)."""
    import ctypes as C

    torch = pytest.importorskip("torch")
    N = pf._native
    img = golden_arrays["synthetic_700x500"]
    L = N.lib()
    h = C.c_void_p()
    N.check(L.pf_slide_create(700, 500, 0.25, 128, 2, C.byref(h)), "pf_slide_create")
    try:
        N.check(L.pf_slide_upload_level0(h, np.ascontiguousarray(img).ctypes.data, 0, 1, None), "upload")
        d = N.SlideDesc()
        N.check(L.pf_slide_get_desc(h, C.byref(d)), "pf_slide_get_desc")
        ref = pf.GpuSlide.from_array(img, "s0", 0.25, tile_size=128, downsample_factor=2)
        assert [d.width[i] for i in range(d.n_levels)] == [lv.width for lv in ref.record.levels]
        descs = torch.frombuffer(bytearray(bytes(d)), dtype=torch.uint8).cuda()
        reqs = [(0, (10, 20, 128, 128), 0.25, 128), (0, (40, 33, 124, 124), 0.97, 32), (0, (0, 0, 496, 496), 2.0, 62)]
        for r in reqs:
            spec = pf.store.plan_specs([r], [ref.record])
            dspec = torch.from_numpy(spec.view(np.uint8).reshape(1, 64)).cuda()
            out = torch.empty((1, r[3], r[3], 3), dtype=torch.uint8, device="cuda")
            m = (C.c_float * 3)(0.5, 0.5, 0.5)
            N.check(L.pf_plan_regions(descs.data_ptr(), dspec.data_ptr(), 1, None), "plan")
            N.check(L.pf_read_regions(descs.data_ptr(), dspec.data_ptr(), 1, r[3], N.PF_U8, N.PF_HWC,
                                      C.cast(m, C.c_void_p), C.cast(m, C.c_void_p), out.data_ptr(), None), "read")
            torch.cuda.synchronize()
            assert np.array_equal(out[0].cpu().numpy(), ref.read_region(r[1], r[2], r[3]))
        assert L.pf_slide_status(C.byref(d), 1, None) == 0
    finally:
        assert L.pf_slide_destroy(h) == 0
