"""BASELINE configs[1] at full size (40000 x 30000 slides, batch 1024): sampled oracle parity
where the oracle finishes in seconds, size-independent properties everywhere else.

* pyramid / thumbnail: every sampled level-1 tile and thumbnail block equals the oracle's
  _box_downsample (pkg/store.py:429-441) of the device's own level-0 pixels;
* sampler: the first specs of the full-size stream equal oracle/port.epoch_stream on the
  traced polygons (FP64 lattice at coordinates up to 40000); the stream does not depend on
  how it is split into batches; every spec of a 1024 batch meets min_foreground on the
  device and, for a sample, in the oracle;
* read_region (configs 1 and 3): sampled specs of a mixed-mpp batch (0.25 mpp passthrough,
  0.5 mpp PIL-bilinear resample) against port.read_region on the device's level-0 pixels,
  u8 bit-exact and the normalised f32 bit-exact;
* multi-crop: sampled patches of a 1024-patch batch against torchvision on the raw level-0
  window (<= 1 LSB, the small-size bar); the batch split and a repeated launch give
  bit-identical crops (checksum of per-patch checksums).
"""

import numpy as np
import pytest

from oracle import augment as A
from oracle import port

pytestmark = pytest.mark.gpu

W, H = 40000, 30000
SEED = 5


@pytest.fixture(scope="module")
def pf(cuda):
    import paper_2404_15217_b200 as pf
    from paper_2404_15217_b200 import multicrop as mc

    pf.mc = mc
    return pf


@pytest.fixture(scope="module")
def c2(pf):
    """Two BASELINE C2 slides: render, saturation mask on the 1/32 thumbnail, trace."""
    from paper_2404_15217_b200.synthetic import synthetic_slide

    out = []
    for gi in range(2):
        for k in range(8):  # redraw tissue whose traced rings have negative total area (as bench.py)
            s = synthetic_slide(f"s{gi}", W, H, seed=1000 + gi + 100_000 * k, downsample_factor=4)
            thumb, scale = s.thumbnail_device(32)
            mask = pf.foreground.mask_device(thumb, 1, 0.07, 1)
            bm = pf.BinaryMask(mask.cpu().numpy().astype(bool), scale)
            try:
                poly = pf.polygon_from_mask(bm, slide_id=f"s{gi}")
                break
            except ValueError:
                del s
        out.append((s, poly))
    return out


def _region(slide, level, x0, y0, w, h):
    """Raw pixels [y0, y0+h) x [x0, x0+w) of a dense level, straight from the tile storage."""
    T = slide.record.tile_size
    lv = slide.levels[level]
    tx0, ty0, tx1, ty1 = x0 // T, y0 // T, (x0 + w - 1) // T + 1, (y0 + h - 1) // T + 1
    blk = lv[ty0:ty1, tx0:tx1].permute(0, 2, 1, 3, 4).reshape((ty1 - ty0) * T, (tx1 - tx0) * T, 3)
    return blk[y0 - ty0 * T:y0 - ty0 * T + h, x0 - tx0 * T:x0 - tx0 * T + w].cpu().numpy()


def test_pyramid_and_thumbnail_are_box_downsamples(pf, c2):
    rs = np.random.default_rng(0)
    for s, _ in c2:
        rec = s.record
        assert (rec.levels[0].width, rec.levels[0].height) == (W, H)
        nx1, ny1 = rec.tile_grid(1)
        for _ in range(6):  # interior level-1 tiles: 4x4 level-0 tiles each
            tx, ty = int(rs.integers(0, nx1 - 1)), int(rs.integers(0, ny1 - 1))
            src = _region(s, 0, tx * 1024, ty * 1024, 1024, 1024)
            assert np.array_equal(_region(s, 1, tx * 256, ty * 256, 256, 256), port.box_downsample(src, 4))
        thumb, _ = s.thumbnail_device(32)
        thumb = thumb.cpu().numpy()
        for _ in range(6):  # 8 x 8 thumbnail blocks = 256 x 256 level-0 px
            u, v = int(rs.integers(0, W // 32 - 8)), int(rs.integers(0, H // 32 - 8))
            src = _region(s, 0, u * 32, v * 32, 256, 256)
            assert np.array_equal(thumb[v:v + 8, u:u + 8], port.box_downsample(src, 32))


def _oracle_slides(c2):
    return [{"id": s.record.slide_id, "width": W, "height": H, "base_mpp": 0.25, "rings": p.rings} for s, p in c2]


@pytest.fixture()
def chunked_oracle(monkeypatch):
    """port.points_in_polygon over point chunks (per-point results are independent of the
    chunking): the full-size lattice x 10^4 edges would not fit in host memory at once."""
    whole = port.points_in_polygon

    def chunked(points, rings):
        pts = np.asarray(points, dtype=np.float64)
        return np.concatenate([whole(pts[i:i + 1024], rings) for i in range(0, len(pts), 1024)])

    monkeypatch.setattr(port, "points_in_polygon", chunked)


def _sampler_cfg(pf):
    return pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=[(0.25, 1.0)], seed=SEED)


def test_full_size_stream_matches_reference_golden(pf, c2):
    """The first 256 specs of the full-size C2 stream equal the REAL reference's epoch_stream
    (tests/golden/make_c2_stream_golden.py: patchforge run offline on the committed masks of
    these two slides, after checking its polygon_from_mask gives the committed rings).  The
    slides rendered here must trace to those rings, and the GPU sampler run on the committed
    rings (records only, no pixels) must reproduce the reference stream spec for spec."""
    import json
    from pathlib import Path

    gold = Path(__file__).resolve().parent / "golden"
    z = np.load(gold / "c2_polygons.npz")
    want = json.loads((gold / "c2_stream_golden.json").read_text())
    rings = [[z[f"s{g}_ring{r}"] for r in range(int(z[f"s{g}_nrings"][0]))] for g in range(2)]
    for (s, poly), rr in zip(c2, rings):  # this box's render traces to the committed rings
        assert len(poly.rings) == len(rr) and all(np.array_equal(a, b) for a, b in zip(poly.rings, rr))
    smp = pf.GpuSampler(_sampler_cfg(pf), c2)
    got = smp.to_patch_specs(smp.next_batch(len(want["specs"])))
    assert [json.loads(g.to_json_line()) for g in got] == want["specs"]
    # batch-split invariance against the same golden
    smp2 = pf.GpuSampler(_sampler_cfg(pf), c2)
    parts = []
    for k in (7, 100, 1, 148):
        parts += smp2.to_patch_specs(smp2.next_batch(k))
    assert [json.loads(g.to_json_line()) for g in parts] == want["specs"]


def test_full_size_stream_is_batch_split_invariant_and_admissible(pf, c2, chunked_oracle):
    torch = pytest.importorskip("torch")
    a = pf.GpuSampler(_sampler_cfg(pf), c2).next_batch(1024)
    b_smp = pf.GpuSampler(_sampler_cfg(pf), c2)
    b = torch.cat([b_smp.next_batch(n) for n in (100, 412, 1, 511)])
    assert torch.equal(a, b)
    specs = pf.GpuSampler(_sampler_cfg(pf), c2).to_patch_specs(a)
    assert [s.seq for s in specs] == list(range(1024))
    by_slide = {s.record.slide_id: (s, p) for s, p in c2}
    for sid, (s, poly) in by_slide.items():
        rects = np.array([(sp.x, sp.y, sp.width, sp.height) for sp in specs if sp.slide_id == sid], np.float64)
        assert len(rects) > 300  # both slides drawn (uniform slide choice)
        fr = pf.foreground.overlap_fractions(poly, rects).cpu().numpy()
        assert np.all(fr >= 0.40)
        for r, f in zip(rects[:2], fr[:2]):  # the oracle on a sample: same FP64 fraction
            assert port.overlap_fraction(poly.rings, tuple(r), 128) == f


def test_full_size_read_regions_mixed_mpp(pf, c2):
    ss = pf.SlideSet([s for s, _ in c2])
    cfg = pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=[(0.25, 1.0), (0.5, 1.0)], seed=SEED)
    smp = pf.GpuSampler(cfg, c2, slide_set=ss)
    specs = smp.next_batch(256)
    mean, std = pf.IMAGENET_MEAN, pf.IMAGENET_STD
    u8 = ss.read_regions(specs, 224).cpu().numpy()
    f32 = ss.read_regions(specs, 224, dtype="f32", mean=mean, std=std).cpu().numpy()
    hs = smp.to_patch_specs(specs)
    slides = {s.record.slide_id: s for s, _ in c2}
    picked = [i for i in range(256) if hs[i].target_mpp == 0.25][:32] + [i for i in range(256) if hs[i].target_mpp == 0.5][:32]
    assert len(picked) == 64
    for i in picked:
        sp = hs[i]
        s = slides[sp.slide_id]
        x0, y0 = max(0, sp.x - 2), max(0, sp.y - 2)
        crop = _region(s, 0, x0, y0, min(W, sp.x + sp.width + 2) - x0, min(H, sp.y + sp.height + 2) - y0)
        mpps = [lv.mpp for lv in s.record.levels]
        want = port.read_region([crop], mpps, [1.0] * len(mpps), (sp.x - x0, sp.y - y0, sp.width, sp.height),
                                sp.target_mpp, 224)
        assert np.array_equal(u8[i], want), (i, sp)
        assert np.array_equal(f32[i], port.normalize_patch(want, mean, std))


def test_full_size_mixed_mpp_multicrop_vs_torchvision(pf, c2):
    """C3 at full size: 0.5-mpp specs are PIL-resampled 448 -> 224 (resample2x_kernel) and cut by
    the multi-crop from that buffer; both stages against their oracles for 48 patches."""
    torch = pytest.importorskip("torch")
    ss = pf.SlideSet([s for s, _ in c2])
    cfg = pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=[(0.25, 1.0), (0.5, 1.0)], seed=SEED + 1)
    smp = pf.GpuSampler(cfg, c2, slide_set=ss)
    specs = smp.next_batch(256)
    mc = pf.mc.MultiCropConfig()
    params = pf.mc.crop_params(mc, 256, seed=11, step=2)
    src = ss.read_regions(specs, 224, planned=True)
    g, l = pf.mc.multicrop(ss, specs, params, mc, dtype="u8", src_hwc=src)
    torch.cuda.synchronize()
    hs, prm = smp.to_patch_specs(specs), pf.mc.params_host(params)
    g, l, srcs = g.cpu().numpy(), l.cpu().numpy(), src.cpu().numpy()
    slides = {s.record.slide_id: s for s, _ in c2}
    picked = [i for i in range(256) if hs[i].target_mpp == 0.5][:24] + [i for i in range(256) if hs[i].target_mpp == 0.25][:24]
    for i in picked:
        sp = hs[i]
        s = slides[sp.slide_id]
        x0, y0 = max(0, sp.x - 2), max(0, sp.y - 2)
        crop = _region(s, 0, x0, y0, min(W, sp.x + sp.width + 2) - x0, min(H, sp.y + sp.height + 2) - y0)
        mpps = [lv.mpp for lv in s.record.levels]
        want_src = port.read_region([crop], mpps, [1.0] * len(mpps), (sp.x - x0, sp.y - y0, sp.width, sp.height),
                                    sp.target_mpp, 224)
        if sp.target_mpp == 0.5:
            assert np.array_equal(srcs[i], want_src), i
        for c in range(mc.n_crops):
            want = A.torchvision_crop(want_src, prm[i, c])
            got = (g[c, i] if c < mc.n_global else l[c - mc.n_global, i]).transpose(1, 2, 0)
            assert np.abs(got.astype(int) - want.astype(int)).max() <= 1, (i, c)


@pytest.fixture(scope="module")
def batch(pf, c2):
    torch = pytest.importorskip("torch")
    ss = pf.SlideSet([s for s, _ in c2])
    smp = pf.GpuSampler(_sampler_cfg(pf), c2, slide_set=ss)
    specs = smp.next_batch(1024)
    cfg = pf.mc.MultiCropConfig()
    params = pf.mc.crop_params(cfg, 1024, seed=3, step=0)
    g, l = pf.mc.multicrop(ss, specs, params, cfg, dtype="u8")
    torch.cuda.synchronize()
    return ss, smp, specs, cfg, params, g, l


def test_full_batch_sampled_patches_vs_torchvision(pf, c2, batch):
    ss, smp, specs, cfg, params, g, l = batch
    hs = smp.to_patch_specs(specs)
    prm = pf.mc.params_host(params)
    slides = {s.record.slide_id: s for s, _ in c2}
    g, l = g.cpu().numpy(), l.cpu().numpy()
    diff, total = 0, 0
    for i in np.random.default_rng(1).choice(1024, 128, replace=False):  # 1280 crops vs torchvision
        sp = hs[i]
        src = _region(slides[sp.slide_id], 0, sp.x, sp.y, 224, 224)  # C2: 0.25 mpp = level 0, no resample
        for c in range(cfg.n_crops):
            want = A.torchvision_crop(src, prm[i, c])
            got = (g[c, i] if c < cfg.n_global else l[c - cfg.n_global, i]).transpose(1, 2, 0)
            d = np.abs(got.astype(int) - want.astype(int))
            assert d.max() <= 1, (i, c)
            diff += int((d > 0).sum())
            total += d.size
    assert diff / total < 1e-3


def _checksums(torch, g, l):
    """Per-patch checksums of every crop -> one checksum of checksums per patch."""
    def per_patch(t):
        n = t.shape[1]
        v = t.permute(1, 0, 2, 3, 4).reshape(n, -1).to(torch.int64)
        w = torch.arange(1, v.shape[1] + 1, device=v.device, dtype=torch.int64) % 65521
        return (v * w).sum(1)
    return per_patch(g) * 1_000_003 + per_patch(l)


def test_full_batch_split_and_repeat_are_bit_identical(pf, batch):
    torch = pytest.importorskip("torch")
    ss, smp, specs, cfg, params, g, l = batch
    ref = _checksums(torch, g, l)
    g2, l2 = pf.mc.multicrop(ss, specs, params, cfg, dtype="u8")
    assert torch.equal(_checksums(torch, g2, l2), ref)
    parts = []
    for a, b in ((0, 300), (300, 301), (301, 1024)):
        ga, la = pf.mc.multicrop(ss, specs[a:b].contiguous(), params[a:b].contiguous(), cfg, dtype="u8")
        parts.append(_checksums(torch, ga, la))
    assert torch.equal(torch.cat(parts), ref)
    assert torch.equal(g2, g) and torch.equal(l2, l)


def test_config4_size_slide_compacted_matches_dense(pf):
    """BASELINE configs[3] (residency): a 70000 x 55000 slide (the C4 mean size) compacted to its
    reachable tiles serves a 1024-spec batch with the dense pyramid's bytes (crops and regions)."""
    torch = pytest.importorskip("torch")
    from paper_2404_15217_b200 import residency as R
    from paper_2404_15217_b200.synthetic import synthetic_slide

    s = synthetic_slide("c4", 70000, 55000, seed=4, downsample_factor=4)
    thumb, scale = s.thumbnail_device(32)
    bm = pf.BinaryMask(pf.foreground.mask_device(thumb, 1, 0.07, 1).cpu().numpy().astype(bool), scale)
    poly = pf.polygon_from_mask(bm, slide_id="c4")
    mpps = [(0.25, 1.0), (0.5, 1.0)]
    cfg = pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=mpps, seed=SEED)
    ss = pf.SlideSet([s])
    specs = pf.GpuSampler(cfg, [(s, poly)], slide_set=ss).next_batch(1024)
    mc = pf.mc.MultiCropConfig()
    params = pf.mc.crop_params(mc, 1024, seed=4)
    src = ss.read_regions(specs, 224)
    g0, l0 = pf.mc.multicrop(ss, specs, params, mc, dtype="bf16", src_hwc=src)
    plan = R.reachable_tiles(s.record, bm.bits, scale, R.max_footprint(s.record, 224, mpps))
    dense = R.dense_bytes(s.record)
    s.compact(plan)
    torch.cuda.empty_cache()
    assert R.resident_bytes(s.record, plan) < 0.9 * dense
    ss2 = pf.SlideSet([s])
    src2 = ss2.read_regions(specs, 224)
    g1, l1 = pf.mc.multicrop(ss2, specs, params, mc, dtype="bf16", src_hwc=src2)
    assert torch.equal(src, src2) and torch.equal(g0, g1) and torch.equal(l0, l1)
