"""GPU parity: pyramid build, thumbnails, read_region (gather + PIL resample) and normalisation
against the oracle and the reference goldens.  Bit-exact (integer / byte work)."""

import os

import numpy as np
import pytest

from oracle import port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf(cuda):
    import paper_2404_15217_b200 as pf

    return pf


def test_pyramid_and_thumbnail_match_reference(pf, goldens, golden_arrays):
    img = golden_arrays["synthetic_700x500"]
    s = pf.GpuSlide.from_array(img, "s0", 0.25, tile_size=128, downsample_factor=2)
    assert [(lv.width, lv.height, lv.mpp, lv.downsample) for lv in s.record.levels] == [tuple(x) for x in goldens["levels_f2_t128"]]
    for li in range(len(s.record.levels)):
        assert np.array_equal(s.level_array(li).cpu().numpy(), golden_arrays[f"level_f2_{li}"]), li
    th, sc = s.thumbnail()
    assert np.array_equal(th, golden_arrays["thumb_f2"]) and sc == goldens["thumb_f2_scale"]
    t32, sc32 = s.thumbnail(32)
    assert np.array_equal(t32, golden_arrays["box32_700x500"]) and sc32 == 1 / 32
    t7, _ = s.thumbnail(7)
    assert np.array_equal(t7, golden_arrays["box7_700x500"])
    s4 = pf.GpuSlide.from_array(img, "s1", 0.25, tile_size=64, downsample_factor=4)
    assert np.array_equal(s4.level_array(1).cpu().numpy(), golden_arrays["level_f4_1"])


def test_box32_fast_path_large(pf):
    rs = np.random.default_rng(0)
    img = rs.integers(0, 256, size=(1000, 1333, 3), dtype=np.uint8)
    s = pf.GpuSlide.from_array(img, "big", 0.25, tile_size=256, downsample_factor=4)
    t, _ = s.thumbnail(32)
    assert np.array_equal(t, port.box_downsample(img, 32))
    for li, want in enumerate(port.pyramid(img, 256, 4)):
        assert np.array_equal(s.level_array(li).cpu().numpy(), want)


def test_read_region_matches_reference(pf, goldens, golden_arrays):
    img = golden_arrays["synthetic_700x500"]
    s = pf.GpuSlide.from_array(img, "s0", 0.25, tile_size=128, downsample_factor=2)
    for r in goldens["reads"]:
        got = s.read_region(tuple(r["rect"]), r["mpp"], r["out"])
        assert np.array_equal(got, golden_arrays[f"read_{r['k']}"]), r


def test_read_regions_batched_all_layouts(pf, goldens, golden_arrays, cuda):
    torch = cuda
    img = golden_arrays["synthetic_700x500"]
    s = pf.GpuSlide.from_array(img, "s0", 0.25, tile_size=128, downsample_factor=2)
    ss = pf.SlideSet([s])
    reads = [r for r in goldens["reads"] if r["out"] == 32]
    specs = pf.store.plan_specs([(0, r["rect"], r["mpp"], 32) for r in reads], ss.records)
    want = np.stack([golden_arrays[f"read_{r['k']}"] for r in reads])
    hwc = ss.read_regions(specs, 32).cpu().numpy()
    assert np.array_equal(hwc, want)
    nchw = ss.read_regions(specs, 32, layout="nchw").cpu().numpy()
    assert np.array_equal(nchw, want.transpose(0, 3, 1, 2))
    f32 = ss.read_regions(specs, 32, dtype="f32", layout="nchw").cpu().numpy()
    assert np.array_equal(f32, port.normalize_patch(want).transpose(0, 3, 1, 2))  # bit-exact FP32
    mean, std = pf.IMAGENET_MEAN, pf.IMAGENET_STD
    f32i = ss.read_regions(specs, 32, dtype="f32", layout="nchw", mean=mean, std=std).cpu().numpy()
    assert np.array_equal(f32i, port.normalize_patch(want, mean, std).transpose(0, 3, 1, 2))
    b16 = ss.read_regions(specs, 32, dtype="bf16", layout="nchw", mean=mean, std=std)
    ref16 = torch.from_numpy(port.normalize_patch(want, mean, std).transpose(0, 3, 1, 2).copy()).to(torch.bfloat16)
    assert torch.equal(b16.cpu(), ref16)


def test_edge_replication_and_bounds(pf):
    rs = np.random.default_rng(3)
    img = rs.integers(0, 256, size=(301, 257, 3), dtype=np.uint8)
    s = pf.GpuSlide.from_array(img, "e", 0.25, tile_size=64, downsample_factor=2)
    lv = port.pyramid(img, 64, 2)
    mpps = [lv_.mpp for lv_ in s.record.levels]
    ds = [lv_.downsample for lv_ in s.record.levels]
    # windows at the far edges at coarse levels overrun by the 1-px slack
    for rect, mpp, out in [((256, 300, 1, 1), 0.5, 3), ((250, 290, 7, 11), 1.0, 5), ((0, 0, 257, 301), 2.0, 32),
                           ((255, 299, 2, 2), 4.0, 2), ((254, 298, 3, 3), 0.5, 3), ((252, 296, 5, 5), 2.0, 1), ((3, 5, 200, 200), 0.25, 200), ((0, 0, 4, 4), 8.0, 9)]:
        try:
            want = port.read_region(lv, mpps, ds, rect, mpp, out)
        except IndexError:  # the reference's _read_window slack rule rejects it too
            with pytest.raises(pf.OutOfBoundsError):
                s.read_region(rect, mpp, out)
            continue
        assert np.array_equal(s.read_region(rect, mpp, out), want), (rect, mpp, out)
    with pytest.raises(pf.OutOfBoundsError):
        s.read_region((250, 0, 10, 10), 0.25, 10)
    with pytest.raises(pf.OutOfBoundsError):
        s.read_region((0, 0, 0, 10), 0.25, 10)
    with pytest.raises(ValueError):
        s.read_region((0, 0, 10, 10), 0.25, 0)


def test_normalize_patch_kats(pf, goldens):
    v = pf.normalize_patch(np.array([[0, 255, 128], [1, 254, 7]], np.uint8).reshape(1, 2, 3))
    assert v.reshape(-1)[:3].tolist() == goldens["normalize"][:3]
    assert v.reshape(-1)[3:5].tolist() == goldens["normalize"][3:5]


def test_store_roundtrip_from_reference_format(pf, tmp_path, golden_arrays):
    """A store written in the reference on-disk format (raw, packed) loads into HBM byte-exactly."""
    import json

    img = golden_arrays["synthetic_700x500"]
    levels = port.pyramid(img, 128, 4)
    root = tmp_path / "store"
    (root / "chunks").mkdir(parents=True)
    (root / "slides").mkdir()
    chunks, off, blob = {}, 0, bytearray()
    for li, a in enumerate(levels):
        ny, nx = -(-a.shape[0] // 128), -(-a.shape[1] // 128)
        for ty in range(ny):
            for tx in range(nx):
                t = np.ascontiguousarray(a[ty * 128:(ty + 1) * 128, tx * 128:(tx + 1) * 128]).tobytes()
                chunks[f"{li}/{tx}_{ty}"] = {"kind": "byte-range", "path": "chunks/s.bin", "codec": "raw", "offset": off,
                                             "length": len(t)}
                blob += t
                off += len(t)
    (root / "chunks" / "s.bin").write_bytes(bytes(blob))
    rec = {"slide_id": "s", "base_mpp": 0.25, "tile_size": 128, "chunks": chunks,
           "levels": [{"width_px": a.shape[1], "height_px": a.shape[0], "mpp": 0.25 * 4**i, "downsample": 4**i}
                      for i, a in enumerate(levels)]}
    (root / "slides" / "s.json").write_text(json.dumps(rec))
    (root / "index.json").write_text(json.dumps({"format_version": 1, "slides": ["s"], "records": {"s": "slides/s.json"}}))
    s = pf.GpuSlide.from_store(root, "s")
    for li, a in enumerate(levels):
        assert np.array_equal(s.level_array(li).cpu().numpy(), a)
    with pytest.raises(pf.SlideNotFoundError):
        pf.GpuSlide.from_store(root, "nope")


@pytest.mark.parametrize("codec,layout", [("raw", "packed"), ("png", "files"), ("jpeg", "packed")])
def test_ingest_image_writes_the_reference_store(cuda, golden_arrays, goldens, tmp_path, codec, layout):
    """ingest_image with the GPU pyramid writes byte-identical files (tiles, record, index) to the
    reference's ingest_image on the same image (sha256 of every file)."""
    import hashlib

    import paper_2404_15217_b200 as pf

    img = golden_arrays["synthetic_700x500"]
    rec, slide = pf.store.ingest_image(img, "s0", 0.25, tmp_path, tile_size=128, downsample_factor=2, codec=codec,
                                       layout=layout, return_slide=True)
    got = {str(p.relative_to(tmp_path)): hashlib.sha256(p.read_bytes()).hexdigest()
           for p in sorted(tmp_path.rglob("*")) if p.is_file()}
    assert got == goldens["ingest_sha256"][f"{codec}/{layout}"]
    if codec != "jpeg":  # lossless: the store reads back to the same resident pyramid
        back = pf.GpuSlide.from_store(tmp_path, "s0")
        for li in range(len(rec.levels)):
            assert cuda.equal(back.level_array(li), slide.level_array(li))


def test_resample_2x_fast_path_exact(pf, cuda):
    """side == 2 * out windows take resample2x_kernel (PIL's 2:1 weights as exact integer taps):
    byte-identical with the oracle's PIL resize for every layout and dtype, including the
    first/last output rows and columns (clipped, renormalised taps) and out sizes that are not
    multiples of 4 (general kernel)."""
    rs = np.random.default_rng(21)
    img = rs.integers(0, 256, size=(900, 1100, 3), dtype=np.uint8)
    s = pf.GpuSlide.from_array(img, "r2", 0.25, tile_size=128, downsample_factor=4)
    ss = pf.SlideSet([s])
    levels = port.pyramid(img, 128, 4)
    mpps = [lv.mpp for lv in s.record.levels]
    dss = [lv.downsample for lv in s.record.levels]
    for out in (8, 12, 32, 60, 96, 224, 30):
        reqs = []
        for _ in range(6):
            fp = 2 * out
            x, y = int(rs.integers(0, 1100 - fp)), int(rs.integers(0, 900 - fp))
            reqs.append((0, (x, y, fp, fp), 0.5, out))
        specs = pf.store.plan_specs(reqs, ss.records)
        assert all(int(sp["side"]) == 2 * out for sp in specs)
        want = np.stack([port.read_region(levels, mpps, dss, r[1], 0.5, out) for r in reqs])
        assert np.array_equal(ss.read_regions(specs, out).cpu().numpy(), want), out
        f32 = ss.read_regions(specs, out, dtype="f32", layout="nchw").cpu().numpy()
        assert np.array_equal(f32, port.normalize_patch(want).transpose(0, 3, 1, 2)), out


@pytest.mark.parametrize("case", range(int(os.environ.get("PF_FUZZ_CASES_RR", "4"))))
def test_random_reads_vs_oracle(pf, case):
    """Random windows (edges and overruns included), target mpps, output sizes, dtypes and
    layouts through the batched device read and the drop-in read_region, against the oracle's
    read_region (PIL) + normalize_patch: bit-exact, OutOfBoundsError where the reference raises."""
    rs = np.random.default_rng(700 + case)
    H, W = int(rs.integers(300, 900)), int(rs.integers(300, 900))
    img = rs.integers(0, 256, size=(H, W, 3), dtype=np.uint8)
    T = int(rs.choice([64, 128, 256]))
    f = int(rs.choice([2, 4]))
    s = pf.GpuSlide.from_array(img, f"r{case}", 0.25, tile_size=T, downsample_factor=f)
    ss = pf.SlideSet([s])
    lv = port.pyramid(img, T, f)
    mpps = [x.mpp for x in s.record.levels]
    ds = [x.downsample for x in s.record.levels]
    reqs, wants = [], []
    for _ in range(40):
        mpp = float(rs.choice([0.25, 0.3, 0.5, 0.7, 1.0, 2.0]))
        out = int(rs.choice([8, 32, 96, 224, 300]))
        side = int(rs.integers(4, min(H, W)))
        x, y = int(rs.integers(-2, W - side + 3)), int(rs.integers(-2, H - side + 3))
        try:
            want = port.read_region(lv, mpps, ds, (x, y, side, side), mpp, out)
        except IndexError:
            with pytest.raises(pf.OutOfBoundsError):
                s.read_region((x, y, side, side), mpp, out)
            continue
        got = s.read_region((x, y, side, side), mpp, out)
        assert np.array_equal(got, want), (x, y, side, mpp, out)
        if out == 96:
            reqs.append((0, (x, y, side, side), mpp, 96))
            wants.append(want)
    if reqs:  # the same windows batched, every dtype and layout
        specs = pf.store.plan_specs(reqs, ss.records)
        want = np.stack(wants)
        assert np.array_equal(ss.read_regions(specs, 96).cpu().numpy(), want)
        f32 = ss.read_regions(specs, 96, dtype="f32", layout="nchw").cpu().numpy()
        assert np.array_equal(f32, port.normalize_patch(want).transpose(0, 3, 1, 2))


def test_passthrough_only_reads_match_the_general_kernel(pf):
    """PF_SKIP_RESAMPLED (RegionLoader when every target mpp reads its window unresampled): the
    lean passthrough kernel's output equals read_regions_kernel's for every dtype and layout,
    windows at the level edges (edge replication) included, and a resampled spec in the batch
    is left untouched."""
    import torch

    rs = np.random.default_rng(41)
    H, W = 700, 900
    img = rs.integers(0, 256, size=(H, W, 3), dtype=np.uint8)
    # tile 120: rows of 360 B are not 16-byte multiples, so slide 1 takes the per-pixel staging path
    ss = pf.SlideSet([pf.GpuSlide.from_array(img, "pt", 0.25, tile_size=128, downsample_factor=4),
                      pf.GpuSlide.from_array(img, "pt120", 0.25, tile_size=120, downsample_factor=4)])
    for S in (224, 96, 300, 512):  # 512: the largest out_size, the most shared memory per band
        reqs = [(int(rs.integers(0, 2)), (int(rs.integers(0, W - S)), int(rs.integers(0, H - S)), S, S), 0.25, S)
                for _ in range(21)]
        reqs += [(0, (0, 0, S, S), 0.25, S), (0, (W - S, H - S, S, S), 0.25, S)]  # windows at the edges
        specs = pf.store.plan_specs(reqs, ss.records)
        for dtype, layout in (("f32", "nchw"), ("bf16", "nchw"), ("u8", "nchw"), ("u8", "hwc"), ("f32", "hwc")):
            want = ss.read_regions(specs, S, dtype=dtype, layout=layout).cpu()
            got = ss.read_regions(specs, S, dtype=dtype, layout=layout, passthrough_only=True).cpu()
            assert torch.equal(got, want), (S, dtype, layout)
        # a resampled spec (side != S) is left as it was
        r, mpp = (2 * S, 0.5) if S < 512 else (600, 0.3)  # a window that fits the 900 x 700 slide
        mixed = pf.store.plan_specs(reqs[:3] + [(0, (10, 10, r, r), mpp, S)], ss.records)
        sentinel = torch.full((4, 3, S, S), -7.0, device="cuda")
        ss.read_regions(mixed, S, dtype="f32", layout="nchw", out=sentinel, passthrough_only=True)
        ref = ss.read_regions(mixed, S, dtype="f32", layout="nchw").cpu()
        assert torch.equal(sentinel[:3].cpu(), ref[:3]) and bool((sentinel[3] == -7.0).all())
