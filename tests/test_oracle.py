"""Pin the CPU oracle (oracle/port.py) against vectors produced by the real reference."""

import hashlib

import numpy as np
import pytest

from oracle import port


def test_rng_streams(goldens):
    r = goldens["rng"]
    for seed in (0, 1, 12345, (1 << 63) + 5):
        for purpose in ("slide", "coords", "mpp", "cache", "synthetic-image"):
            s = port.Stream(seed, purpose)
            assert [hex(s.u64()) for _ in range(8)] == r[f"{seed}/{purpose}"]
    s = port.Stream(7, "coords")
    assert [s.randint(0, 7968) for _ in range(16)] == r["randint_7"]
    s = port.Stream(7, "mpp")
    assert [s.weighted_index([1.0, 2.0, 0.5, 0.0, 3.0]) for _ in range(32)] == r["weighted_7"]
    s = port.Stream(3, "slide")
    assert [s.randrange(7) for _ in range(32)] == r["randrange3_7"]


def test_survey_appendix_kats():
    # SURVEY.md Appendix A values, themselves produced by the reference
    assert port.fnv1a(b"coords") == 0xF7B5226AAD17FC87
    assert port.mix64(0) == 0
    s = port.Stream(0, "slide")
    assert [s.u64() for _ in range(3)] == [0xE2E224FAEC898B32, 0x17F4F399BB60EE20, 0xD9BF97EED7F60819]
    s = port.Stream(0, "coords")
    assert [s.randint(0, 7968) for _ in range(3)] == [7555, 836, 1247]


def test_select_level_and_rounding(goldens):
    mpps = [0.25, 1.0, 4.0]
    for t, want in goldens["select_level"].items():
        assert port.select_level(mpps, float(t)) == want
    assert port.round_half_away(2.5) == 3 and port.round_half_away(-2.5) == -3
    # 96 px at 0.97 on a 1.0 level -> 93 px window
    assert max(1, port.round_half_away(96 * 0.97 / 1.0)) == 93


def test_box_downsample_and_pyramid(goldens, golden_arrays):
    img = golden_arrays["synthetic_700x500"]
    assert np.array_equal(port.box_downsample(img, 32), golden_arrays["box32_700x500"])
    assert np.array_equal(port.box_downsample(img, 7), golden_arrays["box7_700x500"])
    lv = port.pyramid(img, 128, 2)
    assert [(a.shape[1], a.shape[0]) for a in lv] == [tuple(x[:2]) for x in goldens["levels_f2_t128"]]
    for i, a in enumerate(lv):
        assert np.array_equal(a, golden_arrays[f"level_f2_{i}"])
    assert np.array_equal(port.pyramid(img, 64, 4)[1], golden_arrays["level_f4_1"])
    assert np.array_equal(lv[-1], golden_arrays["thumb_f2"])


def test_read_region(goldens, golden_arrays):
    img = golden_arrays["synthetic_700x500"]
    lv = port.pyramid(img, 128, 2)
    mpps = [m for (_, _, m, _) in goldens["levels_f2_t128"]]
    ds = [d for (_, _, _, d) in goldens["levels_f2_t128"]]
    for r in goldens["reads"]:
        got = port.read_region(lv, mpps, ds, r["rect"], r["mpp"], r["out"])
        assert np.array_equal(got, golden_arrays[f"read_{r['k']}"]), r


def test_aa_resample_pil_flavour(golden_arrays):
    from PIL import Image

    rs = np.random.default_rng(0)
    for _ in range(25):
        s = int(rs.integers(5, 300))
        o = int(rs.integers(5, 260))
        a = rs.integers(0, 256, size=(s, s, 3), dtype=np.uint8)
        ref = np.asarray(Image.fromarray(a).resize((o, o), Image.Resampling.BILINEAR))
        assert np.array_equal(port.aa_resize_hwc(a, o, o, "pil"), ref), (s, o)


def test_aa_resample_torch_flavour():
    torch = pytest.importorskip("torch")
    rs = np.random.default_rng(1)
    for _ in range(25):
        h, w = int(rs.integers(5, 230)), int(rs.integers(5, 230))
        o = int(rs.choice([96, 224, int(rs.integers(5, 230))]))
        a = rs.integers(0, 256, size=(h, w, 3), dtype=np.uint8)
        ref = torch.nn.functional.interpolate(torch.from_numpy(a).permute(2, 0, 1)[None], size=(o, o), mode="bilinear",
                                              antialias=True, align_corners=False)[0].permute(1, 2, 0).numpy()
        assert np.array_equal(port.aa_resize_hwc(a, o, o, "torch"), ref), (h, w, o)


def test_luminance_mask(goldens, golden_arrays):
    assert np.array_equal(port.mask_luminance(golden_arrays["blob_thumb8"], 0.9), golden_arrays["blob_mask_lum"])
    allc = np.arange(1 << 24, dtype=np.uint32)
    rgb = np.stack([(allc >> 16) & 255, (allc >> 8) & 255, allc & 255], axis=1).astype(np.uint8).reshape(4096, 4096, 3)
    for thr in (0.9, 0.5, 0.25):
        bits = port.mask_luminance(rgb, thr)
        assert hashlib.sha256(np.packbits(bits).tobytes()).hexdigest() == goldens[f"allcolors_lum_{thr}_sha256"]
    # numpy's BLAS evaluates each row as fma(B, .0722, fma(R, .2126, G * .7152)); the CUDA kernel
    # restates exactly that.  (245, 231, 169) is the one colour on the 0.9 boundary: 0.8999999999999999
    # with this order, so it is foreground here.
    bits = port.mask_luminance(rgb, 0.9).reshape(-1)
    assert bits[(245 << 16) | (231 << 8) | 169]


def test_polygons(goldens, golden_arrays):
    for key, mask_key, scale, mrp in (("blob_poly", "blob_mask_lum", 1 / 8, 64), ("hand_poly", "hand_mask", 0.5, 4)):
        rings = port.polygon_from_mask(golden_arrays[mask_key], scale, mrp)
        want = goldens[key]["rings"]
        assert len(rings) == len(want)
        for a, b in zip(rings, want):
            assert np.array_equal(a, np.asarray(b))


def test_overlap_fraction(goldens):
    rings = [np.asarray(r) for r in goldens["blob_poly"]["rings"]]
    for x, y, w, h, f in goldens["blob_overlap"]:
        assert port.overlap_fraction(rings, (x, y, w, h)) == f
    hr = [np.asarray(r) for r in goldens["hand_poly"]["rings"]]
    for x, y, w, h, f in goldens["hand_overlap_grid64"]:
        assert port.overlap_fraction(hr, (x, y, w, h), grid=64) == f
    sq = [np.array([[0, 0], [0, 100], [100, 100], [100, 0]], dtype=np.float64)]
    assert [port.overlap_fraction(sq, r) for r in ((10, 10, 20, 20), (200, 200, 20, 20), (90, 10, 20, 20))] == goldens["rect_kats"]
    assert goldens["rect_kats"] == [1.0, 0.0, 0.4921875]


def _sampler_slides(goldens, idx):
    out = []
    for i in idx:
        w, h = goldens[f"sampler_dims_b{i}"]
        out.append({"id": f"b{i}", "width": w, "height": h, "base_mpp": 0.25,
                    "rings": [np.asarray(r) for r in goldens[f"sampler_poly_b{i}"]["rings"]]})
    return out


@pytest.mark.parametrize("case", ["single", "single_seed9", "multi_mpp", "weighted", "nofit", "exhaust"])
def test_epoch_stream(goldens, case):
    c = goldens["epoch_streams"][case]
    cfg = c["cfg"]
    slides = _sampler_slides(goldens, c["slides"])
    specs, _ = port.epoch_stream(slides, patch_size=cfg["patch_size"], min_fg=cfg["min_foreground"],
                                 mpps=[tuple(m) for m in cfg["target_mpps"]], seed=cfg["seed"],
                                 epoch_size=cfg["epoch_size"], max_attempts=cfg["max_attempts_per_slide"],
                                 strategy=cfg["slide_strategy"], weights=cfg["slide_weights"])
    got = [(slides[si]["id"], x, y, fp, mpp, seq) for si, x, y, fp, mpp, seq in specs]
    want = [(s["slide_id"], s["x"], s["y"], s["width"], s["target_mpp"], s["seq"]) for s in c["specs"]]
    assert got == want


def test_normalize(goldens):
    assert port.normalize_patch(np.array([0, 255, 128, 1, 254], np.uint8)).tolist() == goldens["normalize"]


def test_capped_stream_oracle_and_host_vs_reference(goldens):
    """capped_stream (pkg/sampler.py:230-281) over the multi_mpp manifest: the oracle restatement
    and the package's host mirror both replay the reference's seq sequence."""
    from paper_2404_15217_b200 import sampler as S

    specs = [S.PatchSpec(**d) for d in goldens["epoch_streams"]["multi_mpp"]["specs"]]
    for key, want in goldens["capped_streams"].items():
        cap, total, seed = key.split("/")
        cap = None if cap == "None" else int(cap)
        total, seed = int(total), int(seed)
        assert [s.seq for s in port.capped_stream(specs, cap, seed, total)] == want, key
        assert [s.seq for s in S.capped_stream(iter(specs), cap, seed, total)] == want, key
    import pytest

    with pytest.raises(ValueError):
        S.CappedCache(0)


@pytest.mark.parametrize("out_size", [16, 96, 112, 224])
def test_torch_aa_taps_never_need_the_uint8_clamp(out_size):
    """The multi-crop kernel drops torch's [0, 255] clamp after each resample pass
    (pf_multicrop.cu kNoClampNote): every output's int16 taps are >= 0 and
    255 * sum(taps) + 2^(prec-1) < 2^(prec+8), for every crop extent the kernel accepts
    (in <= 3.5 * out) of the 224-px source."""
    for in_size in range(1, min(224, int(3.5 * out_size)) + 1):
        _, q, p = port.aa_axis_table(in_size, out_size, "torch")
        assert p >= 14
        for taps in q:
            assert min(taps, default=0) >= 0
            assert 255 * sum(taps) + (1 << (p - 1)) < (1 << (p + 8)), (in_size, out_size)


@pytest.mark.parametrize("out_size", [16, 96, 112, 224])
def test_taps_rescaled_to_precision_16_give_the_same_bytes(out_size):
    """pf_multicrop.cu kAlignNote: for precision p <= 16 the tables hold the taps shifted to
    precision 16 (u16, a lone 1.0 tap at p = 14 stored as 65535), and the resample's result byte
    (sum w v + 2^(p-1)) >> p is unchanged for every crop extent and every uint8 input; an
    output whose 1.0 tap shares the row with another non-zero tap (which keeps its precision)
    never occurs."""
    rs = np.random.default_rng(out_size)
    for in_size in range(1, min(224, int(3.5 * out_size)) + 1):
        _, q, p = port.aa_axis_table(in_size, out_size, "torch")
        if p > 16:
            continue
        for taps in q:
            taps = [int(t) for t in taps]
            nz = sum(t != 0 for t in taps)
            assert not (p == 14 and (1 << 14) in taps and nz > 1), (in_size, out_size)
            w16 = [min(t << (16 - p), 65535) for t in taps]
            assert max(w16, default=0) <= 65535
            vals = rs.integers(0, 256, size=(64, len(taps)))
            vals[0] = 255
            vals[1] = 0
            want = ((vals * np.array(taps)).sum(1) + (1 << (p - 1))) >> p
            got = ((vals * np.array(w16)).sum(1) + (1 << 15)) >> 16
            assert np.array_equal(want, got), (in_size, out_size, taps)
