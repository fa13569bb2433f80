"""GPU parity: fused gather + DINOv2 multi-crop vs torchvision v2 on the same explicit crop
parameters (<= 1 uint8 LSB before normalisation; the normalising epilogue is bit-exact)."""

import os

import numpy as np
import pytest

from oracle import augment as A
from oracle import port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pf(cuda):
    import paper_2404_15217_b200 as pf
    from paper_2404_15217_b200 import multicrop as mc

    pf.mc = mc
    return pf


@pytest.fixture(scope="module")
def scene(pf, golden_arrays):
    img = np.ascontiguousarray(np.tile(golden_arrays["blob_640x480"], (2, 2, 1)))  # 960 x 1280
    s = pf.GpuSlide.from_array(img, "a", 0.25, tile_size=128, downsample_factor=4)
    ss = pf.SlideSet([s])
    rs = np.random.default_rng(0)
    reqs = []
    for k in range(14):
        x, y = int(rs.integers(0, 1280 - 224)), int(rs.integers(0, 960 - 224))
        reqs.append((0, (x, y, 224, 224), 0.25, 224))
    for k in range(4):  # read at 0.5 mpp: 448 px window resampled to 224 (config 3 path)
        x, y = int(rs.integers(0, 1280 - 448)), int(rs.integers(0, 960 - 448))
        reqs.append((0, (x, y, 448, 448), 0.5, 224))
    reqs.append((0, (1280 - 224, 960 - 224, 224, 224), 0.25, 224))  # slide corner
    specs = pf.store.plan_specs(reqs, ss.records)
    levels = port.pyramid(img, 128, 4)
    mpps = [lv.mpp for lv in s.record.levels]
    ds = [lv.downsample for lv in s.record.levels]
    srcs = [port.read_region(levels, mpps, ds, r[1], r[2], r[3]) for r in reqs]
    return ss, specs, srcs


def _run(pf, ss, specs, cfg, dtype, seed=3, step=0):
    torch = pytest.importorskip("torch")
    dspecs = ss.specs_to_device(specs)
    src = ss.read_regions(dspecs, cfg.src_size)  # plans sx/sy; resampled patches for off-level reads
    params = pf.mc.crop_params(cfg, len(specs), seed=seed, step=step)
    g, l = pf.mc.multicrop(ss, dspecs, params, cfg, dtype=dtype, src_hwc=src)
    torch.cuda.synchronize()
    return g, l, pf.mc.params_host(params)


def _check_against_torchvision(pf, scene, cfg):
    ss, specs, srcs = scene
    g, l, prm = _run(pf, ss, specs, cfg, "u8")
    g, l = g.cpu().numpy(), l.cpu().numpy()
    worst, diff_px, total = 0, 0, 0
    for i, src in enumerate(srcs):
        for c in range(cfg.n_crops):
            want = A.torchvision_crop(src, prm[i, c])
            got = (g[c, i] if c < cfg.n_global else l[c - cfg.n_global, i]).transpose(1, 2, 0)
            d = np.abs(got.astype(int) - want.astype(int))
            if prm[i, c]["flags"] & 16:  # solarize: a 1-LSB difference before it that straddles the
                # threshold comes out as v against 255 - v' (|v - v'| <= 1); count it as that LSB
                thr = float(prm[i, c]["solarize_threshold"])
                g_, w_ = got.astype(int), want.astype(int)
                crossing = (d > 1) & (np.abs(g_ + w_ - 255) <= 1) & \
                    (np.minimum(np.abs(g_ - thr), np.abs(255 - g_ - thr)) <= 1.5)
                d = np.where(crossing, 1, d)
            worst = max(worst, int(d.max()))
            diff_px += int((d > 0).sum())
            total += d.size
            assert d.max() <= 1, (i, c, dict(zip(prm.dtype.names, prm[i, c].tolist())))
    return worst, diff_px / total


def test_multicrop_dinov2_config_vs_torchvision(pf, scene):
    worst, frac = _check_against_torchvision(pf, scene, pf.mc.MultiCropConfig())
    assert frac < 1e-3, frac


def test_multicrop_every_op_vs_torchvision(pf, scene):
    cfg = pf.mc.MultiCropConfig(p_jitter=1.0, p_gray=0.3, p_blur=[0.5] * 10, p_solarize=[0.5] * 10)
    worst, frac = _check_against_torchvision(pf, scene, cfg)
    assert frac < 1e-3, frac


def test_normalising_epilogue_exact(pf, scene):
    torch = pytest.importorskip("torch")
    ss, specs, _ = scene
    cfg = pf.mc.MultiCropConfig()
    g8, l8, _ = _run(pf, ss, specs, cfg, "u8")
    gf, lf, _ = _run(pf, ss, specs, cfg, "f32")
    gb, lb, _ = _run(pf, ss, specs, cfg, "bf16")
    mean = np.asarray(pf.IMAGENET_MEAN, np.float32)[:, None, None]
    std = np.asarray(pf.IMAGENET_STD, np.float32)[:, None, None]
    for u8, f32, b16 in ((g8, gf, gb), (l8, lf, lb)):
        want = (u8.cpu().numpy().astype(np.float32) / np.float32(255.0) - mean) / std
        assert np.array_equal(f32.cpu().numpy(), want)
        assert torch.equal(b16.cpu(), torch.from_numpy(want).to(torch.bfloat16))


def test_crop_params_deterministic_and_distributed(pf):
    cfg = pf.mc.MultiCropConfig()
    a = pf.mc.params_host(pf.mc.crop_params(cfg, 4096, seed=11, rank=0, step=5))
    b = pf.mc.params_host(pf.mc.crop_params(cfg, 4096, seed=11, rank=0, step=5))
    c = pf.mc.params_host(pf.mc.crop_params(cfg, 4096, seed=11, rank=1, step=5))
    d = pf.mc.params_host(pf.mc.crop_params(cfg, 4096, seed=11, rank=0, step=6))
    assert a.tobytes() == b.tobytes() and a.tobytes() != c.tobytes() and a.tobytes() != d.tobytes()
    fl = a["flags"]
    assert abs((fl & 1).astype(bool).mean() - 0.5) < 0.02
    assert abs((fl & 2).astype(bool).mean() - 0.8) < 0.02
    assert abs((fl & 4).astype(bool).mean() - 0.2) < 0.02
    blur = (fl & 8).astype(bool).mean(axis=0)
    assert blur[0] == 1.0 and abs(blur[1] - 0.1) < 0.02 and np.all(np.abs(blur[2:] - 0.5) < 0.04)
    sol = (fl & 16).astype(bool).mean(axis=0)
    assert sol[0] == 0 and abs(sol[1] - 0.2) < 0.03 and np.all(sol[2:] == 0)
    area = a["height"] * a["width"] / 224.0**2
    assert np.all(area[:, :2] >= 0.30) and np.all(area[:, :2] <= 1.0)
    assert np.all(area[:, 2:] >= 0.04) and np.all(area[:, 2:] <= 0.34)
    assert np.all(a["top"] + a["height"] <= 224) and np.all(a["left"] + a["width"] <= 224)
    assert np.all((a["brightness"] >= 0.6) & (a["brightness"] <= 1.4))
    assert np.all((a["hue"] >= -0.1) & (a["hue"] <= 0.1))
    assert np.all((a["sigma"] >= 0.1) & (a["sigma"] <= 2.0))
    perms = {tuple(o) for o in a["order"].reshape(-1, 4).tolist()}
    assert len(perms) == 24


def test_loader_end_to_end(pf):
    """Synthetic slide -> thumbnail -> saturation mask -> polygon -> sampler -> multi-crop."""
    from paper_2404_15217_b200.synthetic import synthetic_slide

    s = synthetic_slide("syn", 6000, 4500, seed=1, blob_px=800)
    thumb, scale = s.thumbnail(32)
    poly = pf.polygon_from_mask(pf.mask_from_saturation(thumb, 0.07, 1, scale=scale), slide_id="syn")
    cfg = pf.SamplerConfig(patch_size=224, seed=0, target_mpps=[(0.25, 1.0), (0.5, 1.0)])
    loader = pf.mc.MultiCropLoader([(s, poly)], cfg, batch_size=32)
    out = loader.next_batch()
    out2 = loader.next_batch()
    assert out["global_crops"].shape == (2, 32, 3, 224, 224) and out["local_crops"].shape == (8, 32, 3, 96, 96)
    torch = pytest.importorskip("torch")
    torch.cuda.synchronize()
    st = loader.sampler.check()
    assert st.seq == 3 * 32  # two consumed batches + one prefetched
    # the prefetched stream is the plain stream: same specs as sampling without prefetch
    ref = pf.mc.MultiCropLoader([(s, poly)], cfg, batch_size=32, prefetch=False)
    ref.next_batch()
    b2 = ref.next_batch()
    assert torch.equal(b2["specs"], out2["specs"]) and torch.equal(b2["global_crops"], out2["global_crops"])
    assert bool(out2["global_crops"].float().abs().sum() > 0)


def test_hue_every_colour_exact(pf):
    """Every one of the 2^24 RGB colours through the kernel's adjust_hue (random shift in
    [-0.5, 0.5] per crop, the other jitter factors pinned to 1, identity crop): bit-exact
    against the float32 restatement (pinned to torchvision by test_aug_semantics)."""
    torch = pytest.importorskip("torch")
    gx, gy = 19, 18  # 342 patches of 224^2 >= 2^24 pixels
    n = gx * gy
    idx = (np.arange(n * 224 * 224, dtype=np.int64) % (1 << 24)).reshape(gy, gx, 224, 224)
    rgb = np.stack([(idx >> 16) & 255, (idx >> 8) & 255, idx & 255], -1).astype(np.uint8)
    img = np.ascontiguousarray(rgb.transpose(0, 2, 1, 3, 4).reshape(gy * 224, gx * 224, 3))
    s = pf.GpuSlide.from_array(img, "hue", 0.25, tile_size=256, downsample_factor=4)
    ss = pf.SlideSet([s])
    reqs = [(0, (224 * (k % gx), 224 * (k // gx), 224, 224), 0.25, 224) for k in range(n)]
    specs = pf.store.plan_specs(reqs, ss.records)
    cfg = pf.mc.MultiCropConfig(n_global=1, n_local=0, global_scale=(1.0, 1.0), ratio=(1.0, 1.0), p_flip=0.0,
                                p_jitter=1.0, p_gray=0.0, brightness=0.0, contrast=0.0, saturation=0.0, hue=0.5,
                                p_blur=[0.0], p_solarize=[0.0])
    g, _, prm = _run(pf, ss, specs, cfg, "u8", seed=7)
    g = g.cpu().numpy()
    for k in range(n):
        p = prm[k, 0]
        assert p["height"] == 224 and p["width"] == 224 and p["brightness"] == 1.0
        src = rgb[k // gx, k % gx]
        want = A.hue(src, float(p["hue"]))
        got = g[0, k].transpose(1, 2, 0)
        assert np.array_equal(got, want), (k, float(p["hue"]), int((got != want).any(-1).sum()))


@pytest.mark.parametrize("n_local,local_size", [(0, 96), (4, 112)])
def test_crop_count_and_size_variants_vs_torchvision(pf, scene, n_local, local_size):
    """BASELINE config 5 shapes: no local crops, or 4 local crops of another size (generic-size
    kernel path), against torchvision on the same parameters."""
    cfg = pf.mc.MultiCropConfig(n_local=n_local, local_size=local_size, p_jitter=1.0, p_gray=0.3,
                                p_blur=[0.5] * (2 + n_local), p_solarize=[0.5] * (2 + n_local))
    worst, frac = _check_against_torchvision(pf, scene, cfg)
    assert frac < 1e-3, frac


def test_f32_and_bf16_outputs_agree_with_u8(pf, scene):
    """The normalised outputs of a config without blur are exactly the u8 crops through the LUT."""
    torch = pytest.importorskip("torch")
    ss, specs, _ = scene
    cfg = pf.mc.MultiCropConfig(p_blur=[0.0] * 10)
    g8, l8, _ = _run(pf, ss, specs, cfg, "u8", seed=9)
    gf, lf, _ = _run(pf, ss, specs, cfg, "f32", seed=9)
    mean = np.asarray(pf.IMAGENET_MEAN, np.float32)[:, None, None]
    std = np.asarray(pf.IMAGENET_STD, np.float32)[:, None, None]
    for u8, f32 in ((g8, gf), (l8, lf)):
        want = (u8.cpu().numpy().astype(np.float32) / np.float32(255.0) - mean) / std
        assert np.array_equal(f32.cpu().numpy(), want)


@pytest.mark.parametrize("case", range(int(os.environ.get("PF_FUZZ_CASES_MC", "6"))))
def test_random_configs_vs_torchvision(pf, scene, case):
    """Random multi-crop configurations (crop counts and sizes across the compile-time and
    generic kernel paths -- sizes down to src/3.5, the resample's tap limit -- scale/ratio ranges, jitter strengths, op probabilities, solarize
    threshold) against torchvision on the same parameters: <= 1 LSB, < 0.1 % of values."""
    rs = np.random.default_rng(500 + case)
    n_global = int(rs.integers(1, 3))
    n_local = int(rs.choice([0, 2, 4, 8]))
    n = n_global + n_local
    lo = float(rs.uniform(0.08, 0.5))
    cfg = pf.mc.MultiCropConfig(
        n_global=n_global, n_local=n_local,
        global_size=int(rs.choice([224, 192, 160])), local_size=int(rs.choice([96, 112, 128])),
        global_scale=(lo, 1.0), local_scale=(0.05, lo), ratio=(float(rs.uniform(0.5, 0.9)), float(rs.uniform(1.1, 2.0))),
        p_flip=float(rs.uniform()), p_jitter=float(rs.uniform(0.5, 1.0)), p_gray=float(rs.uniform(0, 0.5)),
        brightness=float(rs.uniform(0, 0.6)), contrast=float(rs.uniform(0, 0.6)), saturation=float(rs.uniform(0, 0.6)),
        hue=float(rs.uniform(0, 0.5)), p_blur=[float(v) for v in rs.uniform(0, 1, n)],
        p_solarize=[float(v) for v in rs.uniform(0, 0.5, n)], solarize_threshold=float(rs.choice([64.0, 128.0, 200.5])))
    worst, frac = _check_against_torchvision(pf, scene, cfg)
    assert frac < 1e-3, (frac, cfg)
