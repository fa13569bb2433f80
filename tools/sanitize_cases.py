"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck), one per kernel
family: multi-crop (TMA bulk-copy ring on mbarriers, both launch shapes), sampler (speculative
eval + ordered walk, sequential fallback), read_regions (passthrough + band-parallel PIL
resample + generic path), on-GPU tracing, PNG inflate/unfilter and JPEG decode.

usage: compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]
"""
import io
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2404_15217_b200 as pf  # noqa: E402
from paper_2404_15217_b200 import multicrop as mc  # noqa: E402


def _slide():
    yy, xx = np.mgrid[0:1100, 0:1300]
    blob = (np.sin(xx / 97.0) + np.cos(yy / 61.0)) > 0.3
    rs = np.random.default_rng(0)
    img = np.where(blob[..., None], np.array([180, 90, 170]), np.array([240, 240, 240])).astype(np.int64)
    img = np.clip(img + rs.normal(0, 4, img.shape), 0, 255).astype(np.uint8)
    s = pf.GpuSlide.from_array(img, "san", 0.25, tile_size=256, downsample_factor=4)
    thumb, scale = s.thumbnail(8)
    poly = pf.polygon_from_mask(pf.mask_from_rgb(thumb, 0.9, scale=scale), slide_id="san")
    return s, poly


def case_multicrop():
    s, poly = _slide()
    ld = mc.MultiCropLoader([(s, poly)], pf.SamplerConfig(patch_size=224, seed=1), batch_size=8, dtype="bf16")
    for _ in range(2):
        ld.next_batch()
    torch.cuda.synchronize()


def case_multicrop_mixed():
    s, poly = _slide()
    cfg = pf.SamplerConfig(patch_size=224, seed=2, target_mpps=[(0.25, 1.0), (0.5, 1.0)])
    ld = mc.MultiCropLoader([(s, poly)], cfg, batch_size=8, dtype="u8")
    ld.next_batch()
    torch.cuda.synchronize()


def case_sampler():
    s, poly = _slide()
    smp = pf.GpuSampler(pf.SamplerConfig(patch_size=224, seed=3), [(s, poly)])
    smp.next_batch(64)
    smp.next_batch(16)
    slow = pf.GpuSampler(pf.SamplerConfig(patch_size=224, seed=3), [(s, poly)], rounds=0)
    slow.next_batch(4)
    torch.cuda.synchronize()


def case_read_regions():
    s, _ = _slide()
    reqs = [(0, (10, 20, 224, 224), 0.25, 224), (0, (300, 77, 448, 448), 0.5, 224), (0, (5, 5, 1000, 1000), 4.0, 60),
            (0, (0, 0, 1200, 1000), 0.3, 600)]
    for r in reqs:
        specs = pf.store.plan_specs([r], [s.record])
        pf.SlideSet([s]).read_regions(specs, r[3], dtype="f32", layout="nchw")
    torch.cuda.synchronize()


def case_trace():
    rs = np.random.default_rng(4)
    m = torch.from_numpy((rs.random((60, 80)) < 0.5).astype(np.uint8)).cuda()
    pf.polygon_from_mask_device(m, 1.0, 1.0)
    torch.cuda.synchronize()


def case_png_jpeg():
    from PIL import Image

    from paper_2404_15217_b200 import store

    rs = np.random.default_rng(5)
    img = rs.integers(0, 255, (64, 64, 3), dtype=np.uint8)
    buf = io.BytesIO()
    Image.fromarray(img).save(buf, format="PNG")
    b = buf.getvalue()
    lv = torch.zeros((1, 1, 64, 64, 3), dtype=torch.uint8, device="cuda")
    store._decode_png_tiles(lv, 64, [(0, 0, 64, 64, store._png_zlib_stream(b, 64, 64))])
    torch.cuda.synchronize()
    assert np.array_equal(lv[0, 0].cpu().numpy(), img)
    buf = io.BytesIO()
    Image.fromarray(img).save(buf, format="JPEG", quality=90)
    lv.zero_()
    left = store._decode_jpeg_tiles(lv, 64, [(0, 0, 64, 64, buf.getvalue())])
    torch.cuda.synchronize()
    assert not left


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print("ok", name, flush=True)
