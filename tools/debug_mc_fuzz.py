"""Reproduce one random multi-crop configuration of tests/test_gpu_multicrop.py and report the
crops that differ from torchvision (debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import pytest  # noqa: F401

from oracle import augment as A
from oracle import port

case = int(sys.argv[1])
import paper_2404_15217_b200 as pf
from paper_2404_15217_b200 import multicrop as mc

pf.mc = mc
import torch

ga = np.load("tests/golden/reference_arrays.npz")
img = np.ascontiguousarray(np.tile(ga["blob_640x480"], (2, 2, 1)))  # the test's scene
s0 = pf.GpuSlide.from_array(img, "a", 0.25, tile_size=128, downsample_factor=4)
ss = pf.SlideSet([s0])
rq = np.random.default_rng(0)
reqs = []
for k in range(14):
    x, y = int(rq.integers(0, 1280 - 224)), int(rq.integers(0, 960 - 224))
    reqs.append((0, (x, y, 224, 224), 0.25, 224))
for k in range(4):
    x, y = int(rq.integers(0, 1280 - 448)), int(rq.integers(0, 960 - 448))
    reqs.append((0, (x, y, 448, 448), 0.5, 224))
reqs.append((0, (1280 - 224, 960 - 224, 224, 224), 0.25, 224))
specs = pf.store.plan_specs(reqs, ss.records)
levels = port.pyramid(img, 128, 4)
srcs = [port.read_region(levels, [lv.mpp for lv in s0.record.levels], [lv.downsample for lv in s0.record.levels],
                         r[1], r[2], r[3]) for r in reqs]
rs = np.random.default_rng(500 + case)
n_global = int(rs.integers(1, 3))
n_local = int(rs.choice([0, 2, 4, 8]))
n = n_global + n_local
lo = float(rs.uniform(0.08, 0.5))
cfg = mc.MultiCropConfig(
    n_global=n_global, n_local=n_local,
    global_size=int(rs.choice([224, 192, 160])), local_size=int(rs.choice([96, 112, 128])),
    global_scale=(lo, 1.0), local_scale=(0.05, lo), ratio=(float(rs.uniform(0.5, 0.9)), float(rs.uniform(1.1, 2.0))),
    p_flip=float(rs.uniform()), p_jitter=float(rs.uniform(0.5, 1.0)), p_gray=float(rs.uniform(0, 0.5)),
    brightness=float(rs.uniform(0, 0.6)), contrast=float(rs.uniform(0, 0.6)), saturation=float(rs.uniform(0, 0.6)),
    hue=float(rs.uniform(0, 0.5)), p_blur=[float(v) for v in rs.uniform(0, 1, n)],
    p_solarize=[float(v) for v in rs.uniform(0, 0.5, n)], solarize_threshold=float(rs.choice([64.0, 128.0, 200.5])))
print(cfg)
dspecs = ss.specs_to_device(specs)
src = ss.read_regions(dspecs, cfg.src_size)
params = mc.crop_params(cfg, len(specs), seed=3, step=0)
g, l = mc.multicrop(ss, dspecs, params, cfg, dtype="u8", src_hwc=src)
torch.cuda.synchronize()
prm = mc.params_host(params)
g, l = g.cpu().numpy(), l.cpu().numpy()
for i, src in enumerate(srcs):
    for c in range(cfg.n_crops):
        want = A.torchvision_crop(src, prm[i, c])
        got = (g[c, i] if c < cfg.n_global else l[c - cfg.n_global, i]).transpose(1, 2, 0)
        d = np.abs(got.astype(int) - want.astype(int))
        if d.max() > 1:
            p = dict(zip(prm.dtype.names, prm[i, c].tolist()))
            ys, xs = np.nonzero(d.max(-1) > 1)
            print(i, c, p, "bad px", len(ys), "at", list(zip(ys[:5], xs[:5])), "got", got[ys[0], xs[0]], "want", want[ys[0], xs[0]])
