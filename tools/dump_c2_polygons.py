"""Render the two full-size BASELINE C2 test slides (tests/test_gpu_fullsize.py's `c2` fixture),
trace their saturation-mask polygons and dump them (+ the GPU sampler's first 1024 specs) to
gpurun_out/c2_polygons.npz, for the offline reference epoch_stream golden
(tests/golden/make_c2_stream_golden.py).  Run on the GPU box."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2404_15217_b200 as pf  # noqa: E402
from paper_2404_15217_b200.synthetic import synthetic_slide  # noqa: E402

W, H = 40000, 30000
out = {}
pairs = []
for gi in range(2):
    for k in range(8):
        s = synthetic_slide(f"s{gi}", W, H, seed=1000 + gi + 100_000 * k, downsample_factor=4)
        thumb, scale = s.thumbnail_device(32)
        mask = pf.foreground.mask_device(thumb, 1, 0.07, 1)
        bm = pf.BinaryMask(mask.cpu().numpy().astype(bool), scale)
        try:
            poly = pf.polygon_from_mask(bm, slide_id=f"s{gi}")
            break
        except ValueError:
            del s
    out[f"s{gi}_mask"] = np.packbits(bm.bits)
    out[f"s{gi}_mask_shape"] = np.array(bm.bits.shape)
    out[f"s{gi}_scale"] = np.array([scale])
    out[f"s{gi}_nrings"] = np.array([len(poly.rings)])
    for r, ring in enumerate(poly.rings):
        out[f"s{gi}_ring{r}"] = np.asarray(ring, dtype=np.float64)
    pairs.append((s.record, poly))
    print(f"s{gi}: {len(poly.rings)} rings, {sum(len(r) for r in poly.rings)} vertices, scale {scale}")
    del s
smp = pf.GpuSampler(pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=[(0.25, 1.0)], seed=5), pairs)
specs = smp.to_patch_specs(smp.next_batch(1024))
out["gpu_specs"] = np.array([(int(p.slide_id[1:]), p.x, p.y, p.width, p.seq) for p in specs], dtype=np.int64)
Path("gpurun_out").mkdir(exist_ok=True)
np.savez_compressed("gpurun_out/c2_polygons.npz", **out)
print("wrote gpurun_out/c2_polygons.npz")
