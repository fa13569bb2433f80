"""Saturation(0.07)+morphology masks of the 16 BASELINE C2 slides on the 1/32 thumbnail, exactly as
bench.py builds them (same seeds and redraw rule), for the CPU reference arm's polygons
(bench.py _cpu_polygons -> same_config).  Run on the GPU box; writes gpurun_out/c2_masks16.npz."""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

args = argparse.Namespace(config="2", slides=16, width=40000, height=30000)
pf, plan, slides = bench.build_slides(args, 0, 1)
out = {}
for g, (s, poly) in enumerate(slides):
    thumb, scale = s.thumbnail_device(32)
    bits = pf.foreground.mask_device(thumb, 1, 0.07, 1).cpu().numpy().astype(bool)
    assert np.array_equal(bits, np.asarray(bits))
    out[f"s{g}_mask"] = np.packbits(bits)
    out[f"s{g}_shape"] = np.array(bits.shape)
    out[f"s{g}_scale"] = np.array([scale])
    out[f"s{g}_nrings"] = np.array([len(poly.rings)])
    want = pf.polygon_from_mask(pf.BinaryMask(bits, scale), slide_id=s.record.slide_id)
    assert len(want.rings) == len(poly.rings) and all(np.array_equal(a, b) for a, b in zip(want.rings, poly.rings))
Path("gpurun_out").mkdir(exist_ok=True)
np.savez_compressed("gpurun_out/c2_masks16.npz", **out)
print("wrote gpurun_out/c2_masks16.npz")
