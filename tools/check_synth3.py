import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2404_15217_b200 import _native as N
from paper_2404_15217_b200.store import GpuSlide
from paper_2404_15217_b200.synthetic import synthetic_slide, tissue_field
w, h = 3000, 1000
a = synthetic_slide("a", w, h, seed=1002, downsample_factor=4).level_array(0).cpu().numpy().astype(int)
f, thr = tissue_field(w, h, 1002)
ta = (a.max(-1) - a.min(-1)) > 40
fy = np.clip(np.round((np.arange(h) + 0.5) / 64 - 0.5).astype(int), 0, f.shape[0] - 1)
fx = np.clip(np.round((np.arange(w) + 0.5) / 64 - 0.5).astype(int), 0, f.shape[1] - 1)
fm = f[fy][:, fx] > thr
print("agree", (ta == fm).mean(), ta.mean(), fm.mean(), f.shape, thr)
print("rows of ta:"); [print(''.join('#' if v else '.' for v in r[::40])) for r in ta[::100]]
print("rows of fm:"); [print(''.join('#' if v else '.' for v in r[::40])) for r in fm[::100]]
