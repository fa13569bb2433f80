"""Compare the GPU-rendered synthetic slide's tissue layout with the host field it was drawn from."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2404_15217_b200.synthetic import synthetic_slide, tissue_field
for (w, h) in ((3000, 1000), (20000, 6000), (92884, 30214)):
    s = synthetic_slide("c", w, h, seed=1002, downsample_factor=4)
    f, thr = tissue_field(w, h, 1002)
    rs = np.random.default_rng(0)
    xs, ys = rs.integers(0, w, 20000), rs.integers(0, h, 20000)
    T = 256
    lv = s.levels[0]
    px = lv[torch.from_numpy(ys // T).cuda(), torch.from_numpy(xs // T).cuda(), torch.from_numpy(ys % T).cuda(), torch.from_numpy(xs % T).cuda()].cpu().numpy().astype(int)
    tissue = (px.max(1) - px.min(1)) > 40
    fv = f[np.clip(np.round((ys + 0.5) / 64 - 0.5).astype(int), 0, f.shape[0] - 1), np.clip(np.round((xs + 0.5) / 64 - 0.5).astype(int), 0, f.shape[1] - 1)] > thr
    print(w, h, "agree", (tissue == fv).mean(), "tissue frac", tissue.mean())
