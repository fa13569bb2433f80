import sys; sys.path.insert(0, '.')
import numpy as np, paper_2404_15217_b200 as pf
from paper_2404_15217_b200.synthetic import synthetic_slide
s = synthetic_slide("s2", 92884, 30214, seed=1002, downsample_factor=4)
thumb, scale = s.thumbnail_device(32)
mask = pf.foreground.mask_device(thumb, 1, 0.07, 1)
np.savez_compressed("gpurun_out/mask_s2.npz", mask=mask.cpu().numpy(), thumb=thumb.cpu().numpy()[::4, ::4])
print(scale, mask.shape)
