import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2404_15217_b200 import _native as N
from paper_2404_15217_b200.store import GpuSlide
w, h = 3000, 1000
s = GpuSlide.allocate("c", w, h, 0.25, 256, 4)
fw, fh = -(-w // 64) + 1, -(-h // 64) + 1
f = np.tile(np.linspace(0, 1, fw, dtype=np.float32), (fh, 1))
fd = torch.from_numpy(f).cuda()
N.check(N.lib().pf_synth_level0(s.desc, fd.data_ptr(), fh, fw, 64, 0.5, 7, None), "synth")
torch.cuda.synchronize()
img = s.level_array(0).cpu().numpy().astype(int)
tissue = (img.max(-1) - img.min(-1)) > 40
print("row 0 transitions at x =", np.flatnonzero(np.diff(tissue[0].astype(int)))[:10], "expected ~", w // 2)
print("tissue frac by column blocks:", [round(tissue[:, i:i + 300].mean(), 2) for i in range(0, w, 300)])
