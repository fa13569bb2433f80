"""Time the global-crop and local-crop multi-crop launches separately (C2 shapes, 4 slides).

usage: python tools/time_mc.py   (PF_B200_LIB selects another build of the library)
"""
import sys; sys.path.insert(0, '.')
import argparse, os, torch
import bench
from paper_2404_15217_b200.multicrop import MultiCropConfig, MultiCropLoader, crop_params, multicrop

args = argparse.Namespace(config="2", batch=1024, slides=int(os.environ.get("PF_TIME_SLIDES", "4")), width=40000, height=30000, dtype="bf16", gpus=1)
pf, plan, slides = bench.build_slides(args, 0, 1)
scfg = pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=[(0.25, 1.0)], seed=plan.sampler_seed)
L = MultiCropLoader(slides, scfg, MultiCropConfig(), batch_size=1024)
specs = L.next_batch()["specs"]
torch.cuda.synchronize()
for name, mc in (("global", MultiCropConfig(n_local=0)), ("local", MultiCropConfig(n_global=0, p_blur=[0.5] * 8, p_solarize=[0.0] * 8)),
                 ("both", MultiCropConfig())):
    prm = crop_params(mc, 1024, seed=1, step=0)
    outs = {}
    for _ in range(3):
        multicrop(L.slide_set, specs, prm, mc, dtype="bf16")
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        multicrop(L.slide_set, specs, prm, mc, dtype="bf16")
    e.record(); torch.cuda.synchronize()
    print(f"{name}: {s.elapsed_time(e) / 20:.4f} ms")

# bit-identity check across builds: sha256 of u8 crops (every op on, 1024 patches)
import hashlib
mc = MultiCropConfig(p_jitter=1.0, p_gray=0.2, p_blur=[0.5] * 10, p_solarize=[0.2] * 10)
prm = crop_params(mc, 1024, seed=7, step=3)
g, l = multicrop(L.slide_set, specs, prm, mc, dtype="u8")
torch.cuda.synchronize()
print("sha256", hashlib.sha256(g.cpu().numpy().tobytes() + l.cpu().numpy().tobytes()).hexdigest()[:16])
