"""Experiment: C2 multi-crop step time with the live sampler vs capped replay (no sampler work)."""
import sys; sys.path.insert(0, '.')
import argparse, torch
import bench
from paper_2404_15217_b200.multicrop import MultiCropConfig, MultiCropLoader
args = argparse.Namespace(config="2", batch=1024, slides=int(sys.argv[1]) if len(sys.argv) > 1 else 16, width=40000, height=30000,
                          dtype="bf16", gpus=1)
pf, plan, slides = bench.build_slides(args, 0, 1)
for cap in (None, 4096):
    scfg = pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=[(0.25, 1.0)], seed=plan.sampler_seed)
    L = MultiCropLoader(slides, scfg, MultiCropConfig(), batch_size=1024, cap=cap)
    for _ in range(6):
        L.next_batch()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        L.next_batch()
    e.record(); torch.cuda.synchronize()
    print(f"slides {args.slides} cap {cap}: {s.elapsed_time(e) / 10:.3f} ms/step")
