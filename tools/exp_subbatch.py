"""Experiment: multi-crop of fresh (L2-cold) batches of 1024 patches in one call vs k sub-batch
calls (each call's local crops then reread a sub-batch's source windows while still in L2)."""
import sys; sys.path.insert(0, '.')
import argparse, torch
import bench
from paper_2404_15217_b200.multicrop import MultiCropConfig, MultiCropLoader, crop_params, multicrop

args = argparse.Namespace(config="2", batch=1024, slides=16, width=40000, height=30000, dtype="bf16", gpus=1)
pf, plan, slides = bench.build_slides(args, 0, 1)
scfg = pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=[(0.25, 1.0)], seed=plan.sampler_seed)
L = MultiCropLoader(slides, scfg, MultiCropConfig(), batch_size=1024)
n_it = 12
batches = [L.sampler.next_batch(1024).clone() for _ in range(n_it)]
mc = MultiCropConfig()
prms = [crop_params(mc, 1024, seed=1, step=i) for i in range(n_it)]
torch.cuda.synchronize()
G = torch.empty((2, 1024, 3, 224, 224), dtype=torch.bfloat16, device="cuda")
Lo = torch.empty((8, 1024, 3, 96, 96), dtype=torch.bfloat16, device="cuda")
for k in (1, 2, 4, 8):
    sub = 1024 // k
    outs = [(torch.empty((2, sub, 3, 224, 224), dtype=torch.bfloat16, device="cuda"),
             torch.empty((8, sub, 3, 96, 96), dtype=torch.bfloat16, device="cuda")) for _ in range(k)]
    def run(i):
        for j in range(k):
            multicrop(L.slide_set, batches[i][j * sub:(j + 1) * sub], prms[i][j * sub:(j + 1) * sub], mc, dtype="bf16",
                      out_global=outs[j][0], out_local=outs[j][1])
    run(0); run(1)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(2, n_it):
        run(i)
    e.record(); torch.cuda.synchronize()
    print(f"sub-batches {k}: {s.elapsed_time(e) / (n_it - 2):.4f} ms per 1024 patches (fresh windows)")
