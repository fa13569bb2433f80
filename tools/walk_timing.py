"""Phase timestamps of sample_walk_kernel (build ab/walktime.so with -DPF_WALK_TIMING:
python tools/build_variant.py walktime pf_sampler.cu -DPF_WALK_TIMING), C2 sampler, 1024 specs."""
import argparse, os, sys
sys.path.insert(0, '.')
import numpy as np, torch
import bench
args = argparse.Namespace(config="2", slides=16, width=40000, height=30000)
pf, plan, slides = bench.build_slides(args, 0, 1)
smp = pf.GpuSampler(pf.SamplerConfig(patch_size=224, seed=plan.sampler_seed), slides, rounds=2)
for it in range(4):
    smp.next_batch(1024)
    torch.cuda.synchronize()
    for r, off in (("round 1", 32), ("round 2", 96)):
        t = smp._ws[off:off + 6 * 8].cpu().numpy().view(np.uint64).astype(np.int64)
        print(r, "phases (us): start->bitmaps %.1f, ->tables %.1f, ->draws %.1f, ->walk %.1f, ->materialise %.1f"
              % tuple((t[1:] - t[:-1]) / 1000.0))
