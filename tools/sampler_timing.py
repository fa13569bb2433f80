"""Time the C2 sampler alone (pf_sample, 1024 specs, --rounds speculation rounds) with CUDA events.

usage: [PF_B200_LIB=ab/variant.so] python tools/sampler_timing.py [iters]
Prints the median and min per-batch time; also checks the spec stream against the first
library's (pass --dump to write /tmp/specs_<name>.npy for a cross-variant comparison)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench

ap = argparse.ArgumentParser()
ap.add_argument("iters", type=int, nargs="?", default=12)
ap.add_argument("--dump", default=None)
ap.add_argument("--rounds", type=int, default=1)
a = ap.parse_args()
args = argparse.Namespace(config="2", slides=16, width=40000, height=30000)
pf, plan, slides = bench.build_slides(args, 0, 1)
smp = pf.GpuSampler(pf.SamplerConfig(patch_size=224, seed=plan.sampler_seed), slides, rounds=a.rounds)
outs, ts = [], []
for rep in range(a.iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    batch = [smp.next_batch(1024).clone() for _ in range(10)]  # host stays ahead of the GPU
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 100.0)  # us per batch
    outs += [o.cpu().numpy() for o in batch]
ts = np.array(ts[2:])
print(f"{os.environ.get('PF_B200_LIB', 'default')} rounds={a.rounds}: sampler per 1024 specs median {np.median(ts):.1f} us, "
      f"min {ts.min():.1f} us")
if a.dump:
    np.save(a.dump, np.concatenate(outs))
