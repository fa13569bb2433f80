"""Per-candidate latency of sample_eval_kernel (build ab/evaltime.so with -DPF_EVAL_TIMING:
python tools/build_variant.py evaltime pf_sampler.cu -DPF_EVAL_TIMING), C2 sampler, one round.

PF_B200_LIB=ab/evaltime.so python tools/eval_timing.py
Prints the candidates the raster bounds left for the lattice and the warp pass's span (first
warp start to last part end)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench

args = argparse.Namespace(config="2", slides=16, width=40000, height=30000)
pf, plan, slides = bench.build_slides(args, 0, 1)
smp = pf.GpuSampler(pf.SamplerConfig(patch_size=224, seed=plan.sampler_seed), slides, rounds=1)
smp.next_batch(1024)
torch.cuda.synchronize()
n_slides = len(slides)
for it in range(3):
    window = smp._window_for(1024)
    ws = smp._ws
    stamps = ws[:256].view(torch.int64)
    stamps[20] = 2 ** 63 - 1
    stamps[21] = 0
    smp.next_batch(1024)
    torch.cuda.synchronize()
    span = (int(stamps[21]) - int(stamps[20])) / 1000.0
    queued = int(ws[4:8].view(torch.int32)) - 0x7F7F7F7F
    qoff = 256 + (n_slides * (window // 32) * 4 + 255) // 256 * 256 + n_slides * window * 16
    parts = ws[qoff + 16384 * 4:qoff + (16384 + 2 * 4 * queued) * 4].view(torch.int32).view(-1, 2).cpu().numpy()
    lat = parts[:, 0] / 1000.0
    start = (parts[:, 1] - (int(stamps[20]) & 0x7FFFFFFF)) / 1000.0
    q = np.percentile(lat, [50, 90, 99, 100])
    print(f"window {window}: {queued} of {n_slides * window} candidates queued for the lattice, "
          f"warp pass span {span:.1f} us; part latency p50 {q[0]:.1f} p90 {q[1]:.1f} p99 {q[2]:.1f} max {q[3]:.1f} us; "
          f"part start p50 {np.median(start):.1f} max {start.max():.1f} us")
