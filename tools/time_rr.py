"""Time pf_read_regions on C3's mixed-mpp specs (2048 per call; half take the exact 2:1 kernel).

usage: [PF_B200_LIB=ab/x.so] python tools/time_rr.py"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

args = argparse.Namespace(config="3", slides=16, width=40000, height=30000, batch=2048, dtype="bf16", gpus=1)
pf, plan, slides = bench.build_slides(args, 0, 1)
feed = bench.make_feed(args, pf, plan, slides, 0)
L = feed.loader
out = L.next_batch()
torch.cuda.synchronize()
specs = out["specs"]
dst = torch.empty((2048, 224, 224, 3), dtype=torch.uint8, device="cuda")
for _ in range(3):
    L.slide_set.read_regions(specs, 224, out=dst, planned=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    L.slide_set.read_regions(specs, 224, out=dst, planned=True)
e.record()
torch.cuda.synchronize()
print(f"{os.environ.get('PF_B200_LIB', 'tree')}: read_regions (C3 specs, u8 HWC) {s.elapsed_time(e) / 20:.4f} ms")
