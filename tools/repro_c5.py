"""First C5 sweep point (one 100000x80000 slide, batch 256, L=0, bf16) outside the sweep loop,
for debugging under CUDA_LAUNCH_BLOCKING / PF_CHECKS builds."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

args = argparse.Namespace(config="5", slides=1, width=100000, height=80000, batch=256, dtype="bf16", gpus=1,
                          steps=3, warmup=3)
pf, plan, slides = bench.build_slides(args, 0, 1)
print("slides ready", flush=True)
feed = bench.make_feed(args, pf, plan, slides, 0, n_local=int(os.environ.get("NL", "0")),
                       patch=int(os.environ.get("PATCH", "224")))
sync = os.environ.get("SYNC", "1") == "1"
for i in range(8):
    feed.loader.next_batch()
    if sync:
        torch.cuda.synchronize()
    print("step", i, "queued" if not sync else "ok", flush=True)
torch.cuda.synchronize()
feed.loader.check()
print("ok")
