"""C5 sampler at large batches: sample and validate specs on the host (debug aid)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2404_15217_b200 import _native as N

args = argparse.Namespace(config="5", slides=1, width=100000, height=80000, batch=8192, dtype="bf16", gpus=1)
pf, plan, slides = bench.build_slides(args, 0, 1)
smp = pf.GpuSampler(pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=[(0.25, 1.0)],
                                     seed=plan.sampler_seed), slides, rounds=1)
for n in (256, 1024, 4096, 8192, 8192, 8192):
    out = smp.next_batch(n)
    torch.cuda.synchronize()
    a = out.cpu().numpy().view(N.SPEC_DTYPE).reshape(-1)
    st = smp.state_host()
    bad = (a["slide"] != 0) | (a["x"] < 0) | (a["y"] < 0) | (a["x"] > 100000) | (a["y"] > 80000) | (a["width"] != 224)
    print(n, "window", smp._window_for(n), "bad", int(bad.sum()), "first bad", np.flatnonzero(bad)[:5],
          "status", st.status, "emitted", st.emitted, "attempts", st.attempts, "slow", st.slow_evals,
          "seq", a["seq"][:2], a["seq"][-2:], flush=True)
