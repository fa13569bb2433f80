"""Throughput of the drop-in host paths: run_loader (host uint8 arrays out, `patchforge load`
semantics) and GpuSlide.read_region, on one 40000x30000 synthetic slide, uniform 224-px specs at
0.25 and 0.5 mpp.  The reference's loader (run_loader + normalize_patch on all host cores) is
bench.py's cpu_baseline.stages.loader."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2404_15217_b200 as pf  # noqa: E402
from paper_2404_15217_b200.synthetic import synthetic_slide  # noqa: E402

s = synthetic_slide("L", 40000, 30000, seed=1000, downsample_factor=4)
rs = np.random.default_rng(0)
for mpp in (0.25, 0.5):
    fp = int(224 * mpp / 0.25)
    specs = [pf.PatchSpec("L", int(rs.integers(0, 40000 - fp)), int(rs.integers(0, 30000 - fp)), fp, fp, mpp, 224, i)
             for i in range(4096)]
    for batch in (64, 512):
        list(pf.run_loader(specs[:256], s, batch=batch))  # warm
        t0 = time.perf_counter()
        n = sum(1 for _ in pf.run_loader(specs, s, batch=batch))
        dt = time.perf_counter() - t0
        print(f"run_loader mpp {mpp} chunk {batch}: {n / dt:.0f} patches/s (host arrays)")
    t0 = time.perf_counter()
    for sp in specs[:512]:
        s.read_region(sp.rect(), sp.target_mpp, 224)
    print(f"read_region mpp {mpp}: {512 / (time.perf_counter() - t0):.0f} patches/s (one call per patch)")
