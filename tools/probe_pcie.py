"""D2H / H2D bandwidth of pinned copies on one vs several streams (the e2e path's bound)."""
import time

import torch

n = 1 << 30
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
hosts = [torch.empty(n // k, dtype=torch.uint8).pin_memory() for k in (1,)]
host = torch.empty(n, dtype=torch.uint8).pin_memory()
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = n // ns
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                host[i * chunk:(i + 1) * chunk].copy_(dev[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"D2H {ns} stream(s): {n / dt / 1e9:.1f} GB/s")
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dev[i * chunk:(i + 1) * chunk].copy_(host[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"H2D {ns} stream(s): {n / dt / 1e9:.1f} GB/s")

# the e2e pattern: two D2H copies per step (global 616 MB + local 453 MB), with and without a
# concurrent compute stream busy in the background
g = torch.empty(616 * 1024 * 1024, dtype=torch.uint8, device="cuda")
l_ = torch.empty(453 * 1024 * 1024, dtype=torch.uint8, device="cuda")
hg = torch.empty_like(g, device="cpu").pin_memory()
hl = torch.empty_like(l_, device="cpu").pin_memory()
cs, comp = torch.cuda.Stream(), torch.cuda.Stream()
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for busy in (False, True):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(10):
        if busy:
            with torch.cuda.stream(comp):
                for _ in range(20):
                    a = a @ a * 1e-4
        with torch.cuda.stream(cs):
            hg.copy_(g, non_blocking=True)
            hl.copy_(l_, non_blocking=True)
    cs.synchronize()
    dt = time.perf_counter() - t0
    torch.cuda.synchronize()
    print(f"e2e pattern busy={busy}: {10 * (g.numel() + l_.numel()) / dt / 1e9:.1f} GB/s")
