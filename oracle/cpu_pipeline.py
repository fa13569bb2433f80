"""CPU reference pipeline for bench.py's cpu_baseline / --impl reference legs (TEST INFRASTRUCTURE ONLY).

Runs the reference algorithm restated in oracle/port.py on the host cores:
epoch_stream candidates with the numpy even-odd overlap test (pkg/sampler.py,
pkg/foreground.py), read_region over a tiled level-0 store (pkg/store.py),
then the torchvision multi-crop (not reference code: the reference has no
augmentation) and ImageNet normalisation to bf16.

Slides: the same BASELINE synthetic generator as the GPU arm, restated in numpy
and rendered tile by tile on first touch (cached), the way the reference
decodes tiles on first touch into its TileCache.  Masks come from the smooth
field sampled at the 1/32 thumbnail resolution (setup; not timed).
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from . import augment as A
from . import port

TILE = 256
FIELD_CELL = 64
M64 = np.uint64((1 << 64) - 1)


def _mix64_np(x):
    with np.errstate(over="ignore"):
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def _hash_normal(seed, idx, which):
    with np.errstate(over="ignore"):
        h = _mix64_np(np.uint64(seed) ^ _mix64_np(idx * np.uint64(3) + np.uint64(which) + np.uint64(0x51ED2701)))
    u1 = ((h >> np.uint64(40)).astype(np.float32) + np.float32(0.5)) * np.float32(1.0 / 16777216.0)
    u2 = (h & np.uint64(0xFFFFFF)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(np.float32(6.28318530718) * u2)


class ProceduralSlide:
    """Level-0 tiles rendered on first touch from the synthetic field (numpy restatement of pf_synth)."""

    def __init__(self, width, height, seed, coverage=0.40, blob_px=2048.0, cache_tiles=4096):
        from paper_2404_15217_b200.synthetic import tissue_field  # host-only numpy helper (no GPU)

        self.width, self.height, self.seed = width, height, seed
        self.field, self.thr = tissue_field(width, height, seed, coverage, blob_px)
        self.cache: dict = {}
        self.cache_tiles = cache_tiles

    def _sample_field(self, X, Y):
        fh, fw = self.field.shape
        fx = np.clip((X.astype(np.float32) + 0.5) / FIELD_CELL - 0.5, 0, fw - 1)
        fy = np.clip((Y.astype(np.float32) + 0.5) / FIELD_CELL - 0.5, 0, fh - 1)
        x0, y0 = np.minimum(fx.astype(np.int64), fw - 1), np.minimum(fy.astype(np.int64), fh - 1)
        x1, y1 = np.minimum(x0 + 1, fw - 1), np.minimum(y0 + 1, fh - 1)
        ax, ay = fx - x0, fy - y0
        f = self.field
        return (f[y0, x0] * (1 - ax) + f[y0, x1] * ax) * (1 - ay) + (f[y1, x0] * (1 - ax) + f[y1, x1] * ax) * ay

    def tile(self, tx, ty):
        key = (tx, ty)
        t = self.cache.get(key)
        if t is not None:
            return t
        ys, xs = np.mgrid[ty * TILE:(ty + 1) * TILE, tx * TILE:(tx + 1) * TILE]
        f = self._sample_field(xs, ys)
        idx = ys.astype(np.uint64) * np.uint64(self.width) + xs.astype(np.uint64)
        n = [4.0 * _hash_normal(self.seed, idx, k) for k in range(3)]
        thr = self.thr
        t_ = np.minimum((f - thr) / max(1.0 - thr, 1e-6) * 2.5, 1.0)
        base = 230.0 + 20.0 * np.clip(f / max(thr, 1e-6), 0, 1)
        tissue = f > thr
        out = np.empty((TILE, TILE, 3), np.uint8)
        for c, (a, b) in enumerate(((220.0, 70.0), (140.0, 80.0), (210.0, 70.0))):
            v = np.where(tissue, a - b * t_ + n[c], base + n[c])
            out[..., c] = np.clip(np.rint(v), 0, 255).astype(np.uint8)
        if len(self.cache) >= self.cache_tiles:
            self.cache.pop(next(iter(self.cache)))
        self.cache[key] = out
        return out

    def read_region224(self, x, y, side=224):
        """read_region at level 0, passthrough (pkg/store.py:651-724, tile assembly loop)."""
        out = np.empty((side, side, 3), np.uint8)
        for ty in range(y // TILE, (y + side - 1) // TILE + 1):
            for tx in range(x // TILE, (x + side - 1) // TILE + 1):
                t = self.tile(tx, ty)
                ix0, iy0 = max(x, tx * TILE), max(y, ty * TILE)
                ix1, iy1 = min(x + side, (tx + 1) * TILE), min(y + side, (ty + 1) * TILE)
                out[iy0 - y:iy1 - y, ix0 - x:ix1 - x] = t[iy0 - ty * TILE:iy1 - ty * TILE, ix0 - tx * TILE:ix1 - tx * TILE]
        return out

    def polygon(self):
        """Field-derived tissue mask on the 1/32 thumbnail grid -> reference polygon_from_mask."""
        h, w = -(-self.height // 32), -(-self.width // 32)
        ys, xs = np.mgrid[0:h, 0:w]
        f = self._sample_field(xs * 32 + 16, ys * 32 + 16)
        return port.polygon_from_mask(f > self.thr, 1.0 / 32, 64.0)


def points_in_polygon_chunked(points, rings, chunk=2048):
    out = np.empty(points.shape[0], bool)
    for i in range(0, points.shape[0], chunk):
        out[i:i + chunk] = port.points_in_polygon(points[i:i + chunk], rings)
    return out


def overlap_fraction(rings, bbox, rect, grid=128):
    """port.overlap_fraction with the point set processed in chunks (bounded memory, same result)."""
    x, y, w, h = rect
    bx0, by0, bx1, by1 = bbox
    if x >= bx1 or y >= by1 or x + w <= bx0 or y + h <= by0:
        return 0.0
    ex = x + np.arange(grid + 1) * (w / grid)
    ey = y + np.arange(grid + 1) * (h / grid)
    gx, gy = np.meshgrid(ex, ey, indexing="xy")
    corners = points_in_polygon_chunked(np.stack([gx.ravel(), gy.ravel()], 1), rings).reshape(grid + 1, grid + 1)
    cx, cy = (ex[:-1] + ex[1:]) / 2.0, (ey[:-1] + ey[1:]) / 2.0
    mx, my = np.meshgrid(cx, cy, indexing="xy")
    centres = points_in_polygon_chunked(np.stack([mx.ravel(), my.ravel()], 1), rings).reshape(grid, grid)
    cov = corners[:-1, :-1] & corners[1:, :-1] & corners[:-1, 1:] & corners[1:, 1:] & centres
    return float(cov.sum()) / float(grid * grid)


class Worker:
    """One reference worker: seed + worker_index streams (pkg/sampler.py:5-7) over all slides."""

    def __init__(self, slides, polys, seed, patch=224, min_fg=0.40, max_attempts=100):
        self.slides, self.polys = slides, polys
        self.bboxes = [port.bounding_box(p) for p in polys]
        self.s_slide, self.s_coords, self.s_mpp = port.Stream(seed, "slide"), port.Stream(seed, "coords"), port.Stream(seed, "mpp")
        self.patch, self.min_fg, self.max_attempts = patch, min_fg, max_attempts
        self.cur, self.used = None, 0
        self.candidates = 0

    def candidate(self):
        """One sample_patch attempt (pkg/sampler.py:159-180); returns a spec or None."""
        if self.cur is None or self.used >= self.max_attempts:
            self.cur, self.used = self.s_slide.randrange(len(self.slides)), 0
        si = self.cur
        sl = self.slides[si]
        bx0, by0, bx1, by1 = self.bboxes[si]
        self.s_mpp.weighted_index([1.0])
        self.used += 1
        self.candidates += 1
        fp = self.patch
        x = self.s_coords.randint(max(0, int(bx0)), min(sl.width - fp, int(bx1)))
        y = self.s_coords.randint(max(0, int(by0)), min(sl.height - fp, int(by1)))
        if overlap_fraction(self.polys[si], self.bboxes[si], (x, y, fp, fp)) >= self.min_fg:
            self.cur = None
            return (si, x, y)
        return None


def augment_patch(src, rs, mean, std):
    """torchvision DINOv2 multi-crop of one patch (2 x 224 + 8 x 96), bf16 outputs."""
    import torch

    outs = []
    for c in range(10):
        g = c < 2
        s0, s1 = (0.32, 1.0) if g else (0.05, 0.32)
        area = 224 * 224 * rs.uniform(s0, s1)
        ar = math.exp(rs.uniform(math.log(3 / 4), math.log(4 / 3)))
        w = min(224, max(1, int(round(math.sqrt(area * ar)))))
        h = min(224, max(1, int(round(math.sqrt(area / ar)))))
        p = {"top": int(rs.integers(0, 224 - h + 1)), "left": int(rs.integers(0, 224 - w + 1)), "height": h, "width": w,
             "out_size": 224 if g else 96, "order": list(rs.permutation(4)), "brightness": rs.uniform(0.6, 1.4),
             "contrast": rs.uniform(0.6, 1.4), "saturation": rs.uniform(0.8, 1.2), "hue": rs.uniform(-0.1, 0.1),
             "sigma": rs.uniform(0.1, 2.0), "solarize_threshold": 128.0}
        fl = 0
        fl |= A.AUG_FLIP if rs.random() < 0.5 else 0
        fl |= A.AUG_JITTER if rs.random() < 0.8 else 0
        fl |= A.AUG_GRAY if rs.random() < 0.2 else 0
        fl |= A.AUG_BLUR if rs.random() < (1.0, 0.1, 0.5, 0.5, 0.5, 0.5, 0.5, 0.5, 0.5, 0.5)[c] else 0
        fl |= A.AUG_SOLARIZE if (c == 1 and rs.random() < 0.2) else 0
        p["flags"] = fl
        u8 = A.torchvision_crop(src, p)
        outs.append(torch.from_numpy(A.normalize(u8, mean, std)).permute(2, 0, 1).to(torch.bfloat16))
    return outs


def _worker_main(args):
    """Process worker: build its slides, then per step time the three stages BASELINE.md §4 asks for:
    sampler (`candidates` epoch_stream attempts), loader (read_region + normalize_patch over a
    manifest of `loads` rects, `patchforge load` semantics) and augmentation (torchvision multi-crop
    of `augs` patches, not reference code)."""
    (wid, seed, n_slides, width, height, candidates, steps, mean, std, q, polys, augment, loads, augs) = args
    import torch

    torch.set_num_threads(1)
    slides = [ProceduralSlide(width, height, 1000 + i) for i in range(n_slides)]
    augment_patch(np.zeros((224, 224, 3), np.uint8), np.random.default_rng(0), mean, std)  # warm imports
    w = Worker(slides, polys, seed + wid)
    rs = np.random.default_rng(seed + wid)
    q.put(("ready", wid, 0, None, 0))
    for step in range(steps):
        # sampler
        t0 = time.perf_counter()
        made = 0
        for _ in range(candidates):
            if w.candidate() is not None:
                made += 1
        ts = time.perf_counter() - t0
        # loader over a pre-sampled manifest (uniform level-0 rects: read cost does not depend on them)
        man = [(int(rs.integers(n_slides)), int(rs.integers(0, width - 224)), int(rs.integers(0, height - 224)))
               for _ in range(loads)]
        t0 = time.perf_counter()
        pix = []
        for si, x, y in man:
            px = slides[si].read_region224(x, y)
            np.ascontiguousarray(port.normalize_patch(px, mean, std).transpose(2, 0, 1))
            pix.append(px)
        tl = time.perf_counter() - t0
        # augmentation (config 1 has none)
        ta = 0.0
        if augment:
            t0 = time.perf_counter()
            for px in pix[:augs]:
                augment_patch(px, rs, mean, std)
            ta = time.perf_counter() - t0
        q.put(("step", wid, step, (ts, made, tl, len(man), ta, min(augs, len(pix)) if augment else 0), 0))
    q.put(("done", wid, 0, None, w.candidates))


def _slide_polygon(a):
    w, h, seed = a
    return ProceduralSlide(w, h, seed).polygon()


def run(n_workers, n_slides, width, height, candidates_per_step, steps, seed=0, mean=(0.485, 0.456, 0.406),
        std=(0.229, 0.224, 0.225), augment=True, loads_per_step=48, augs_per_step=4, polygons=None):
    """Per-step stage timings aggregated over the worker pool.  Returns (steps, total candidates),
    each step a dict: sampler (seconds, accepted), loader (seconds, patches), augment (seconds,
    patches) -- the max over workers of each stage's time and the sum of its units.
    ``polygons``: rings per slide (e.g. the GPU arm's traced polygons); default: the field mask."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    if polygons is None:
        with ctx.Pool(min(n_workers, n_slides)) as pool:
            polys = pool.map(_slide_polygon, [(width, height, 1000 + i) for i in range(n_slides)])
    else:
        polys = [[np.asarray(r, dtype=np.float64) for r in p] for p in polygons]
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_main, args=((i, seed, n_slides, width, height, candidates_per_step, steps, mean,
                                                    std, q, polys, augment, loads_per_step, augs_per_step),))
             for i in range(n_workers)]
    for p in procs:
        p.start()
    ready = 0
    while ready < n_workers:
        if q.get()[0] == "ready":
            ready += 1
    per_step: dict = {}
    done = 0
    total_cands = 0
    while done < n_workers:
        kind, wid, step, st, made = q.get()
        if kind == "step":
            ts, acc, tl, nl, ta, na = st
            agg = per_step.setdefault(step, {"sampler": [0.0, 0], "loader": [0.0, 0], "augment": [0.0, 0]})
            for k, (t, m) in (("sampler", (ts, acc)), ("loader", (tl, nl)), ("augment", (ta, na))):
                agg[k][0] = max(agg[k][0], t)
                agg[k][1] += m
        elif kind == "done":
            done += 1
            total_cands += made
    for p in procs:
        p.join()
    return [per_step[s] for s in sorted(per_step)], total_cands


def summarize(steps, cores, candidates, augment=True):
    """Stage rates (patches/s over all workers) and the end-to-end rate of a worker running the three
    stages per patch: 1 / (1/sampler + 1/loader + 1/augment)."""
    def rate(k):
        t = sum(s[k][0] for s in steps)
        n = sum(s[k][1] for s in steps)
        return (n / t if t > 0 else 0.0), n, t

    rs, ns, tsam = rate("sampler")
    rl, nl, tl = rate("loader")
    ra, na, ta = rate("augment") if augment else (float("inf"), 0, 0.0)
    inv = (1.0 / rs if rs > 0 else float("inf")) + 1.0 / rl + (1.0 / ra if augment else 0.0)
    e2e = 1.0 / inv if inv < float("inf") else 0.0
    stages = {"sampler": {"value": round(rs, 4), "unit": "specs/s", "specs": ns, "seconds": round(tsam, 2),
                          "what": "reference epoch_stream attempts (numpy even-odd overlap, 128x128 lattice)"},
              "loader": {"value": round(rl, 1), "unit": "patches/s", "patches": nl, "seconds": round(tl, 2),
                         "what": "read_region 224 passthrough + normalize_patch over a manifest (patchforge load)"}}
    if augment:
        stages["augment"] = {"value": round(ra, 2), "unit": "patches/s", "patches": na, "seconds": round(ta, 2),
                             "what": "torchvision v2 multi-crop 2x224+8x96 bf16 (NOT reference code)"}
    return e2e, stages


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_count():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
