"""Reference epoch_stream golden at BASELINE C2's full size (run offline, in the build container).

Inputs: tests/golden/c2_polygons.npz -- the saturation masks of the two 40000 x 30000 C2 test
slides (tests/test_gpu_fullsize.py, rendered on the B200 by tools/dump_c2_polygons.py) and the
rings the product traced from them.  This script

1. re-traces both masks with the REAL reference ``polygon_from_mask`` (pkg/foreground.py:169-220;
   ``skimage.measure.find_contours`` stubbed with the oracle's marching-squares restatement,
   scikit-image is not installed) and checks the rings equal the product's;
2. runs the REAL reference ``epoch_stream`` (pkg/sampler.py:196-227) for N_SPECS specs with
   seed 5, patch 224, min_foreground 0.40 on (SlideRecord, ForegroundPolygon) of both slides.

The reference's ``overlap_fraction`` costs seconds per candidate on these 18k-vertex polygons,
so candidate rects are pre-evaluated in a process pool -- each by the reference's own
``foreground.overlap_fraction`` (points_in_polygon over point chunks of 2048: per-point results
do not depend on the chunking) -- and served to ``sampler.overlap_fraction`` from that cache;
a rect the speculation missed is evaluated on the spot.  The stream itself is the reference's.

Run: python tests/golden/make_c2_stream_golden.py  -> tests/golden/c2_stream_golden.json
"""

from __future__ import annotations

import json
import math
import multiprocessing as mp
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent.parent))

N_SPECS = 256
SEED = 5
W, H = 40000, 30000

_REF = None


def _ref():
    global _REF
    if _REF is None:
        from make_goldens import import_reference

        _REF = import_reference()
        rng, store, foreground, sampler, pipeline = _REF
        whole = foreground.points_in_polygon

        def chunked(points, rings):
            pts = np.asarray(points, dtype=np.float64)
            return np.concatenate([whole(pts[i:i + 2048], rings) for i in range(0, len(pts), 2048)])

        foreground.points_in_polygon = chunked  # overlap_fraction looks it up in the module
    return _REF


def load():
    z = np.load(HERE / "c2_polygons.npz")
    out = []
    for g in range(2):
        bits = np.unpackbits(z[f"s{g}_mask"])[: int(np.prod(z[f"s{g}_mask_shape"]))].reshape(z[f"s{g}_mask_shape"])
        rings = [z[f"s{g}_ring{r}"] for r in range(int(z[f"s{g}_nrings"][0]))]
        out.append((bits.astype(bool), float(z[f"s{g}_scale"][0]), rings))
    return out


_POLYS = None


def _worker_init():
    global _POLYS
    rng, store, foreground, sampler, pipeline = _ref()
    _POLYS = [foreground.ForegroundPolygon(rings=rings, source_scale=sc, slide_id=f"s{g}")
              for g, (_, sc, rings) in enumerate(load())]


def _eval(job):
    g, rect = job
    rng, store, foreground, sampler, pipeline = _ref()
    return job, foreground.overlap_fraction(_POLYS[g], rect)


def record(store, sid):
    levels, w, h, ds = [], W, H, 1
    while True:
        levels.append(store.LevelInfo(w, h, 0.25 * ds, ds))
        if max(w, h) <= 256:
            break
        w, h, ds = math.ceil(w / 4), math.ceil(h / 4), ds * 4
    return store.SlideRecord(sid, 0.25, 256, levels)


def main():
    rng, store, foreground, sampler, pipeline = _ref()
    data = load()
    polys = []
    for g, (bits, sc, rings) in enumerate(data):
        ref_poly = foreground.polygon_from_mask(foreground.BinaryMask(bits, sc), slide_id=f"s{g}")
        assert len(ref_poly.rings) == len(rings), (g, len(ref_poly.rings), len(rings))
        for a, b in zip(ref_poly.rings, rings):
            assert np.array_equal(np.asarray(a), b), g
        polys.append(ref_poly)
    print("reference polygon_from_mask == product rings for both C2 masks")
    slides = [(record(store, f"s{g}"), polys[g]) for g in range(2)]
    cfg = sampler.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=[(0.25, 1.0)],
                                epoch_size=N_SPECS, seed=SEED)
    # speculation: global attempt a draws coords 2a+1, 2a+2 on whichever slide it lands on
    fp = 224
    jobs = []
    for a in range(int(N_SPECS / 0.38) + 48):
        for g, (rec, poly) in enumerate(slides):
            bx0, by0, bx1, by1 = poly.bounding_box()
            x_lo, y_lo = max(0, int(bx0)), max(0, int(by0))
            x_hi, y_hi = min(rec.width - fp, int(bx1)), min(rec.height - fp, int(by1))
            cs = rng.RandomStream(SEED, "coords")
            cs._counter = 2 * a
            x = cs.randint(x_lo, x_hi)
            y = cs.randint(y_lo, y_hi)
            jobs.append((g, (x, y, fp, fp)))
    t0 = time.time()
    cache = {}
    with mp.get_context("fork").Pool(8, initializer=_worker_init) as pool:
        for i, (job, frac) in enumerate(pool.imap_unordered(_eval, jobs, chunksize=4)):
            cache[job] = frac
            if i % 200 == 0:
                print(f"{i}/{len(jobs)} candidates, {time.time() - t0:.0f} s", flush=True)
    orig = foreground.overlap_fraction
    index = {p.slide_id: g for g, p in enumerate(polys)}
    misses = [0]

    def cached(poly, rect, grid=foreground.OVERLAP_GRID):
        key = (index[poly.slide_id], tuple(int(v) for v in rect))
        if grid == foreground.OVERLAP_GRID and key in cache:
            return cache[key]
        misses[0] += 1
        return orig(poly, rect, grid)

    sampler.overlap_fraction = cached
    specs = list(sampler.epoch_stream(cfg, slides))
    print(f"{len(specs)} specs, {misses[0]} cache misses, {time.time() - t0:.0f} s")
    out = {"seed": SEED, "patch_size": 224, "min_foreground": 0.40, "width": W, "height": H,
           "specs": [json.loads(s.to_json_line()) for s in specs],
           "accepted_fraction": [cache.get((index[s.slide_id], (s.x, s.y, s.width, s.height))) for s in specs]}
    (HERE / "c2_stream_golden.json").write_text(json.dumps(out))
    print("wrote", HERE / "c2_stream_golden.json")


if __name__ == "__main__":
    main()
