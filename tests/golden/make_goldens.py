"""Generate golden vectors by running the REAL reference (patchforge) in the build container.

Run: python tests/golden/make_goldens.py   (needs /root/reference; not available on GPU boxes)

scikit-image is not installed here, so ``skimage.measure.find_contours`` is
stubbed with the oracle's marching-squares restatement before import; every
other function is the reference's own code.  Outputs land next to this file
and are committed; the tests never read /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
import types
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle import port  # noqa: E402


def import_reference():
    sk = types.ModuleType("skimage")
    meas = types.ModuleType("skimage.measure")

    def find_contours(arr, level):
        assert level == 0.5
        return port.find_contours_binary(arr)

    meas.find_contours = find_contours
    sk.measure = meas
    sys.modules["skimage"] = sk
    sys.modules["skimage.measure"] = meas
    sys.path.insert(0, "/root/reference/pkg/src")
    import patchforge  # noqa: F401
    from patchforge import foreground, pipeline, rng, sampler, store

    return rng, store, foreground, sampler, pipeline


def blob_image(w: int, h: int, seed: int) -> np.ndarray:
    """H&E-like test image: pink/purple blobs on near-white (BASELINE look, small)."""
    rs = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:h, 0:w].astype(np.float64)
    f = np.zeros((h, w))
    for _ in range(10):
        cx, cy = rs.uniform(0, w), rs.uniform(0, h)
        s = rs.uniform(0.05, 0.18) * max(w, h)
        f += rs.uniform(0.4, 1.0) * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * s * s))
    f /= f.max()
    tissue = f > np.quantile(f, 0.6)
    img = np.empty((h, w, 3), np.float64)
    base = 240 + rs.normal(0, 4, (h, w, 3))
    img[:] = base
    t = np.clip((f - np.quantile(f, 0.6)) * 4, 0, 1)[..., None]
    col = np.array([220, 140, 210]) - t * np.array([70, 80, 70]) + rs.normal(0, 4, (h, w, 3))
    img = np.where(tissue[..., None], col, img)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def main():
    rng, store, foreground, sampler, pipeline = import_reference()
    out: dict = {}
    arrays: dict = {}

    # ---- rng (pkg/rng.py)
    r = {}
    for seed in (0, 1, 12345, (1 << 63) + 5):
        for purpose in ("slide", "coords", "mpp", "cache", "synthetic-image"):
            s = rng.RandomStream(seed, purpose)
            r[f"{seed}/{purpose}"] = [hex(s.next_u64()) for _ in range(8)]
    s = rng.RandomStream(7, "coords")
    r["randint_7"] = [s.randint(0, 7968) for _ in range(16)]
    s = rng.RandomStream(7, "mpp")
    r["weighted_7"] = [s.weighted_index([1.0, 2.0, 0.5, 0.0, 3.0]) for _ in range(32)]
    s = rng.RandomStream(3, "slide")
    r["randrange3_7"] = [s.randrange(7) for _ in range(32)]
    out["rng"] = r

    # ---- store (pkg/store.py): ingest + select_level + read_region + thumbnail
    img = pipeline.synthetic_image(700, 500, seed=3)
    arrays["synthetic_700x500"] = img
    rs = np.random.default_rng(11)
    reads = []
    with tempfile.TemporaryDirectory() as td:
        rec = store.ingest_image(img, "s0", 0.25, td, tile_size=128, downsample_factor=2, codec="raw", layout="packed")
        sl = store.open_slide(td, "s0")
        out["levels_f2_t128"] = [(lv.width, lv.height, lv.mpp, lv.downsample) for lv in rec.levels]
        for li in range(len(rec.levels)):
            lv = rec.levels[li]
            arrays[f"level_f2_{li}"] = sl._read_window(li, 0, 0, lv.width, lv.height)
        th, sc = sl.thumbnail()
        arrays["thumb_f2"] = th
        out["thumb_f2_scale"] = sc
        for k in range(48):
            out_size = int(rs.choice([16, 32, 48, 64]))
            mpp = float(rs.choice([0.25, 0.25, 0.3, 0.5, 0.6, 0.97, 1.0, 1.7, 2.0]))
            fp = max(1, store.round_half_away(out_size * mpp / 0.25))
            if fp > 480:
                out_size = 16
                fp = max(1, store.round_half_away(out_size * mpp / 0.25))
            x = int(rs.integers(0, 700 - fp + 1))
            y = int(rs.integers(0, 500 - fp + 1))
            px = sl.read_region((x, y, fp, fp), mpp, out_size)
            arrays[f"read_{k}"] = px
            reads.append({"k": k, "rect": [x, y, fp, fp], "mpp": mpp, "out": out_size,
                          "level": sl.select_level(mpp)})
    with tempfile.TemporaryDirectory() as td:
        rec4 = store.ingest_image(img, "s1", 0.25, td, tile_size=64, downsample_factor=4, codec="raw", layout="files")
        out["levels_f4_t64"] = [(lv.width, lv.height, lv.mpp, lv.downsample) for lv in rec4.levels]
        sl4 = store.open_slide(td, "s1")
        arrays["level_f4_1"] = sl4._read_window(1, 0, 0, rec4.levels[1].width, rec4.levels[1].height)
    out["reads"] = reads
    lvl = store.SlideRecord("x", 0.25, 256, [store.LevelInfo(1000, 1000, 0.25, 1), store.LevelInfo(250, 250, 1.0, 4),
                                              store.LevelInfo(63, 63, 4.0, 16)])
    out["select_level"] = {str(t): store.select_level(lvl, t) for t in (0.1, 0.25, 0.3, 0.5, 0.97, 1.0, 2.0, 3.9, 8.0, 64.0)}
    out["box32_700x500"] = None
    arrays["box32_700x500"] = store._box_downsample(img, 32)
    arrays["box7_700x500"] = store._box_downsample(img, 7)

    # ---- foreground (pkg/foreground.py)
    blob = blob_image(640, 480, seed=5)
    arrays["blob_640x480"] = blob
    thumb = store._box_downsample(blob, 8)  # 80 x 60
    arrays["blob_thumb8"] = thumb
    m = foreground.mask_from_rgb(thumb, 0.9, scale=1.0 / 8)
    arrays["blob_mask_lum"] = m.bits
    allc = np.arange(1 << 24, dtype=np.uint32)
    rgb = np.stack([(allc >> 16) & 255, (allc >> 8) & 255, allc & 255], axis=1).astype(np.uint8).reshape(4096, 4096, 3)
    for thr in (0.9, 0.5, 0.25):
        bits = foreground.mask_from_rgb(rgb, thr).bits
        out[f"allcolors_lum_{thr}_sha256"] = hashlib.sha256(np.packbits(bits).tobytes()).hexdigest()
    poly = foreground.polygon_from_mask(m, slide_id="blob")
    out["blob_poly"] = poly.to_json_dict()
    # hand-made mask with a hole, saddles and a small island
    hm = np.zeros((40, 50), bool)
    hm[5:30, 5:40] = True
    hm[8:14, 8:16] = False  # hole (off-centre: the reference probes with the ring mean)
    hm[22, 30] = False
    hm[32:38, 2:12] = True  # island touching nothing
    hm[30, 40] = True  # diagonal saddle neighbour
    hm[0:4, 44:50] = True  # border-touching region
    arrays["hand_mask"] = hm
    hpoly = foreground.polygon_from_mask(foreground.BinaryMask(hm, 0.5), min_region_px=4, slide_id="hand")
    out["hand_poly"] = hpoly.to_json_dict()
    ov = []
    bx0, by0, bx1, by1 = poly.bounding_box()
    for k in range(40):
        w = float(rs.choice([16, 40, 64, 96, 150]))
        x = float(rs.integers(int(bx0) - 40, int(bx1)))
        y = float(rs.integers(int(by0) - 40, int(by1)))
        ov.append([x, y, w, w, foreground.overlap_fraction(poly, (x, y, w, w))])
    out["blob_overlap"] = ov
    hov = []
    for k in range(20):
        w = float(rs.choice([3, 7, 12, 25]))
        x = float(rs.uniform(-5, 100))
        y = float(rs.uniform(-5, 80))
        hov.append([x, y, w, w * 0.75, foreground.overlap_fraction(hpoly, (x, y, w, w * 0.75), grid=64)])
    out["hand_overlap_grid64"] = hov
    rp = foreground.rect_polygon(0, 0, 100, 100)
    out["rect_kats"] = [foreground.overlap_fraction(rp, (10, 10, 20, 20)), foreground.overlap_fraction(rp, (200, 200, 20, 20)),
                        foreground.overlap_fraction(rp, (90, 10, 20, 20))]

    # ---- sampler (pkg/sampler.py): epoch_stream manifests
    recs = []
    slides = []
    for i, (w, h, seed) in enumerate([(640, 480, 5), (512, 512, 6), (800, 300, 7)]):
        b = blob_image(w, h, seed)
        t = store._box_downsample(b, 8)
        mm = foreground.mask_from_rgb(t, 0.9, scale=1.0 / 8)
        pg = foreground.polygon_from_mask(mm, slide_id=f"b{i}")
        rec = store.SlideRecord(f"b{i}", 0.25, 128, [store.LevelInfo(w, h, 0.25, 1)])
        recs.append(rec)
        slides.append((rec, pg))
        out[f"sampler_poly_b{i}"] = pg.to_json_dict()
        out[f"sampler_dims_b{i}"] = [w, h]
    cases = {
        "single": dict(cfg=sampler.SamplerConfig(patch_size=32, epoch_size=60, seed=0), slides=[0]),
        "single_seed9": dict(cfg=sampler.SamplerConfig(patch_size=48, epoch_size=40, seed=9, min_foreground=0.7), slides=[0]),
        "multi_mpp": dict(cfg=sampler.SamplerConfig(patch_size=16, epoch_size=60, seed=3,
                                                    target_mpps=[(0.25, 1.0), (0.5, 1.0), (1.0, 1.0), (2.0, 1.0)]),
                          slides=[0, 1, 2]),
        "weighted": dict(cfg=sampler.SamplerConfig(patch_size=24, epoch_size=50, seed=4, slide_strategy="weighted",
                                                   slide_weights={"b0": 1.0, "b1": 0.0, "b2": 3.0}), slides=[0, 1, 2]),
        # footprints that do not fit some slides' bbox ranges (big patch on the 800x300 slide)
        "nofit": dict(cfg=sampler.SamplerConfig(patch_size=100, epoch_size=30, seed=5,
                                                target_mpps=[(0.25, 1.0), (0.75, 1.0)]), slides=[0, 2]),
        # a high threshold forces exhausted draws
        "exhaust": dict(cfg=sampler.SamplerConfig(patch_size=64, epoch_size=12, seed=6, min_foreground=0.97,
                                                  max_attempts_per_slide=20), slides=[0, 1]),
    }
    man = {}
    for name, c in cases.items():
        ss = [slides[i] for i in c["slides"]]
        specs = list(sampler.epoch_stream(c["cfg"], ss))
        man[name] = {"slides": c["slides"], "cfg": {k: getattr(c["cfg"], k) for k in (
            "patch_size", "min_foreground", "target_mpps", "slide_strategy", "slide_weights", "epoch_size", "seed",
            "max_attempts_per_slide")}, "specs": [json.loads(s.to_json_line()) for s in specs]}
    out["epoch_streams"] = man

    # ---- capped replay (pkg/sampler.py:230-281) over the multi_mpp stream
    base = [sampler.PatchSpec(**d) for d in man["multi_mpp"]["specs"]]
    cap = {}
    for c, total, seed in ((7, 40, 13), (1, 9, 2), (25, 60, 13), (None, 20, 13)):
        got = list(sampler.capped_stream(iter(base), c, rng.RandomStream(seed, "cache"), total=total))
        cap[f"{c}/{total}/{seed}"] = [s.seq for s in got]
    out["capped_streams"] = cap

    # ---- ingest_image on-disk format (pkg/store.py:462-565): sha256 of every written file
    ing = {}
    for codec, layout in (("raw", "packed"), ("png", "files"), ("jpeg", "packed")):
        with tempfile.TemporaryDirectory() as td:
            store.ingest_image(img, "s0", 0.25, td, tile_size=128, downsample_factor=2, codec=codec, layout=layout)
            ing[f"{codec}/{layout}"] = {str(p.relative_to(td)): hashlib.sha256(p.read_bytes()).hexdigest()
                                        for p in sorted(Path(td).rglob("*")) if p.is_file()}
    out["ingest_sha256"] = ing

    # ---- pipeline
    out["normalize"] = [float(v) for v in pipeline.normalize_patch(np.array([0, 255, 128, 1, 254], np.uint8))]

    (HERE / "reference_goldens.json").write_text(json.dumps(out, indent=1, default=float))
    np.savez_compressed(HERE / "reference_arrays.npz", **arrays)
    print("wrote", HERE / "reference_goldens.json", HERE / "reference_arrays.npz")


if __name__ == "__main__":
    main()
