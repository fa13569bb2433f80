"""Round-2 goldens from the REAL reference (run in the build container, like make_goldens.py).

Covers the loader contract and the persistence formats:
* run_loader (pkg/pipeline.py:79-149) over a spec list with an out-of-bounds rect, an unknown
  slide, out_size 0, a down-ratio of 20 (PIL resize 60 -> 3) and an out_size of 600: ordered and
  unordered, on_error "skip" and "raise" -- emitted seqs + sha256 of every patch, LoaderRun.errors
  (seq, exception class), the seqs yielded before LoaderError and its cause's class;
* write_manifest / read_manifest (pkg/sampler.py:284-297): the manifest bytes;
* write_patch_pack (pkg/pipeline.py:158-205): sha256 of the u8 pack, the f32 pack of
  normalize_patch and the manifest sidecar.

Run: python tests/golden/make_goldens_r2.py  -> reference_goldens_r2.json
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

from make_goldens import import_reference  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def loader_specs(sampler):
    S = sampler.PatchSpec
    specs = [
        S("s0", 10, 20, 128, 128, 0.25, 128, 0),    # passthrough, 2x2 tiles
        S("s0", 301, 77, 96, 96, 0.5, 48, 1),       # level 1, passthrough
        S("s0", 40, 33, 124, 124, 0.97, 32, 2),     # resample at level 1 (+-1 px edge case region)
        S("s0", 650, 460, 50, 40, 0.25, 50, 3),     # OOB: y + h > 500
        S("nope", 0, 0, 32, 32, 0.25, 32, 4),       # unknown slide
        S("s0", 5, 5, 32, 32, 0.25, 0, 5),          # out_size 0 -> ValueError
        S("s0", 0, 0, 480, 480, 40.0, 3, 6),        # down-ratio 20: level 3 window of 60 -> 3
        S("s0", 100, 10, 480, 480, 0.2, 600, 7),    # out_size 600: level 0 window 480 -> 600
        S("s0", 596, 396, 64, 64, 1.7, 16, 8),      # level 2 window overruns both edges by 1 px
        S("s0", 0, 0, 496, 496, 2.0, 62, 9),        # passthrough at the coarsest level
        S("s0", 333, 222, 64, 64, 0.3, 77, 10),     # odd out size, level 0 resample
        S("s0", -1, 0, 16, 16, 0.25, 16, 11),       # negative origin -> OOB
        S("s0", 200, 300, 128, 128, 0.25, 128, 12),  # passthrough (packed with seq 0)
    ]
    return specs


def main():
    rng, store, foreground, sampler, pipeline = import_reference()
    out: dict = {}
    img = pipeline.synthetic_image(700, 500, seed=3)
    with tempfile.TemporaryDirectory() as td:
        store.ingest_image(img, "s0", 0.25, td, tile_size=128, downsample_factor=2, codec="raw", layout="packed")
        sl = store.open_slide(td, "s0")
        specs = loader_specs(sampler)
        out["loader_specs"] = [json.loads(s.to_json_line()) for s in specs]
        runs = {}
        for ordered in (True, False):
            for policy in ("skip", "raise"):
                cfg = pipeline.LoaderConfig(concurrency=3, prefetch_depth=5, ordered=ordered, on_error=policy)
                run = pipeline.run_loader(specs, {"s0": sl}, cfg)
                got, exc = [], None
                try:
                    for sp, px in run:
                        got.append([sp.seq, list(px.shape), sha(px)])
                except pipeline.LoaderError as e:
                    exc = {"class": type(e).__name__, "cause": type(e.__cause__).__name__, "message": str(e)}
                runs[f"{'ordered' if ordered else 'unordered'}/{policy}"] = {
                    "yielded": got if ordered else sorted(got),
                    "errors": [[f.spec.seq, type(f.error).__name__] for f in run.errors],
                    "raised": exc,
                }
        out["run_loader"] = runs
        # the patches themselves (for the pack goldens): the ordered/skip stream
        pix = [(sp, px) for sp, px in pipeline.run_loader([specs[0], specs[12]], {"s0": sl})]
    with tempfile.TemporaryDirectory() as td:
        man_specs = [sampler.PatchSpec("s0", 10 * i, 7 * i, 64, 64, 0.25 * (1 + i % 3), 32 + i, i) for i in range(6)]
        mp = Path(td) / "m.jsonl"
        n = sampler.write_manifest(man_specs, mp)
        out["manifest"] = {"n": n, "text": mp.read_text(encoding="utf-8"),
                           "specs": [json.loads(s.to_json_line()) for s in man_specs]}
        assert sampler.read_manifest(mp) == man_specs
        same = [(sp, px) for sp, px in pix if px.shape == pix[0][1].shape]
        u8 = np.stack([px for _, px in same])
        f32 = np.stack([pipeline.normalize_patch(px) for _, px in same])
        packs = {}
        for name, arr in (("u8", u8), ("f32", f32)):
            p = Path(td) / f"{name}.kpb"
            pipeline.write_patch_pack(arr, p, specs=[sp for sp, _ in same])
            packs[name] = {"sha256": hashlib.sha256(p.read_bytes()).hexdigest(),
                           "manifest_sha256": hashlib.sha256(Path(str(p) + ".manifest.jsonl").read_bytes()).hexdigest(),
                           "bytes": p.stat().st_size}
            back = pipeline.read_patch_pack(p)
            assert back.dtype == arr.dtype and np.array_equal(back, arr)
        out["patch_pack"] = {"seqs": [sp.seq for sp, _ in same], "packs": packs}
    (HERE / "reference_goldens_r2.json").write_text(json.dumps(out, indent=1))
    print("wrote", HERE / "reference_goldens_r2.json")


if __name__ == "__main__":
    main()
