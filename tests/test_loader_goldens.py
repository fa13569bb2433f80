"""run_loader (pkg/pipeline.py:79-149), manifests (pkg/sampler.py:284-297) and KPB1 packs
(pkg/pipeline.py:158-205) against goldens from the real reference (tests/golden/make_goldens_r2.py).

CPU: manifest text and pack bytes (host I/O).  GPU: run_loader over the reference's spec list --
ordered and unordered, skip and raise -- with out-of-bounds rects, an unknown slide, out_size 0, a
down-ratio of 20 and out_size 600 (the generic PIL path), and normalize_patch into the f32 pack.
"""

import hashlib
import json

import numpy as np
import pytest

from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def g2():
    return json.loads((GOLDEN / "reference_goldens_r2.json").read_text())


def _specs(pf, rows):
    return [pf.PatchSpec(**d) for d in rows]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _pack_patches(golden_arrays, g2):
    img = golden_arrays["synthetic_700x500"]
    spec = {d["seq"]: d for d in g2["loader_specs"]}
    out = []
    for q in g2["patch_pack"]["seqs"]:  # passthrough specs at 0.25 mpp: the rect itself
        d = spec[q]
        out.append(img[d["y"]:d["y"] + d["height"], d["x"]:d["x"] + d["width"]])
    return np.stack(out)


def test_manifest_text_matches_reference(g2, tmp_path):
    import paper_2404_15217_b200 as pf

    specs = _specs(pf, g2["manifest"]["specs"])
    p = tmp_path / "m.jsonl"
    assert pf.write_manifest(specs, p) == g2["manifest"]["n"]
    assert p.read_text(encoding="utf-8") == g2["manifest"]["text"]
    assert pf.read_manifest(p) == specs


def test_patch_pack_bytes_match_reference(g2, golden_arrays, tmp_path):
    import paper_2404_15217_b200 as pf

    u8 = _pack_patches(golden_arrays, g2)
    specs = [s for s in _specs(pf, g2["loader_specs"]) if s.seq in g2["patch_pack"]["seqs"]]
    f32 = (u8.astype(np.float32) / np.float32(255.0) - np.float32(0.5)) / np.float32(0.5)  # normalize_patch
    for name, arr in (("u8", u8), ("f32", f32)):
        p = tmp_path / f"{name}.kpb"
        pf.write_patch_pack(arr, p, specs=specs)
        want = g2["patch_pack"]["packs"][name]
        assert hashlib.sha256(p.read_bytes()).hexdigest() == want["sha256"]
        assert hashlib.sha256((tmp_path / f"{name}.kpb.manifest.jsonl").read_bytes()).hexdigest() == want["manifest_sha256"]
        back = pf.read_patch_pack(p)
        assert back.dtype == arr.dtype and np.array_equal(back, arr)


def test_patch_pack_rejects_malformed(tmp_path):
    import paper_2404_15217_b200 as pf
    from paper_2404_15217_b200.errors import PackFormatError

    p = tmp_path / "bad.kpb"
    p.write_bytes(b"KPB")
    with pytest.raises(PackFormatError):
        pf.read_patch_pack(p)
    p.write_bytes(b"XXXX" + bytes(16))
    with pytest.raises(PackFormatError):
        pf.read_patch_pack(p)
    with pytest.raises(PackFormatError):
        pf.write_patch_pack(np.zeros((2, 4, 5, 3), np.uint8), tmp_path / "x.kpb")


@pytest.fixture(scope="module")
def slide(cuda, golden_arrays):
    import paper_2404_15217_b200 as pf

    return pf.GpuSlide.from_array(golden_arrays["synthetic_700x500"], "s0", 0.25, tile_size=128, downsample_factor=2)


def _run(pf, specs, slide, ordered, policy):
    cfg = pf.LoaderConfig(concurrency=3, prefetch_depth=5, ordered=ordered, on_error=policy)
    run = pf.run_loader(specs, {"s0": slide}, cfg)
    got, exc = [], None
    try:
        for sp, px in run:
            got.append([sp.seq, list(px.shape), _sha(px)])
    except pf.LoaderError as e:
        exc = {"class": type(e).__name__, "cause": type(e.__cause__).__name__, "message": str(e)}
    return got, [[f.spec.seq, type(f.error).__name__] for f in run.errors], exc


@pytest.mark.gpu
@pytest.mark.parametrize("ordered", [True, False])
@pytest.mark.parametrize("policy", ["skip", "raise"])
def test_run_loader_matches_reference(g2, slide, ordered, policy):
    import paper_2404_15217_b200 as pf

    specs = _specs(pf, g2["loader_specs"])
    want = g2["run_loader"][f"{'ordered' if ordered else 'unordered'}/{policy}"]
    got, errors, exc = _run(pf, specs, slide, ordered, policy)
    if ordered:  # every patch byte-identical, in order; failures at their positions
        assert got == want["yielded"]
        assert errors == want["errors"]
        if want["raised"] is None:
            assert exc is None
        else:
            assert {k: exc[k] for k in ("class", "cause")} == {k: want["raised"][k] for k in ("class", "cause")}
            assert exc["message"].startswith(want["raised"]["message"].split(":")[0])
    else:  # completion order: the same sets
        if policy == "skip":
            assert sorted(got) == sorted(want["yielded"])
            assert sorted(errors) == sorted(want["errors"])
        else:
            ok = {q for q, _, _ in g2["run_loader"]["ordered/skip"]["yielded"]}
            bad = dict((q, c) for q, c in g2["run_loader"]["ordered/skip"]["errors"])
            assert {q for q, _, _ in got} <= ok and exc is not None
            assert exc["cause"] in set(bad.values())


@pytest.mark.gpu
def test_loader_exactly_once_and_ordered_equals_serial(g2, slide):
    """every spec exactly once; ordered output == serial read_region order."""
    import paper_2404_15217_b200 as pf

    specs = [s for s in _specs(pf, g2["loader_specs"]) if s.seq in {0, 1, 2, 6, 7, 8, 9, 10, 12}] * 3
    specs = [pf.PatchSpec(s.slide_id, s.x, s.y, s.width, s.height, s.target_mpp, s.out_size, i)
             for i, s in enumerate(specs)]
    got = list(pf.run_loader(specs, slide, pf.LoaderConfig(prefetch_depth=8), batch=7))
    assert [sp.seq for sp, _ in got] == list(range(len(specs)))
    for sp, px in got:
        assert np.array_equal(px, slide.read_region(sp.rect(), sp.target_mpp, sp.out_size))


@pytest.mark.gpu
def test_normalized_pack_matches_reference(g2, golden_arrays, slide, tmp_path):
    import paper_2404_15217_b200 as pf

    specs = [s for s in _specs(pf, g2["loader_specs"]) if s.seq in g2["patch_pack"]["seqs"]]
    pix = np.stack([px for _, px in pf.run_loader(specs, slide)])
    assert np.array_equal(pix, _pack_patches(golden_arrays, g2))
    f32 = pf.normalize_patch(pix)
    p = tmp_path / "f32.kpb"
    pf.write_patch_pack(f32, p, specs=specs)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == g2["patch_pack"]["packs"]["f32"]["sha256"]
