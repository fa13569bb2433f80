"""GPU parity: the device epoch_stream reproduces the reference's spec stream bit-exactly."""

import numpy as np
import pytest

from oracle import port

pytestmark = pytest.mark.gpu

CASES = ["single", "single_seed9", "multi_mpp", "weighted", "nofit", "exhaust"]


@pytest.fixture(scope="module")
def pf(cuda):
    import paper_2404_15217_b200 as pf

    return pf


def _slides(pf, goldens, idx):
    out = []
    for i in idx:
        w, h = goldens[f"sampler_dims_b{i}"]
        rec = pf.store.make_record(f"b{i}", w, h, 0.25, tile_size=128, downsample_factor=2)
        out.append((rec, pf.ForegroundPolygon.from_json_dict(goldens[f"sampler_poly_b{i}"])))
    return out


def _cfg(pf, c):
    d = dict(c["cfg"])
    d["target_mpps"] = [tuple(m) for m in d["target_mpps"]]
    return pf.SamplerConfig(**d)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("batch", [7, 64])
def test_epoch_stream_matches_reference(pf, goldens, case, batch):
    c = goldens["epoch_streams"][case]
    got = list(pf.epoch_stream(_cfg(pf, c), _slides(pf, goldens, c["slides"]), batch=batch))
    want = [pf.PatchSpec(**s) for s in c["specs"]]
    assert got == want


@pytest.mark.parametrize("window,rounds", [(32, 1), (64, 2), (4096, 4), (None, 0)])
def test_window_and_round_settings_do_not_change_stream(pf, goldens, window, rounds):
    c = goldens["epoch_streams"]["multi_mpp"]
    smp = pf.GpuSampler(_cfg(pf, c), _slides(pf, goldens, c["slides"]), window=window, rounds=rounds)
    got = []
    for n in (5, 17, 38):
        got += smp.to_patch_specs(smp.next_batch(n))
    assert got == [pf.PatchSpec(**s) for s in c["specs"]]
    st = smp.check()
    assert st.seq == 60


def test_long_stream_vs_oracle(pf, goldens):
    """A longer stream (300 specs, 3 slides, 2 mpps) against the CPU oracle."""
    slides = _slides(pf, goldens, [0, 1, 2])
    cfg = pf.SamplerConfig(patch_size=32, epoch_size=300, seed=21, target_mpps=[(0.25, 2.0), (0.5, 1.0)])
    got = list(pf.epoch_stream(cfg, slides, batch=128))
    orc = [{"id": r.slide_id, "width": r.width, "height": r.height, "base_mpp": 0.25, "rings": p.rings} for r, p in slides]
    want, _ = port.epoch_stream(orc, patch_size=32, min_fg=0.4, mpps=[(0.25, 2.0), (0.5, 1.0)], seed=21, epoch_size=300)
    assert [(s.slide_id, s.x, s.y, s.width, s.target_mpp, s.seq) for s in got] == \
        [(orc[si]["id"], x, y, fp, m, q) for si, x, y, fp, m, q in want]


@pytest.mark.parametrize("batch", [64, 300])
def test_stream_with_frequent_exhaustion_vs_oracle(pf, goldens, batch):
    """max_attempts 3: draws exhaust in the middle of a batch, so the walk's table loop hands
    over to its general step and back many times per call (a stale "specs still wanted" count
    there once over-emitted); against the CPU oracle."""
    slides = _slides(pf, goldens, [0, 1, 2])
    cfg = pf.SamplerConfig(patch_size=32, epoch_size=300, seed=5, target_mpps=[(0.25, 1.0)], max_attempts_per_slide=3)
    got = list(pf.epoch_stream(cfg, slides, batch=batch))
    orc = [{"id": r.slide_id, "width": r.width, "height": r.height, "base_mpp": 0.25, "rings": p.rings} for r, p in slides]
    want, _ = port.epoch_stream(orc, patch_size=32, min_fg=0.4, mpps=[(0.25, 1.0)], seed=5, epoch_size=300,
                                max_attempts=3)
    assert [(s.slide_id, s.x, s.y, s.width, s.target_mpp, s.seq) for s in got] == \
        [(orc[si]["id"], x, y, fp, m, q) for si, x, y, fp, m, q in want]


def test_specs_carry_read_plan(pf, goldens):
    c = goldens["epoch_streams"]["multi_mpp"]
    slides = _slides(pf, goldens, c["slides"])
    smp = pf.GpuSampler(_cfg(pf, c), slides)
    arr = smp.next_batch(60).cpu().numpy().view(pf._native.SPEC_DTYPE).reshape(-1)
    for r in arr:
        rec = slides[r["slide"]][0]
        li = pf.select_level(rec, float(r["target_mpp"]))
        lv = rec.levels[li]
        assert r["level"] == li
        assert r["side"] == max(1, pf.round_half_away(r["out_size"] * r["target_mpp"] / lv.mpp))
        assert r["sx"] == pf.round_half_away(r["x"] / lv.downsample)
        assert r["sy"] == pf.round_half_away(r["y"] / lv.downsample)


def test_no_samplable_slide(pf, goldens):
    # polygon far from any admissible footprint: min_fg 1.0 with a tiny polygon
    tiny = pf.rect_polygon(10, 10, 5, 5)
    rec = pf.store.make_record("t", 200, 200, 0.25, tile_size=64)
    cfg = pf.SamplerConfig(patch_size=64, epoch_size=3, min_foreground=1.0, max_attempts_per_slide=3)
    with pytest.raises(pf.NoSamplableSlideError):
        list(pf.epoch_stream(cfg, [(rec, tiny)]))


def test_determinism_and_seed_sensitivity(pf, goldens):
    c = goldens["epoch_streams"]["single"]
    sl = _slides(pf, goldens, [0])
    a = list(pf.epoch_stream(pf.SamplerConfig(patch_size=32, epoch_size=50, seed=1), sl))
    b = list(pf.epoch_stream(pf.SamplerConfig(patch_size=32, epoch_size=50, seed=1), sl))
    d = list(pf.epoch_stream(pf.SamplerConfig(patch_size=32, epoch_size=50, seed=2), sl))
    assert a == b and a != d
    assert c["cfg"]["seed"] == 0


@pytest.mark.parametrize("key", ["7/40/13", "25/60/13", "1/9/2"])
def test_capped_replay_on_device_matches_reference(pf, goldens, key):
    """CappedSampler (pf_capped_draw) over the device sampler reproduces the reference's
    capped_stream seq sequence across batch boundaries."""
    cap, total, seed = (int(v) for v in key.split("/"))
    c = goldens["epoch_streams"]["multi_mpp"]
    smp = pf.GpuSampler(_cfg(pf, c), _slides(pf, goldens, c["slides"]))
    cs = pf.CappedSampler(smp, cap, seed)
    got = []
    for n in (3, 5, 11, 64):
        if len(got) >= total:
            break
        got += [s.seq for s in smp.to_patch_specs(cs.next_batch(min(n, total - len(got))))]
    assert got == goldens["capped_streams"][key]
