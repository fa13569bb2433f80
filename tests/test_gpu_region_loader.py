"""GPU: the config-1 loader (sampler -> read_region -> normalise) serves the same batches
whatever its sampler prefetch chunking, and each batch equals read_region of its specs."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup(cuda):
    import paper_2404_15217_b200 as pf
    from paper_2404_15217_b200.synthetic import synthetic_slide

    s = synthetic_slide("rl", 6000, 4500, seed=2, blob_px=800)
    thumb, scale = s.thumbnail(32)
    poly = pf.polygon_from_mask(pf.mask_from_saturation(thumb, 0.07, 1, scale=scale), slide_id="rl")
    return pf, [(s, poly)]


@pytest.mark.parametrize("chunk", [1, 3, 4])
def test_region_loader_chunked_prefetch_is_the_plain_stream(setup, chunk):
    torch = pytest.importorskip("torch")
    pf, slides = setup
    cfg = pf.SamplerConfig(patch_size=224, seed=4, target_mpps=[(0.25, 1.0), (0.5, 1.0)])
    ref = pf.pipeline.RegionLoader(slides, cfg, batch_size=32, prefetch=False)
    got = pf.pipeline.RegionLoader(slides, cfg, batch_size=32, chunk=chunk)
    for _ in range(7):  # crosses several chunk boundaries
        a, b = ref.next_batch(), got.next_batch()
        assert torch.equal(a["specs"], b["specs"])
        assert torch.equal(a["patches"], b["patches"])
    torch.cuda.synchronize()
    hs = got.sampler.to_patch_specs(b["specs"])
    assert [s.seq for s in hs] == list(range(6 * 32, 7 * 32))
    want = got.slide_set.read_regions(b["specs"], 224, dtype="f32", layout="nchw", mean=got.mean, std=got.std)
    assert torch.equal(want, b["patches"])
