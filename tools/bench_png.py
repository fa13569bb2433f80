"""Time GpuSlide.from_store on a PNG store: GPU inflate+unfilter vs host Pillow decode."""
import sys; sys.path.insert(0, '.')
import tempfile, time
import numpy as np, torch
import paper_2404_15217_b200 as pf
from paper_2404_15217_b200.synthetic import synthetic_slide
from paper_2404_15217_b200 import store

s = synthetic_slide("p", 8192, 8192, seed=3, downsample_factor=4)
img = s.level_array(0).cpu().numpy()
with tempfile.TemporaryDirectory() as td:
    t = time.time(); store.ingest_image(img, "p", 0.25, td, tile_size=256, downsample_factor=4, codec="png"); enc = time.time() - t
    res = {}
    for gpu in (True, False, True):
        torch.cuda.synchronize(); t = time.time()
        g = pf.GpuSlide.from_store(td, "p", gpu_png=gpu); torch.cuda.synchronize()
        res[gpu] = time.time() - t
    assert torch.equal(g.level_array(0), s.level_array(0))
    # decode-only timing of the level-0 tiles (host file reads / PNG parse excluded)
    rec = g.record
    tiles = []
    for ty in range(rec.tile_grid(0)[1]):
        for tx in range(rec.tile_grid(0)[0]):
            tw, th = rec.tile_dims(0, tx, ty)
            tiles.append((tx, ty, tw, th, store._png_zlib_stream(store._read_chunk_bytes(__import__('pathlib').Path(td), rec.chunks[(0, tx, ty)]), tw, th)))
    lvl = torch.zeros_like(g.levels[0])
    store._decode_png_tiles(lvl, 256, tiles); torch.cuda.synchronize()
    t = time.time(); store._decode_png_tiles(lvl, 256, tiles); torch.cuda.synchronize(); dec = time.time() - t
    assert torch.equal(lvl, g.levels[0])
print(f"ingest png {enc:.1f}s; from_store gpu {res[True]:.2f}s, host pillow {res[False]:.2f}s; "
      f"GPU decode of {len(tiles)} level-0 tiles {dec * 1e3:.1f} ms ({len(tiles) / dec:.0f} tiles/s, "
      f"{len(tiles) * 256 * 256 * 3 / dec / 1e9:.2f} GB/s)")
