"""GPU baseline JPEG decode throughput vs Pillow on all host cores (same q90 tiles)."""
import sys; sys.path.insert(0, '.')
import io, os, time
import numpy as np, torch
from concurrent.futures import ProcessPoolExecutor
from PIL import Image
from paper_2404_15217_b200 import store
from paper_2404_15217_b200.synthetic import synthetic_slide

def enc(a):
    b = io.BytesIO(); Image.fromarray(a).save(b, format="JPEG", quality=90); return b.getvalue()

def dec(blobs):
    return [np.asarray(Image.open(io.BytesIO(b)).convert("RGB")).sum() for b in blobs]

if __name__ == "__main__":
    s = synthetic_slide("p", 16384, 16384, seed=3, downsample_factor=4)
    lv = s.levels[0].cpu().numpy()
    ny, nx = lv.shape[:2]
    cores = len(os.sched_getaffinity(0))
    with ProcessPoolExecutor(cores) as ex:
        blobs = list(ex.map(enc, [lv[ty, tx] for ty in range(ny) for tx in range(nx)], chunksize=64))
    part = [(i % nx, i // nx, 256, 256, b) for i, b in enumerate(blobs)]
    out = torch.zeros_like(s.levels[0])
    store._decode_jpeg_tiles(out, 256, part[:64]); torch.cuda.synchronize()
    t = time.time(); store._decode_jpeg_tiles(out, 256, part); torch.cuda.synchronize(); g = time.time() - t
    import paper_2404_15217_b200._native as N
    real = N.lib()
    orig = real.pf_jpeg_decode
    times = []
    class Wrap:
        def __getattr__(self, k): return getattr(real, k)
        def pf_jpeg_decode(self, *a):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); r = orig(*a); e1.record(); torch.cuda.synchronize(); times.append(e0.elapsed_time(e1)); return r
    lib_fn = N.lib
    N.lib = lambda: Wrap()
    t = time.time(); store._decode_jpeg_tiles(out, 256, part); torch.cuda.synchronize(); g2 = time.time() - t
    N.lib = lib_fn
    print(f"kernels {times[-1]:.1f} ms of {g2 * 1e3:.0f} ms")
    want = np.stack([np.asarray(Image.open(io.BytesIO(b)).convert("RGB")) for b in blobs[:64]])
    assert np.array_equal(out.view(-1, 256, 256, 3)[:64].cpu().numpy(), want)
    chunks = [blobs[i:i + 64] for i in range(0, len(blobs), 64)]
    with ProcessPoolExecutor(cores) as ex:
        list(ex.map(dec, chunks[:cores]))
        t = time.time(); list(ex.map(dec, chunks)); c = time.time() - t
    n = len(blobs)
    print(f"{n} JPEG q90 tiles ({sum(map(len, blobs)) / n / 1e3:.0f} kB each): "
          f"GPU decode {g * 1e3:.0f} ms incl. H2D of tables/streams ({n / g:.0f} tiles/s); "
          f"Pillow on {cores} cores {c * 1e3:.0f} ms ({n / c:.0f} tiles/s)")
