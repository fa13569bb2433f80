"""GPU PNG decode throughput at scale vs Pillow on all host cores (same tiles)."""
import sys; sys.path.insert(0, '.')
import io, os, time
import numpy as np, torch
from concurrent.futures import ProcessPoolExecutor
from PIL import Image
from paper_2404_15217_b200 import store
from paper_2404_15217_b200.synthetic import synthetic_slide

def enc(a):
    b = io.BytesIO(); Image.fromarray(a).save(b, format="PNG"); return b.getvalue()

def dec(blobs):
    return [np.asarray(Image.open(io.BytesIO(b)).convert("RGB")).sum() for b in blobs]

if __name__ == "__main__":
    s = synthetic_slide("p", 16384, 16384, seed=3, downsample_factor=4)
    lv = s.levels[0].cpu().numpy()  # [64, 64, 256, 256, 3]
    ny, nx = lv.shape[:2]
    cores = len(os.sched_getaffinity(0))
    with ProcessPoolExecutor(cores) as ex:
        blobs = list(ex.map(enc, [lv[ty, tx] for ty in range(ny) for tx in range(nx)], chunksize=64))
    part = [(i % nx, i // nx, 256, 256, store._png_zlib_stream(b, 256, 256)) for i, b in enumerate(blobs)]
    out = torch.zeros_like(s.levels[0])
    store._decode_png_tiles(out, 256, part[:256]); torch.cuda.synchronize()
    t = time.time(); store._decode_png_tiles(out, 256, part); torch.cuda.synchronize(); g = time.time() - t
    assert torch.equal(out, s.levels[0])
    # kernels alone (inputs already on the device)
    from paper_2404_15217_b200 import _native as N
    n = len(part)
    zl = np.array([len(p[4]) for p in part]); zoff = np.zeros(n + 1, np.int64); zoff[1:] = np.cumsum(zl)
    rlen = np.full(n, 256 * 769, np.int64); roff = np.zeros(n, np.int64); roff[1:] = np.cumsum(rlen)[:-1]
    dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    z = dv(np.frombuffer(b"".join(p[4] for p in part), np.uint8)); zo, ro, rl = dv(zoff), dv(roff), dv(rlen)
    raw = torch.empty(int(rlen.sum()), dtype=torch.uint8, device="cuda"); st = torch.zeros(n, dtype=torch.int32, device="cuda")
    dst = dv(np.array([out.data_ptr() + (p[1] * nx + p[0]) * 196608 for p in part], np.int64))
    tw = dv(np.full(n, 256, np.int32))
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); N.lib().pf_png_inflate(z.data_ptr(), zo.data_ptr(), n, raw.data_ptr(), ro.data_ptr(), rl.data_ptr(), st.data_ptr(), None)
    e[1].record(); N.lib().pf_png_unfilter(raw.data_ptr(), ro.data_ptr(), tw.data_ptr(), tw.data_ptr(), dst.data_ptr(), 256, n, st.data_ptr(), None)
    e[2].record(); torch.cuda.synchronize()
    ki, ku = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
    chunks = [blobs[i:i + 64] for i in range(0, len(blobs), 64)]
    with ProcessPoolExecutor(cores) as ex:
        list(ex.map(dec, chunks[:cores]))
        t = time.time(); list(ex.map(dec, chunks)); c = time.time() - t
    n = len(blobs)
    print(f"{n} PNG tiles (256^2 RGB, {sum(map(len, blobs)) / n / 1e3:.0f} kB each): GPU {g * 1e3:.0f} ms "
          f"({n / g:.0f} tiles/s, {n * 196608 / g / 1e9:.2f} GB/s decoded) incl. H2D; Pillow on {cores} cores "
          f"{c * 1e3:.0f} ms ({n / c:.0f} tiles/s); kernels only: inflate {ki:.1f} ms + unfilter {ku:.1f} ms "
          f"({n / (ki + ku) * 1e3:.0f} tiles/s)")
