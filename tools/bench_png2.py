"""Split GPU PNG decode time into inflate and unfilter."""
import sys; sys.path.insert(0, '.')
import tempfile, pathlib
import numpy as np, torch
from paper_2404_15217_b200 import store, _native as N
from paper_2404_15217_b200.synthetic import synthetic_slide
s = synthetic_slide("p", 4096, 4096, seed=3, downsample_factor=4)
img = s.level_array(0).cpu().numpy()
with tempfile.TemporaryDirectory() as td:
    rec = store.ingest_image(img, "p", 0.25, td, tile_size=256, downsample_factor=4, codec="png")
    part = []
    for ty in range(16):
        for tx in range(16):
            part.append((tx, ty, 256, 256, store._png_zlib_stream(store._read_chunk_bytes(pathlib.Path(td), rec.chunks[(0, tx, ty)]), 256, 256)))
n = len(part)
zl = np.array([len(t[4]) for t in part]); zoff = np.zeros(n + 1, np.int64); zoff[1:] = np.cumsum(zl)
rlen = np.full(n, 256 * 769, np.int64); roff = np.zeros(n, np.int64); roff[1:] = np.cumsum(rlen)[:-1]
print("compressed bytes/tile", zl.mean(), "raw", 256 * 769)
z = torch.from_numpy(np.frombuffer(b"".join(t[4] for t in part), np.uint8).copy()).cuda()
raw = torch.empty(int(rlen.sum()), dtype=torch.uint8, device="cuda"); st = torch.zeros(n, dtype=torch.int32, device="cuda")
lvl = torch.zeros((16, 16, 256, 256, 3), dtype=torch.uint8, device="cuda")
dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
zo, ro, rl = dv(zoff), dv(roff), dv(rlen)
dst = dv(np.array([lvl.data_ptr() + (t[1] * 16 + t[0]) * 196608 for t in part], np.int64))
tw = dv(np.full(n, 256, np.int32)); th = dv(np.full(n, 256, np.int32))
L = N.lib()
for rep in range(2):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); L.pf_png_inflate(z.data_ptr(), zo.data_ptr(), n, raw.data_ptr(), ro.data_ptr(), rl.data_ptr(), st.data_ptr(), None)
    e[1].record(); L.pf_png_unfilter(raw.data_ptr(), ro.data_ptr(), tw.data_ptr(), th.data_ptr(), dst.data_ptr(), 256, n, st.data_ptr(), None)
    e[2].record(); torch.cuda.synchronize()
    print(f"{n} tiles: inflate {e[0].elapsed_time(e[1]):.1f} ms, unfilter {e[1].elapsed_time(e[2]):.1f} ms, status ok {int((st == 0).sum())}")
assert torch.equal(lvl.permute(0, 2, 1, 3, 4).reshape(4096, 4096, 3), s.level_array(0))
