"""HBM-resident slide pyramids and the batched region reader.

Mirrors the read side of pkg/store.py: ``SlideRecord``/``LevelInfo``
(115-237), ``select_level`` (568-581), ``round_half_away`` (70-72),
``Slide.thumbnail`` (604-609) and ``Slide.read_region`` (651-688).  Instead of
a host tile cache fed by a transport, every level lives in HBM in the padded
tile-major layout of include/pf_b200.h, built on the GPU by the reference's
box filter (``_box_downsample``, 429-441) with the ingest stopping rule
(496-498).  ``GpuSlide`` duck-types the reference ``Slide`` (``.record`` +
``.read_region``) so it plugs into ``run_loader``; ``read_regions`` is the
batched device path.
"""

from __future__ import annotations

import json
import math
import weakref
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _native as N
from .errors import DecodeError, IntegrityError, OutOfBoundsError, SlideNotFoundError, StoreError

STORE_FORMAT_VERSION = 1


def round_half_away(x: float) -> int:
    """Round half away from zero (pkg/store.py:70-72)."""
    return int(math.floor(x + 0.5)) if x >= 0 else int(math.ceil(x - 0.5))


@dataclass(frozen=True)
class LevelInfo:
    width: int
    height: int
    mpp: float
    downsample: int


@dataclass
class SlideRecord:
    """Pyramid metadata (pkg/store.py:122-237); ``chunks`` only for store-backed slides."""

    slide_id: str
    base_mpp: float
    tile_size: int
    levels: list
    chunks: dict = field(default_factory=dict)

    @property
    def width(self) -> int:
        return self.levels[0].width

    @property
    def height(self) -> int:
        return self.levels[0].height

    def tile_grid(self, level: int) -> tuple:
        lv = self.levels[level]
        t = self.tile_size
        return -(-lv.width // t), -(-lv.height // t)

    def tile_dims(self, level: int, tx: int, ty: int) -> tuple:
        lv = self.levels[level]
        t = self.tile_size
        return min(t, lv.width - tx * t), min(t, lv.height - ty * t)

    def validate(self) -> None:
        """Level invariants of SlideRecord.validate (pkg/store.py:151-176)."""
        if self.tile_size < 16:
            raise IntegrityError(f"tile_size {self.tile_size} < 16")
        if not self.levels:
            raise IntegrityError("record has no levels")
        l0 = self.levels[0]
        if l0.downsample != 1:
            raise IntegrityError("level 0 must have downsample 1")
        if not math.isclose(l0.mpp, self.base_mpp, rel_tol=1e-9):
            raise IntegrityError("level 0 mpp must equal base_mpp")
        prev = 0.0
        for i, lv in enumerate(self.levels):
            if lv.mpp <= prev:
                raise IntegrityError(f"levels not sorted by increasing mpp at {i}")
            prev = lv.mpp
            if not math.isclose(lv.mpp, self.base_mpp * lv.downsample, rel_tol=1e-9):
                raise IntegrityError(f"level {i} mpp {lv.mpp} != base_mpp * downsample")
            ew, eh = -(-l0.width // lv.downsample), -(-l0.height // lv.downsample)
            if abs(lv.width - ew) > 1 or abs(lv.height - eh) > 1:
                raise IntegrityError(
                    f"level {i} dims ({lv.width}x{lv.height}) do not match level 0 / downsample ({ew}x{eh})"
                )

    def to_json_dict(self) -> dict:
        return {
            "slide_id": self.slide_id,
            "base_mpp": self.base_mpp,
            "tile_size": self.tile_size,
            "levels": [
                {"width_px": lv.width, "height_px": lv.height, "mpp": lv.mpp, "downsample": lv.downsample}
                for lv in self.levels
            ],
            "chunks": {f"{k[0]}/{k[1]}_{k[2]}": v for k, v in sorted(self.chunks.items())},
        }

    @classmethod
    def from_json_dict(cls, doc: dict) -> "SlideRecord":
        try:
            levels = [
                LevelInfo(int(d["width_px"]), int(d["height_px"]), float(d["mpp"]), int(d["downsample"]))
                for d in doc["levels"]
            ]
            chunks = {}
            for key, loc in doc.get("chunks", {}).items():
                li, rest = key.split("/")
                tx, ty = rest.split("_")
                chunks[(int(li), int(tx), int(ty))] = dict(loc)
            return cls(str(doc["slide_id"]), float(doc["base_mpp"]), int(doc["tile_size"]), levels, chunks)
        except (KeyError, ValueError) as exc:
            raise IntegrityError(f"malformed slide record: {exc}") from exc


def select_level(record: SlideRecord, target_mpp: float) -> int:
    """argmin |ln(mpp_i / target)|, ties (within 1e-12) to the finer level (pkg/store.py:568-581)."""
    if target_mpp <= 0:
        raise ValueError("target_mpp must be positive")
    best, best_d = 0, math.inf
    for i, lv in enumerate(record.levels):
        d = abs(math.log(lv.mpp / target_mpp))
        if d < best_d - 1e-12:
            best, best_d = i, d
    return best


def pyramid_dims(width: int, height: int, tile_size: int, factor: int) -> list:
    """Level dims of ingest_image: repeat ceil-divide by `factor` until max(dim) <= tile (store.py:496-498)."""
    dims = [(width, height)]
    while max(dims[-1]) > tile_size:
        w, h = dims[-1]
        dims.append((-(-w // factor), -(-h // factor)))
    return dims


def make_record(slide_id: str, width: int, height: int, base_mpp: float, tile_size: int = 256,
                downsample_factor: int = 2) -> SlideRecord:
    dims = pyramid_dims(width, height, tile_size, downsample_factor)
    levels = [
        LevelInfo(w, h, base_mpp * downsample_factor**i, downsample_factor**i) for i, (w, h) in enumerate(dims)
    ]
    rec = SlideRecord(slide_id, base_mpp, tile_size, levels)
    rec.validate()
    return rec


def _tiles_from_hwc(arr: np.ndarray, tile: int) -> np.ndarray:
    """(H, W, 3) -> padded tile-major (ty, tx, T, T, 3)."""
    h, w = arr.shape[:2]
    ny, nx = -(-h // tile), -(-w // tile)
    pad = np.zeros((ny * tile, nx * tile, 3), dtype=np.uint8)
    pad[:h, :w] = arr
    return np.ascontiguousarray(pad.reshape(ny, tile, nx, tile, 3).transpose(0, 2, 1, 3, 4))


class GpuSlide:
    """A slide pyramid resident in HBM (drop-in for the reference ``Slide``)."""

    def __init__(self, record: SlideRecord, levels, factor: int):
        self.record = record
        self.levels = levels  # torch uint8 [ty, tx, T, T, 3] per level (dense) or [slots, T, T, 3]
        self.tile_maps = [None] * len(levels)  # int32 [ty * tx] slot map for compacted levels
        self.resident = [None] * len(levels)  # host bool [ty, tx] of compacted levels
        self.factor = factor
        # fault word of the descriptor (pf_slide_desc.status_word): a read of a non-resident tile
        # of a compacted level sets it; check_status() raises OutOfBoundsError
        self.status = None
        if levels:
            import torch

            self.status = torch.zeros(1, dtype=torch.int32, device=levels[0].device)
        self.desc = self._make_desc()
        self._sets = weakref.WeakSet()  # SlideSets holding a device copy of self.desc

    def compact(self, plan, levels=None) -> None:
        """Keep only the planned tiles resident (residency.reachable_tiles): each level becomes
        [1 + n_resident] tile slots (slot 0 = zero hole) plus an int32 slot map; the dense level is
        freed.  Reads of non-resident tiles return zeros (pf_slide_desc.tile_map)."""
        torch = N.require_cuda()
        T = self.record.tile_size
        # in-flight reads (any stream) of the dense levels finish before they are freed
        torch.cuda.synchronize()
        for li, keep in enumerate(plan):
            if levels is not None and li not in levels:
                continue
            if self.tile_maps[li] is not None:
                raise ValueError(f"level {li} is already compacted")
            nx, ny = self.record.tile_grid(li)
            keep = np.asarray(keep, dtype=bool)
            if keep.shape != (ny, nx):
                raise ValueError(f"plan for level {li} must be ({ny}, {nx})")
            idx = np.flatnonzero(keep.ravel())
            slots = torch.empty((len(idx) + 1, T, T, 3), dtype=torch.uint8, device="cuda")
            slots[0].zero_()
            src = self.levels[li].view(ny * nx, T, T, 3)
            for i in range(0, len(idx), 4096):  # bounded temporaries (<= 0.8 GB at T = 256)
                sel = torch.from_numpy(idx[i:i + 4096]).cuda()
                slots[1 + i:1 + i + len(sel)] = src[sel]
            del src
            m = np.zeros(ny * nx, dtype=np.int32)
            m[idx] = np.arange(1, len(idx) + 1, dtype=np.int32)
            self.levels[li] = slots
            self.tile_maps[li] = torch.from_numpy(m).cuda()
            self.resident[li] = keep
        self.desc = self._make_desc()
        self._own_set = None
        # every SlideSet built earlier (and the samplers / loaders sharing its descriptor tensor)
        # sees the new level pointers and slot maps: no read can reach the freed dense levels
        for ss in list(self._sets):
            ss._refresh(self)

    @property
    def compacted(self) -> bool:
        return any(m is not None for m in self.tile_maps)

    # -- construction -----------------------------------------------------
    @classmethod
    def allocate(cls, slide_id: str, width: int, height: int, base_mpp: float, tile_size: int = 256,
                 downsample_factor: int = 2, device=None) -> "GpuSlide":
        torch = N.require_cuda()
        rec = make_record(slide_id, width, height, base_mpp, tile_size, downsample_factor)
        levels = []
        for li in range(len(rec.levels)):
            nx, ny = rec.tile_grid(li)
            levels.append(torch.empty((ny, nx, tile_size, tile_size, 3), dtype=torch.uint8, device=device or "cuda"))
        return cls(rec, levels, downsample_factor)

    @classmethod
    def from_array(cls, pixels, slide_id: str, base_mpp: float, *, tile_size: int = 256,
                   downsample_factor: int = 2, stream=None) -> "GpuSlide":
        """ingest_image (pkg/store.py:462-565) into HBM: level 0 uploaded, upper levels box-filtered on device."""
        torch = N.require_cuda()
        arr = pixels.cpu().numpy() if hasattr(pixels, "cpu") else np.asarray(pixels)
        if arr.ndim != 3 or arr.shape[2] != 3 or arr.dtype != np.uint8:
            raise ValueError("pixels must be an (H, W, 3) uint8 array")
        if arr.shape[0] < 1 or arr.shape[1] < 1:
            raise ValueError("image must be at least 1x1")
        if tile_size < 16:
            raise ValueError("tile_size must be >= 16")
        if downsample_factor < 2:
            raise ValueError("downsample_factor must be >= 2")
        slide = cls.allocate(slide_id, arr.shape[1], arr.shape[0], base_mpp, tile_size, downsample_factor)
        slide.levels[0].copy_(torch.from_numpy(_tiles_from_hwc(arr, tile_size)))
        slide.build_pyramid(stream)
        return slide

    @classmethod
    def from_store(cls, store_root, slide_id: str, stream=None, gpu_png: bool = True) -> "GpuSlide":
        """Load a reference store slide (index.json + slides/<id>.json + chunks) into HBM.

        Every level is read as stored (raw/png/jpeg via the store's locators) so the
        HBM pyramid holds the exact bytes the reference serves.  PNG tiles (the store's
        default codec) are inflated and unfiltered on the GPU (pf_png_inflate /
        pf_png_unfilter) after a host check of the chunk CRCs; other codecs and PNG
        variants Pillow writes only for non-RGB images decode on the host.
        """
        torch = N.require_cuda()
        root = Path(store_root)
        idx_path = root / "index.json"
        if not idx_path.exists():
            raise StoreError(f"no store at {store_root} (missing index.json)")
        index = json.loads(idx_path.read_text(encoding="utf-8"))
        if int(index.get("format_version", -1)) != STORE_FORMAT_VERSION:
            raise IntegrityError(f"unsupported store format_version {index.get('format_version')}")
        if slide_id not in index.get("slides", []):
            raise SlideNotFoundError(f"slide {slide_id!r} not in store {root}")
        rel = index.get("records", {}).get(slide_id, f"slides/{slide_id}.json")
        rec = SlideRecord.from_json_dict(json.loads((root / rel).read_text(encoding="utf-8")))
        if rec.slide_id != slide_id:
            raise IntegrityError(f"record names slide {rec.slide_id!r}, expected {slide_id!r}")
        rec.validate()
        factor = rec.levels[1].downsample if len(rec.levels) > 1 else 2
        T = rec.tile_size
        levels = []
        for li, lv in enumerate(rec.levels):
            nx, ny = rec.tile_grid(li)
            host = np.zeros((ny, nx, T, T, 3), dtype=np.uint8)
            png, jpg = [], []  # (tx, ty, tw, th, zlib stream | JPEG file) decoded on the GPU
            for ty in range(ny):
                for tx in range(nx):
                    loc = rec.chunks.get((li, tx, ty))
                    if loc is None:
                        raise IntegrityError(f"missing chunk locator ({li}, {tx}, {ty})")
                    tw, th = rec.tile_dims(li, tx, ty)
                    if gpu_png and loc["codec"] == "png" and tw <= 256:
                        z = _png_zlib_stream(_read_chunk_bytes(root, loc), tw, th)
                        if z is not None:
                            png.append((tx, ty, tw, th, z))
                            continue
                    if gpu_png and loc["codec"] == "jpeg":
                        jpg.append((tx, ty, tw, th, _read_chunk_bytes(root, loc)))
                        continue
                    host[ty, tx, :th, :tw] = _read_chunk(root, loc, tw, th)
            dev = torch.from_numpy(host).cuda()
            if png:
                _decode_png_tiles(dev, T, png, stream)
            if jpg:
                for k in _decode_jpeg_tiles(dev, T, jpg, stream):  # variants the GPU path does not take
                    tx, ty, tw, th, _ = jpg[k]
                    host_tile = _read_chunk(root, rec.chunks[(li, tx, ty)], tw, th)
                    dev[ty, tx, :th, :tw] = torch.from_numpy(np.ascontiguousarray(host_tile)).cuda()
            levels.append(dev)
        return cls(rec, levels, factor)

    def build_pyramid(self, stream=None) -> None:
        """Levels 1.. from level 0 with the reference box filter, on device."""
        for li in range(1, len(self.record.levels)):
            N.check(N.lib().pf_build_level(self.desc, li, self.factor, N.stream_ptr(stream)), "pf_build_level")

    def _make_desc(self) -> N.SlideDesc:
        d = N.SlideDesc()
        rec = self.record
        if len(rec.levels) > N.PF_MAX_LEVELS:
            raise ValueError(f"more than {N.PF_MAX_LEVELS} pyramid levels")
        for i, lv in enumerate(rec.levels):
            nx, ny = rec.tile_grid(i)
            d.level_ptr[i] = int(self.levels[i].data_ptr()) if self.levels else 0
            tm = self.tile_maps[i] if self.levels else None
            d.tile_map[i] = int(tm.data_ptr()) if tm is not None else 0
            d.mpp[i] = lv.mpp
            d.width[i] = lv.width
            d.height[i] = lv.height
            d.tiles_x[i] = nx
            d.tiles_y[i] = ny
            d.downsample[i] = lv.downsample
        d.n_levels = len(rec.levels)
        d.tile_size = rec.tile_size
        d.base_mpp = rec.base_mpp
        d.status_word = int(self.status.data_ptr()) if getattr(self, "status", None) is not None else 0
        return d

    def require_resident(self, spec) -> None:
        """Host check of a planned spec (plan_specs row) against a compacted level: the window
        must lie on resident tiles, else OutOfBoundsError (the device path would read the hole)."""
        li = int(spec["level"])
        if self.resident[li] is None:
            return
        lv, T = self.record.levels[li], self.record.tile_size
        x0, y0, side = int(spec["sx"]), int(spec["sy"]), int(spec["side"])
        tx0, ty0 = max(x0, 0) // T, max(y0, 0) // T
        tx1, ty1 = min(x0 + side - 1, lv.width - 1) // T, min(y0 + side - 1, lv.height - 1) // T
        if not self.resident[li][ty0:ty1 + 1, tx0:tx1 + 1].all():
            raise OutOfBoundsError(f"region {(int(spec['x']), int(spec['y']), int(spec['width']), int(spec['height']))} "
                                   "reads tiles that are not HBM-resident (slide compacted to the sampler's "
                                   "reachable tiles)")

    def check_status(self, stream=None, clear: bool = True) -> None:
        """Raise OutOfBoundsError if a device read since the last check reached a non-resident tile
        (pf_slide_status; synchronises the stream)."""
        rc = N.lib().pf_slide_status(self.desc, 1 if clear else 0, N.stream_ptr(stream))
        if rc != N.PF_OK:
            N.check(rc, f"slide {self.record.slide_id!r}")

    # -- reads ------------------------------------------------------------
    def select_level(self, target_mpp: float) -> int:
        return select_level(self.record, target_mpp)

    def level_array(self, li: int):
        """Level li as a dense (H, W, 3) uint8 device tensor (copy)."""
        if self.tile_maps[li] is not None:
            raise ValueError("level is compacted to its resident tiles; no dense view")
        lv = self.record.levels[li]
        t = self.levels[li]
        ny, nx, T = t.shape[0], t.shape[1], t.shape[2]
        return t.permute(0, 2, 1, 3, 4).reshape(ny * T, nx * T, 3)[: lv.height, : lv.width].contiguous()

    def thumbnail_device(self, factor: int | None = None, src_level: int = 0, stream=None):
        """(device (h, w, 3) uint8, scale).  factor None -> coarsest level (Slide.thumbnail)."""
        torch = N.require_cuda()
        if factor is None:
            src_level, factor = len(self.record.levels) - 1, 1
        lv = self.record.levels[src_level]
        out = torch.empty((-(-lv.height // factor), -(-lv.width // factor), 3), dtype=torch.uint8, device="cuda")
        N.check(N.lib().pf_thumbnail(self.desc, src_level, factor, out.data_ptr(), N.stream_ptr(stream)), "pf_thumbnail")
        return out, 1.0 / (lv.downsample * factor)

    def thumbnail(self, factor: int | None = None) -> tuple:
        """Drop-in Slide.thumbnail (pkg/store.py:604-609): (host ndarray, scale)."""
        t, scale = self.thumbnail_device(factor)
        return t.cpu().numpy(), scale

    def read_region(self, rect_level0, target_mpp: float, out_size: int) -> np.ndarray:
        """Drop-in Slide.read_region (pkg/store.py:651-688): (out, out, 3) uint8 host array."""
        specs = plan_specs([(0, rect_level0, target_mpp, out_size)], [self.record])
        self.require_resident(specs[0])
        if getattr(self, "_own_set", None) is None:
            self._own_set = SlideSet([self])
        if getattr(self, "tier", None) is not None:  # host-backed level: bring the window's tiles in
            from .tier import TierSet

            if getattr(self, "_own_tiers", None) is None:
                self._own_tiers = TierSet(self._own_set)
            import torch

            self._own_tiers.prefetch(torch.from_numpy(specs.view(np.uint8).reshape(1, 64)).cuda(), 1)
        out = self._own_set.read_regions(specs, out_size)
        if self.compacted:
            self.check_status()
        return out[0].cpu().numpy()


def _read_chunk_bytes(root: Path, loc: dict) -> bytes:
    path = loc["path"]
    p = Path(path) if Path(path).is_absolute() else root / path
    try:
        if loc["kind"] == "byte-range":
            with open(p, "rb") as fh:
                fh.seek(int(loc["offset"]))
                return fh.read(int(loc["length"]))
        return p.read_bytes()
    except OSError as exc:
        raise StoreError(f"cannot read {p}: {exc}") from exc


_PNG_SIG = b"\x89PNG\r\n\x1a\n"


def _png_zlib_stream(data: bytes, tw: int, th: int):
    """The zlib stream (concatenated IDAT payloads) of an 8-bit RGB non-interlaced tw x th PNG,
    every chunk CRC checked; None for any other PNG variant (decoded on the host)."""
    import struct
    import zlib

    if data[:8] != _PNG_SIG:
        raise DecodeError("not a PNG tile")
    pos, idat, ok = 8, [], False
    while pos + 12 <= len(data):
        n = int.from_bytes(data[pos:pos + 4], "big")
        typ, body = data[pos + 4:pos + 8], data[pos + 8:pos + 8 + n]
        if len(body) != n or pos + 12 + n > len(data):
            raise DecodeError("truncated PNG chunk")
        if zlib.crc32(typ + body) != int.from_bytes(data[pos + 8 + n:pos + 12 + n], "big"):
            raise DecodeError(f"PNG chunk {typ!r} fails its CRC")
        if typ == b"IHDR":
            ok = struct.unpack(">IIBBBBB", body) == (tw, th, 8, 2, 0, 0, 0)
        elif typ == b"IDAT":
            idat.append(body)
        elif typ == b"IEND":
            break
        pos += 12 + n
    return b"".join(idat) if ok and idat else None


def _decode_png_tiles(level, T: int, tiles, stream=None, chunk: int = 4096) -> None:
    """Inflate + unfilter PNG tiles on the GPU into a dense level [ty, tx, T, T, 3] (tiles up to 256
    px wide; wider tiles decode on the host)."""
    torch = N.require_cuda()
    L = N.lib()
    nx = level.shape[1]
    tb = T * T * 3
    for i in range(0, len(tiles), chunk):
        part = tiles[i:i + chunk]
        n = len(part)
        zl = np.array([len(t[4]) for t in part], dtype=np.int64)
        zoff = np.zeros(n + 1, dtype=np.int64)
        zoff[1:] = np.cumsum(zl)
        rlen = np.array([t[3] * (1 + 3 * t[2]) for t in part], dtype=np.int64)
        roff = np.zeros(n, dtype=np.int64)
        roff[1:] = np.cumsum(rlen)[:-1]
        pinned = torch.empty(int(zoff[-1]), dtype=torch.uint8, pin_memory=True)  # one H2D for all streams
        host = pinned.numpy()
        for k, t in enumerate(part):
            host[zoff[k]:zoff[k + 1]] = np.frombuffer(t[4], dtype=np.uint8)
        zdev = pinned.to("cuda", non_blocking=True)
        raw = torch.empty(int(rlen.sum()), dtype=torch.uint8, device="cuda")
        status = torch.zeros(n, dtype=torch.int32, device="cuda")
        base = int(level.data_ptr())
        dst = np.array([base + (t[1] * nx + t[0]) * tb for t in part], dtype=np.uint64)
        dv = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
        zoff_d, roff_d, rlen_d, dst_d = dv(zoff), dv(roff), dv(rlen), dv(dst.view(np.int64))
        tw_d = dv(np.array([t[2] for t in part], dtype=np.int32))
        th_d = dv(np.array([t[3] for t in part], dtype=np.int32))
        sp = N.stream_ptr(stream)
        N.check(L.pf_png_inflate(zdev.data_ptr(), zoff_d.data_ptr(), n, raw.data_ptr(), roff_d.data_ptr(),
                                 rlen_d.data_ptr(), status.data_ptr(), sp), "pf_png_inflate")
        N.check(L.pf_png_unfilter(raw.data_ptr(), roff_d.data_ptr(), tw_d.data_ptr(), th_d.data_ptr(),
                                  dst_d.data_ptr(), T, n, status.data_ptr(), sp), "pf_png_unfilter")
        st = status.cpu().numpy()
        bad = np.flatnonzero(st)
        if len(bad):
            t = part[int(bad[0])]
            raise DecodeError(f"cannot decode png tile ({t[0]}, {t[1]}): inflate/unfilter status {int(st[bad[0]])}")


_JPEG_TILE_BYTES, _JPEG_HUFF_BYTES = 184, 1420  # sizeof(JpegTile), sizeof(JpegHuff) (csrc/pf_jpeg.h)


def _decode_jpeg_tiles(level, T: int, tiles, stream=None) -> list:
    """Decode JPEG tiles (tx, ty, tw, th, file bytes) on the GPU into a dense level
    [ty, tx, T, T, 3]: native host preparation (pf_jpeg_prepare) + pf_jpeg_decode.  Returns the
    indices of tiles the GPU path does not take (progressive, restart markers, other chroma
    sampling), which the caller decodes on the host."""
    torch = N.require_cuda()
    L = N.lib()
    n = len(tiles)
    if n == 0:
        return []
    nx = level.shape[1]
    tb = T * T * 3
    off = np.zeros(n + 1, np.int64)
    off[1:] = np.cumsum([len(t[4]) for t in tiles])
    data = np.frombuffer(b"".join(t[4] for t in tiles), np.uint8)
    tw = np.array([t[2] for t in tiles], np.int32)
    th = np.array([t[3] for t in tiles], np.int32)
    dst = np.array([int(level.data_ptr()) + (t[1] * nx + t[0]) * tb for t in tiles], np.uint64)
    max_blk = int(np.sum(((tw.astype(np.int64) + 7) // 8) * ((th.astype(np.int64) + 7) // 8) * 3))
    rec = np.zeros(n * _JPEG_TILE_BYTES, np.uint8)
    ok = np.zeros(n, np.int32)
    pool = np.zeros(len(data) + 8, np.uint8)
    huff = np.zeros(4 * n * _JPEG_HUFF_BYTES, np.uint8)
    quant = np.zeros(4 * n * 64, np.uint16)
    bt, bc, bi = (np.zeros(max(max_blk, 1), np.int32) for _ in range(3))
    px = np.zeros(n, np.int64)
    counts = np.zeros(7, np.int64)
    p = lambda a: a.ctypes.data  # noqa: E731
    N.check(L.pf_jpeg_prepare(p(data), p(off), p(tw), p(th), p(dst), n, p(rec), p(ok), p(pool), p(huff), p(quant),
                              p(bt), p(bc), p(bi), p(px), p(counts)), "pf_jpeg_prepare")
    nh, nq, nblk, ndata, ncoef, nplane, npx = (int(v) for v in counts)
    if nblk:
        dv = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", non_blocking=False)  # noqa: E731
        rec_d, pool_d = dv(rec), dv(pool[:ndata + 8])
        huff_d, quant_d = dv(huff[:nh * _JPEG_HUFF_BYTES]), dv(quant[:nq * 64])
        bt_d, bc_d, bi_d, px_d = dv(bt[:nblk]), dv(bc[:nblk]), dv(bi[:nblk]), dv(px)
        coef = torch.empty(ncoef, dtype=torch.int16, device="cuda")
        planes = torch.empty(nplane, dtype=torch.uint8, device="cuda")
        status = torch.from_numpy(ok.copy()).cuda()  # host-path tiles are skipped by the kernels
        N.check(L.pf_jpeg_decode(rec_d.data_ptr(), n, pool_d.data_ptr(), huff_d.data_ptr(), quant_d.data_ptr(),
                                 coef.data_ptr(), planes.data_ptr(), bt_d.data_ptr(), bc_d.data_ptr(), bi_d.data_ptr(),
                                 nblk, px_d.data_ptr(), npx, T, status.data_ptr(), N.stream_ptr(stream)),
                "pf_jpeg_decode")
        st = status.cpu().numpy()
        bad = np.flatnonzero((st != 0) & (ok == 0))
        if len(bad):
            t = tiles[int(bad[0])]
            raise DecodeError(f"cannot decode jpeg tile ({t[0]}, {t[1]}): entropy status {int(st[bad[0]])}")
    return [int(i) for i in np.flatnonzero(ok)]


def _read_chunk(root: Path, loc: dict, tw: int, th: int) -> np.ndarray:
    data = _read_chunk_bytes(root, loc)
    if loc["codec"] == "raw":
        if len(data) != tw * th * 3:
            raise DecodeError(f"raw tile has {len(data)} bytes, expected {tw * th * 3}")
        return np.frombuffer(data, dtype=np.uint8).reshape(th, tw, 3)
    import io

    from PIL import Image

    try:
        arr = np.asarray(Image.open(io.BytesIO(data)).convert("RGB"))
    except Exception as exc:  # noqa: BLE001 - mirrors decode_tile's catch-all
        raise DecodeError(f"cannot decode {loc['codec']} tile: {exc}") from exc
    if arr.shape[:2] != (th, tw):
        raise DecodeError(f"decoded tile is {arr.shape[1]}x{arr.shape[0]}, expected {tw}x{th}")
    return arr


CODECS = ("raw", "png", "jpeg")
_CODEC_EXT = {"raw": ".raw", "png": ".png", "jpeg": ".jpg"}


def encode_tile(arr: np.ndarray, codec: str) -> bytes:
    """encode_tile (pkg/store.py:416-426): raw bytes, or Pillow PNG / JPEG q90."""
    if codec == "raw":
        return np.ascontiguousarray(arr).tobytes()
    import io

    from PIL import Image

    buf = io.BytesIO()
    Image.fromarray(np.ascontiguousarray(arr)).save(buf, format="PNG" if codec == "png" else "JPEG",
                                                    **({"quality": 90} if codec == "jpeg" else {}))
    return buf.getvalue()


def _write_json(path: Path, doc: dict) -> None:
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(json.dumps(doc, indent=2), encoding="utf-8")


def ingest_image(pixels, slide_id: str, base_mpp: float, store_root, *, tile_size: int = 256,
                 downsample_factor: int = 2, codec: str = "png", layout: str = "files", return_slide: bool = False):
    """Drop-in ingest_image (pkg/store.py:462-565) with the pyramid built on the GPU.

    Level 0 is uploaded once, levels 1.. come from pf_build_level (the reference's
    _box_downsample, bit-exact), and the tiles are written in the reference's on-disk format
    (SPEC.md:113): per-tile files or one packed blob with byte-range locators, the slide
    record JSON and the store index.  Returns the SlideRecord (and the HBM-resident GpuSlide
    with ``return_slide``)."""
    if codec not in CODECS:
        raise ValueError(f"codec must be one of {CODECS}")
    if layout not in ("files", "packed"):
        raise ValueError("layout must be 'files' or 'packed'")
    slide = GpuSlide.from_array(pixels, slide_id, base_mpp, tile_size=tile_size,
                                downsample_factor=downsample_factor)
    rec = SlideRecord(slide_id, base_mpp, tile_size, list(slide.record.levels))
    root = Path(store_root)
    T = tile_size
    try:
        pack_fh = None
        pack_rel = f"chunks/{slide_id}.bin"
        if layout == "packed":
            (root / pack_rel).parent.mkdir(parents=True, exist_ok=True)
            pack_fh = open(root / pack_rel, "wb")
        offset = 0
        for li in range(len(rec.levels)):
            nx, ny = rec.tile_grid(li)
            host = slide.levels[li].cpu().numpy()  # [ty, tx, T, T, 3] padded tiles
            for ty in range(ny):
                for tx in range(nx):
                    tw, th = rec.tile_dims(li, tx, ty)
                    data = encode_tile(host[ty, tx, :th, :tw], codec)
                    if layout == "files":
                        rel = f"chunks/{slide_id}/{li}/{tx}_{ty}{_CODEC_EXT[codec]}"
                        (root / rel).parent.mkdir(parents=True, exist_ok=True)
                        (root / rel).write_bytes(data)
                        loc = {"kind": "inline-file", "path": rel, "codec": codec}
                    else:
                        pack_fh.write(data)
                        loc = {"kind": "byte-range", "path": pack_rel, "codec": codec, "offset": offset,
                               "length": len(data)}
                        offset += len(data)
                    rec.chunks[(li, tx, ty)] = loc
        if pack_fh is not None:
            pack_fh.close()
    except OSError as exc:
        raise StoreError(f"cannot write chunks under {root}: {exc}") from exc
    rec.validate()
    try:
        _write_json(root / "slides" / f"{slide_id}.json", rec.to_json_dict())
        idx_path = root / "index.json"
        index = json.loads(idx_path.read_text(encoding="utf-8")) if idx_path.exists() else {
            "format_version": STORE_FORMAT_VERSION, "slides": [], "records": {}}
        if slide_id not in index["slides"]:
            index["slides"].append(slide_id)
        index["records"][slide_id] = f"slides/{slide_id}.json"
        _write_json(idx_path, {"format_version": index["format_version"], "slides": index["slides"],
                               "records": index["records"]})
    except OSError as exc:
        raise StoreError(f"cannot write metadata under {root}: {exc}") from exc
    return (rec, slide) if return_slide else rec


def plan_specs(requests, records, errors: list | None = None) -> np.ndarray:
    """Host read plan for explicit region requests.

    requests: iterable of (slide_index, (x, y, w, h), target_mpp, out_size).
    Validates bounds exactly like read_region/_read_window (pkg/store.py:667-702)
    and fills level/side/sx/sy.  With ``errors`` (a list) a failing request does not raise:
    ``(index, exception)`` is appended and its row is left zeroed (side 0).
    """
    reqs = list(requests)
    specs = np.zeros(len(reqs), dtype=N.SPEC_DTYPE)
    level_cache: dict = {}
    for i, (si, rect, mpp, out_size) in enumerate(reqs):
        if errors is not None:
            try:
                _plan_one(specs, i, si, rect, mpp, out_size, records, level_cache)
            except Exception as exc:  # noqa: BLE001 - the caller's error policy decides
                errors.append((i, exc))
            continue
        _plan_one(specs, i, si, rect, mpp, out_size, records, level_cache)
    return specs


def _plan_one(specs, i, si, rect, mpp, out_size, records, level_cache):
    """One request of plan_specs: read_region's checks (pkg/store.py:667-702), row i filled."""
    rec = records[si]
    x, y, w, h = (int(v) for v in rect)
    if out_size < 1:
        raise ValueError("out_size must be >= 1")
    if w < 1 or h < 1:
        raise OutOfBoundsError("rect must have positive extent")
    if x < 0 or y < 0 or x + w > rec.width or y + h > rec.height:
        raise OutOfBoundsError(f"rect {tuple(rect)} outside level-0 bounds {rec.width}x{rec.height}")
    key = (si, float(mpp))
    if key not in level_cache:
        level_cache[key] = select_level(rec, float(mpp))
    li = level_cache[key]
    lv = rec.levels[li]
    side = max(1, round_half_away(out_size * mpp / lv.mpp))
    sx, sy = round_half_away(x / lv.downsample), round_half_away(y / lv.downsample)
    if sx < -1 or sy < -1 or sx + side > lv.width + 1 or sy + side > lv.height + 1:
        raise OutOfBoundsError(f"window ({sx}, {sy}, {side}, {side}) outside level {li} ({lv.width}x{lv.height})")
    specs[i] = (i, mpp, si, x, y, w, h, out_size, -1, li, side, sx, sy, 0)


_FITS: dict = {}


def _generic_indices(specs, out_size: int, dtype_code: int) -> list:
    """Indices of host specs whose window pf_read_regions' fused kernel cannot stage."""
    arr = np.asarray(specs)
    out = []
    for i, side in enumerate(arr["side"].tolist()):
        key = (int(side), int(out_size), int(dtype_code))
        if key not in _FITS:
            f = N.C.c_int32(0)
            N.check(N.lib().pf_read_region_fits(key[0], key[1], key[2], N.C.byref(f)), "pf_read_region_fits")
            _FITS[key] = bool(f.value)
        if not _FITS[key]:
            out.append(i)
    return out


def _read_generic(descs, spec, out_size, code, lay, m, s, out, stream):
    """pf_read_region_generic for one host spec (level/side/sx/sy planned) into `out` (one patch)."""
    import torch

    st = stream if stream is not None else torch.cuda.current_stream()
    rec = np.ascontiguousarray(np.asarray(spec, dtype=N.SPEC_DTYPE).reshape(1))
    need = N.C.c_int64(0)
    N.check(N.lib().pf_read_region_generic_scratch_bytes(int(rec["side"][0]), out_size, N.C.byref(need)),
            "pf_read_region_generic_scratch_bytes")
    with torch.cuda.stream(st):
        scratch = torch.empty((max(1, need.value),), dtype=torch.uint8, device="cuda")
    N.check(N.lib().pf_read_region_generic(descs.data_ptr(), rec.ctypes.data, out_size, code, lay,
                                           N.C.cast(m, N.C.c_void_p), N.C.cast(s, N.C.c_void_p),
                                           scratch.data_ptr(), need.value, out.data_ptr(), N.stream_ptr(st)),
            "pf_read_region_generic")


class SlideSet:
    """Slides addressed by index in one device call (pf_slide_desc array in HBM)."""

    def __init__(self, slides):
        torch = N.require_cuda()
        self.slides = list(slides)
        self.ids = [s.record.slide_id for s in self.slides]
        if len(set(self.ids)) != len(self.ids):
            raise ValueError("duplicate slide ids")
        self.index = {sid: i for i, sid in enumerate(self.ids)}
        raw = b"".join(bytes(s.desc) for s in self.slides)
        self.descs = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
        for s in self.slides:
            if hasattr(s, "_sets"):
                s._sets.add(self)

    def check_status(self, stream=None) -> None:
        """OutOfBoundsError if any device read since the last check hit a non-resident tile."""
        for s in self.slides:
            if getattr(s, "compacted", False):
                s.check_status(stream)

    def _refresh(self, slide) -> None:
        """Rewrite the device descriptor of ``slide`` in place (GpuSlide.compact)."""
        import torch

        d = bytes(slide.desc)
        for i, s in enumerate(self.slides):
            if s is slide:
                self.descs[i * len(d):(i + 1) * len(d)].copy_(torch.frombuffer(bytearray(d), dtype=torch.uint8))
        torch.cuda.synchronize()

    def __len__(self):
        return len(self.slides)

    @property
    def records(self):
        return [s.record for s in self.slides]

    def specs_to_device(self, specs):
        import torch

        if isinstance(specs, torch.Tensor):
            return specs
        arr = np.ascontiguousarray(specs, dtype=N.SPEC_DTYPE)
        return torch.from_numpy(arr.view(np.uint8).reshape(len(arr), 64)).cuda(non_blocking=False)

    def read_regions(self, specs, out_size: int, *, dtype: str = "u8", layout: str = "hwc", mean=(0.5, 0.5, 0.5),
                     std=(0.5, 0.5, 0.5), out=None, stream=None, planned: bool = False,
                     passthrough_only: bool = False):
        """Batched read_region on device -> tensor [n, S, S, 3] (hwc) or [n, 3, S, S] (nchw).

        dtype "u8" returns raw pixels; "f32"/"bf16" apply (v/255 - mean)/std
        (normalize_patch, pkg/pipeline.py:152-155, for mean = std = 0.5).
        ``passthrough_only``: the caller knows every spec reads its window unresampled
        (side == out_size); the lean passthrough kernel serves the call (PF_SKIP_RESAMPLED:
        a resampled spec's output would be left untouched).
        """
        torch = N.require_cuda()
        dspecs = self.specs_to_device(specs)
        n = dspecs.shape[0]
        dt = {"u8": (N.PF_U8, torch.uint8), "f32": (N.PF_F32, torch.float32), "bf16": (N.PF_BF16, torch.bfloat16)}
        code, tdt = dt[dtype]
        lay = {"hwc": N.PF_HWC, "nchw": N.PF_NCHW}[layout]
        shape = (n, out_size, out_size, 3) if lay == N.PF_HWC else (n, 3, out_size, out_size)
        flags = N.PF_SKIP_RESAMPLED if passthrough_only else 0
        if out is None:
            out = torch.empty(shape, dtype=tdt, device="cuda")
        sp = N.stream_ptr(stream)
        m = (N.C.c_float * 3)(*mean)
        s = (N.C.c_float * 3)(*std)
        big = [] if isinstance(specs, torch.Tensor) else _generic_indices(specs, out_size, code)
        if big:  # windows the fused kernel cannot stage: one generic PIL read each (rare)
            host = np.ascontiguousarray(specs, dtype=N.SPEC_DTYPE)
            keep = np.ones(n, dtype=bool)
            keep[big] = False
            for i in big:
                _read_generic(self.descs, host[i], out_size, code, lay, m, s, out[i], stream)
            if keep.any():
                idx = np.flatnonzero(keep)
                sub = self.read_regions(host[idx], out_size, dtype=dtype, layout=layout, mean=mean, std=std,
                                        stream=stream, planned=planned)
                out[torch.from_numpy(idx).to(out.device)] = sub
            return out
        if not planned:
            N.check(N.lib().pf_plan_regions(self.descs.data_ptr(), dspecs.data_ptr(), n, sp), "pf_plan_regions")
        N.check(
            N.lib().pf_read_regions(self.descs.data_ptr(), dspecs.data_ptr(), n, out_size, code, lay | flags,
                                    N.C.cast(m, N.C.c_void_p), N.C.cast(s, N.C.c_void_p), out.data_ptr(), sp),
            "pf_read_regions",
        )
        return out

    def read_specs(self, patch_specs, *, dtype="u8", layout="hwc", mean=(0.5, 0.5, 0.5), std=(0.5, 0.5, 0.5)):
        """read_regions for reference PatchSpec objects (uniform out_size)."""
        ps = list(patch_specs)
        if not ps:
            raise ValueError("no specs")
        sizes = {p.out_size for p in ps}
        if len(sizes) != 1:
            raise ValueError("read_specs needs a uniform out_size")
        specs = plan_specs([(self.index[p.slide_id], p.rect(), p.target_mpp, p.out_size) for p in ps], self.records)
        specs["seq"] = [p.seq for p in ps]
        return self.read_regions(specs, ps[0].out_size, dtype=dtype, layout=layout, mean=mean, std=std)
