"""Tissue foreground on the GPU: thumbnail masks, traced polygons, overlap tests.

Mirrors pkg/foreground.py: ``BinaryMask`` (37-61), ``ForegroundPolygon``
(64-133), ``mask_from_rgb`` (141-158), ``polygon_from_mask`` (169-220),
``overlap_fraction`` (246-286) and ``rect_polygon`` (289-298).  Masks and
overlap tests run as CUDA kernels; tracing runs once per slide in the native
library (host C++).  ``mask_from_saturation`` adds the BASELINE.json rule
(HSV saturation > 0.07 plus morphology).
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _native as N
from .errors import EmptyForegroundError

DEFAULT_LUMINANCE_THRESHOLD = 0.9
DEFAULT_SATURATION_THRESHOLD = 0.07
DEFAULT_MIN_REGION_PX = 64
OVERLAP_GRID = 128


@dataclass
class BinaryMask:
    """Boolean foreground grid at thumbnail scale (``scale`` = thumbnail px per level-0 px)."""

    bits: np.ndarray
    scale: float = 1.0

    def __post_init__(self):
        self.bits = np.asarray(self.bits, dtype=bool)
        if self.bits.ndim != 2 or self.bits.shape[0] < 1 or self.bits.shape[1] < 1:
            raise ValueError("mask must be a non-empty 2D grid")
        if not (0 < self.scale <= 1):
            raise ValueError(f"scale must be in (0, 1], got {self.scale}")

    @property
    def height(self) -> int:
        return self.bits.shape[0]

    @property
    def width(self) -> int:
        return self.bits.shape[1]


def _shoelace(ring: np.ndarray) -> float:
    x, y = ring[:, 0], ring[:, 1]
    return 0.5 * float(np.sum(x * np.roll(y, -1) - np.roll(x, -1) * y))


@dataclass
class ForegroundPolygon:
    """Closed rings in level-0 pixel coordinates, even-odd semantics."""

    rings: list = field(default_factory=list)
    source_scale: float = 1.0
    slide_id: str = ""

    def __post_init__(self):
        clean = []
        for ring in self.rings:
            a = np.asarray(ring, dtype=np.float64)
            if a.ndim != 2 or a.shape[1] != 2 or a.shape[0] < 3:
                raise ValueError("each ring needs >= 3 (x, y) points")
            if a.shape[0] > 3 and np.array_equal(a[0], a[-1]):
                a = a[:-1]  # closure is implicit
            clean.append(a)
        self.rings = clean
        if not clean:
            raise EmptyForegroundError("polygon has no rings")
        if self.area() <= 0:
            raise ValueError("total signed polygon area must be positive")
        self._blob = None

    def area(self) -> float:
        return float(sum(_shoelace(r) for r in self.rings))

    def bounding_box(self) -> tuple:
        pts = np.concatenate(self.rings, axis=0)
        return (float(pts[:, 0].min()), float(pts[:, 1].min()), float(pts[:, 0].max()), float(pts[:, 1].max()))

    def translated(self, dx: float, dy: float) -> "ForegroundPolygon":
        return ForegroundPolygon([r + np.array([dx, dy]) for r in self.rings], self.source_scale, self.slide_id)

    def to_json_dict(self) -> dict:
        return {"slide_id": self.slide_id, "source_scale": self.source_scale, "rings": [r.tolist() for r in self.rings]}

    @classmethod
    def from_json_dict(cls, doc: dict) -> "ForegroundPolygon":
        return cls([np.asarray(r, dtype=np.float64) for r in doc["rings"]], float(doc.get("source_scale", 1.0)),
                   str(doc.get("slide_id", "")))

    def save(self, path) -> None:
        Path(path).write_text(json.dumps(self.to_json_dict()), encoding="utf-8")

    @classmethod
    def load(cls, path) -> "ForegroundPolygon":
        return cls.from_json_dict(json.loads(Path(path).read_text(encoding="utf-8")))

    # -- device slab index --------------------------------------------------
    def flat(self):
        xy = np.ascontiguousarray(np.concatenate(self.rings, axis=0), dtype=np.float64)
        off = np.zeros(len(self.rings) + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(r) for r in self.rings])
        return xy, off

    def index_blob(self) -> np.ndarray:
        """Host slab index (pf_polygon_index_build)."""
        xy, off = self.flat()
        n = C.c_int64(0)
        L = N.lib()
        N.check(L.pf_polygon_index_size(xy.ctypes.data, off.ctypes.data, len(self.rings), C.byref(n)),
                "pf_polygon_index_size")
        blob = np.zeros(n.value, dtype=np.uint8)
        N.check(L.pf_polygon_index_build(xy.ctypes.data, off.ctypes.data, len(self.rings), blob.ctypes.data, n.value),
                "pf_polygon_index_build")
        return blob

    def device_blob(self):
        """Slab index resident in HBM (cached per device)."""
        torch = N.require_cuda()
        dev = torch.cuda.current_device()
        if self._blob is None:
            self._blob = {}
        if dev not in self._blob:
            self._blob[dev] = torch.from_numpy(self.index_blob()).cuda()
        return self._blob[dev]

    def device_raster(self, cell: float | None = None):
        """Classification raster of the polygon in HBM (pf_polygon_raster_build, cached): 2-bit
        cells of ``cell`` px (default: 32, doubled until the raster has at most 16 M cells)."""
        torch = N.require_cuda()
        bbox = (C.c_double * 4)(*self.bounding_box())
        if cell is None:
            cell = 32.0
            while ((bbox[2] - bbox[0]) / cell + 3) * ((bbox[3] - bbox[1]) / cell + 3) > (1 << 24):
                cell *= 2.0
        key = (torch.cuda.current_device(), float(cell))
        cache = getattr(self, "_rasters", None)
        if cache is None:
            cache = self._rasters = {}
        if key not in cache:
            nbytes = C.c_int64(0)
            N.check(N.lib().pf_polygon_raster_bytes(bbox, key[1], C.byref(nbytes)), "pf_polygon_raster_bytes")
            out = torch.empty((nbytes.value,), dtype=torch.uint8, device="cuda")
            st = torch.cuda.current_stream()
            N.check(N.lib().pf_polygon_raster_build(self.device_blob().data_ptr(), bbox, key[1], out.data_ptr(),
                                                    nbytes.value, N.stream_ptr(st)), "pf_polygon_raster_build")
            cache[key] = out
        return cache[key]


def _to_device_rgb(thumbnail):
    torch = N.require_cuda()
    if isinstance(thumbnail, torch.Tensor):
        t = thumbnail
        if t.device.type != "cuda":
            t = t.cuda()
        t = t.contiguous()  # the C ABI reads the raw row-major buffer
    else:
        arr = np.asarray(thumbnail)
        if arr.ndim != 3 or arr.shape[2] != 3:
            raise ValueError(f"expected an RGB (H, W, 3) image, got shape {arr.shape}")
        t = torch.from_numpy(np.ascontiguousarray(arr.astype(np.uint8))).cuda()
    if t.ndim != 3 or t.shape[2] != 3:
        raise ValueError(f"expected an RGB (H, W, 3) image, got shape {tuple(t.shape)}")
    return t.to(torch.uint8).contiguous()


def mask_device(thumbnail, mode: int, threshold: float, morph_radius: int = 0, stream=None):
    """Run pf_mask; returns a (h, w) uint8 {0,1} device tensor."""
    torch = N.require_cuda()
    t = _to_device_rgb(thumbnail)
    h, w = int(t.shape[0]), int(t.shape[1])
    out = torch.empty((h, w), dtype=torch.uint8, device="cuda")
    scratch = torch.empty((2 * h * w,), dtype=torch.uint8, device="cuda") if morph_radius > 0 else None
    N.check(
        N.lib().pf_mask(t.data_ptr(), h, w, mode, float(threshold), int(morph_radius), out.data_ptr(),
                        scratch.data_ptr() if scratch is not None else None, N.stream_ptr(stream)),
        "pf_mask",
    )
    return out


def mask_from_rgb(thumbnail, luminance_threshold: float = DEFAULT_LUMINANCE_THRESHOLD, scale: float = 1.0) -> BinaryMask:
    """Luminance mask (pkg/foreground.py:141-158) on the GPU; bit-exact."""
    if not (0 < luminance_threshold < 1):
        raise ValueError("luminance_threshold must be in (0, 1)")
    bits = mask_device(thumbnail, N.PF_MASK_LUMINANCE, luminance_threshold)
    return BinaryMask(bits.cpu().numpy().astype(bool), scale)


def mask_from_saturation(thumbnail, saturation_threshold: float = DEFAULT_SATURATION_THRESHOLD, morph_radius: int = 1,
                         scale: float = 1.0) -> BinaryMask:
    """BASELINE mask: HSV saturation > threshold, then binary opening + closing ((2r+1)^2 square)."""
    bits = mask_device(thumbnail, N.PF_MASK_SATURATION, saturation_threshold, morph_radius)
    return BinaryMask(bits.cpu().numpy().astype(bool), scale)


def load_mask_png(path, scale: float = 1.0) -> BinaryMask:
    """External mask image; any nonzero pixel is foreground (pkg/foreground.py:161-166)."""
    from PIL import Image

    arr = np.asarray(Image.open(path))
    if arr.ndim == 3:
        arr = arr.max(axis=2)
    return BinaryMask(arr != 0, scale)


def polygon_from_mask(mask: BinaryMask, min_region_px: float = DEFAULT_MIN_REGION_PX, slide_id: str = "") -> ForegroundPolygon:
    """Marching-squares rings scaled to level 0 (pkg/foreground.py:169-220), native tracer."""
    bits = np.ascontiguousarray(mask.bits, dtype=np.uint8)
    h, w = bits.shape
    L = N.lib()
    npts, nr = C.c_int64(0), C.c_int32(0)
    rc = L.pf_polygon_trace(bits.ctypes.data, h, w, float(mask.scale), float(min_region_px), None, 0, None, 0,
                            C.byref(npts), C.byref(nr))
    if rc != N.PF_ERR_CAPACITY:
        N.check(rc, "pf_polygon_trace")
    xy = np.zeros((npts.value, 2), dtype=np.float64)
    off = np.zeros(nr.value + 1, dtype=np.int64)
    N.check(L.pf_polygon_trace(bits.ctypes.data, h, w, float(mask.scale), float(min_region_px), xy.ctypes.data,
                               npts.value, off.ctypes.data, nr.value + 1, C.byref(npts), C.byref(nr)),
            "pf_polygon_trace")
    rings = [xy[off[i]:off[i + 1]].copy() for i in range(nr.value)]
    return ForegroundPolygon(rings, mask.scale, slide_id)


def polygon_from_mask_device(mask, scale: float, min_region_px: float = DEFAULT_MIN_REGION_PX, slide_id: str = "",
                             stream=None) -> ForegroundPolygon:
    """polygon_from_mask (pkg/foreground.py:169-220) traced on the GPU (pf_polygon_trace_device):
    ``mask`` is a (h, w) device tensor (e.g. mask_device's output), so the mask never leaves HBM.
    The rings equal polygon_from_mask's on the same bits, vertex for vertex."""
    torch = N.require_cuda()
    if not isinstance(mask, torch.Tensor) or mask.dim() != 2:
        raise ValueError("mask must be a (h, w) device tensor")
    m = mask.to(device="cuda", dtype=torch.uint8).contiguous()
    h, w = int(m.shape[0]), int(m.shape[1])
    L = N.lib()
    need = C.c_int64(0)
    N.check(L.pf_polygon_trace_device_scratch_bytes(h, w, C.byref(need)), "pf_polygon_trace_device_scratch_bytes")
    st = stream if stream is not None else torch.cuda.current_stream()
    with torch.cuda.stream(st):
        scratch = torch.empty((need.value,), dtype=torch.uint8, device="cuda")
    npts, nr = C.c_int64(0), C.c_int32(0)
    rc = L.pf_polygon_trace_device(m.data_ptr(), h, w, float(scale), float(min_region_px), scratch.data_ptr(),
                                   need.value, None, 0, None, 0, C.byref(npts), C.byref(nr), N.stream_ptr(st))
    if rc != N.PF_ERR_CAPACITY:
        N.check(rc, "pf_polygon_trace_device")
    with torch.cuda.stream(st):
        xy = torch.empty((npts.value, 2), dtype=torch.float64, device="cuda")
        off = torch.empty((nr.value + 1,), dtype=torch.int64, device="cuda")
    N.check(L.pf_polygon_trace_device(m.data_ptr(), h, w, float(scale), float(min_region_px), scratch.data_ptr(),
                                      need.value, xy.data_ptr(), npts.value, off.data_ptr(), nr.value + 1,
                                      C.byref(npts), C.byref(nr), N.stream_ptr(st)), "pf_polygon_trace_device")
    xy_h, off_h = xy.cpu().numpy(), off.cpu().numpy()
    rings = [xy_h[off_h[i]:off_h[i + 1]].copy() for i in range(nr.value)]
    return ForegroundPolygon(rings, scale, slide_id)


def overlap_fractions(poly: ForegroundPolygon, rects, grid: int = OVERLAP_GRID, stream=None):
    """Batched overlap_fraction on device; rects (n, 4) (x, y, w, h) -> float64 device tensor."""
    torch = N.require_cuda()
    if grid < 32:
        raise ValueError("grid must be at least 32")
    r = rects if isinstance(rects, torch.Tensor) else torch.as_tensor(np.asarray(rects, dtype=np.float64))
    r = r.to(device="cuda", dtype=torch.float64).reshape(-1, 4).contiguous()
    if bool(((r[:, 2] <= 0) | (r[:, 3] <= 0)).any()):
        raise ValueError("rect width and height must be positive")
    out = torch.empty((r.shape[0],), dtype=torch.float64, device="cuda")
    blob = poly.device_blob()
    N.check(N.lib().pf_overlap_fraction(blob.data_ptr(), r.data_ptr(), r.shape[0], grid, out.data_ptr(),
                                        N.stream_ptr(stream)), "pf_overlap_fraction")
    return out


def overlap_fraction(poly: ForegroundPolygon, rect, grid: int = OVERLAP_GRID) -> float:
    """Drop-in overlap_fraction (pkg/foreground.py:246-286) for one rect."""
    x, y, w, h = rect
    if w <= 0 or h <= 0:
        raise ValueError("rect width and height must be positive")
    if grid < 32:
        raise ValueError("grid must be at least 32")
    return float(overlap_fractions(poly, [[x, y, w, h]], grid)[0].item())


def rect_polygon(x: float, y: float, w: float, h: float, slide_id: str = "") -> ForegroundPolygon:
    """Axis-aligned rectangle, positively oriented (pkg/foreground.py:289-298)."""
    ring = np.array([[x, y], [x, y + h], [x + w, y + h], [x + w, y]], dtype=np.float64)
    if _shoelace(ring) < 0:
        ring = ring[::-1]
    return ForegroundPolygon([ring], slide_id=slide_id)
