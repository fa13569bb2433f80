"""CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).

Each function names the reference lines it restates
(pkg/<m>.py = /root/reference/pkg/src/patchforge/<m>.py).
"""

from __future__ import annotations

import math
from collections import deque

import numpy as np

# ---------------------------------------------------------------------------
# rng — pkg/rng.py:13-109
M64 = (1 << 64) - 1


def mix64(x: int) -> int:  # rng.py:25-30
    x &= M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def fnv1a(b: bytes) -> int:  # rng.py:33-37
    h = 0xCBF29CE484222325
    for c in b:
        h = ((h ^ c) * 0x100000001B3) & M64
    return h


class Stream:
    """RandomStream (rng.py:40-109): draw i = mix64(key + i*gamma), i >= 1."""

    def __init__(self, seed: int, purpose: str):
        self.key = mix64((seed & M64) ^ fnv1a(purpose.encode()))
        self.n = 0

    def u64(self) -> int:  # rng.py:60-62
        self.n += 1
        return mix64((self.key + self.n * 0x9E3779B97F4A7C15) & M64)

    def uniform(self, lo=0.0, hi=1.0) -> float:  # rng.py:64-67
        return lo + ((self.u64() >> 11) * 2.0**-53) * (hi - lo)

    def randrange(self, n: int) -> int:  # rng.py:69-77
        lim = ((1 << 64) // n) * n
        while True:
            v = self.u64()
            if v < lim:
                return v % n

    def randint(self, lo: int, hi: int) -> int:  # rng.py:79-83
        return lo + self.randrange(hi - lo + 1)

    def weighted_index(self, ws) -> int:  # rng.py:88-103
        total = 0.0
        for w in ws:
            total += w
        u = self.uniform(0.0, total)
        acc = 0.0
        for i, w in enumerate(ws):
            acc += w
            if u < acc:
                return i
        return len(ws) - 1


# ---------------------------------------------------------------------------
# store — pkg/store.py


def round_half_away(x: float) -> int:  # store.py:70-72
    return int(math.floor(x + 0.5)) if x >= 0 else int(math.ceil(x - 0.5))


def select_level(mpps, target: float) -> int:  # store.py:568-581
    best, bd = 0, math.inf
    for i, m in enumerate(mpps):
        d = abs(math.log(m / target))
        if d < bd - 1e-12:
            best, bd = i, d
    return best


def box_downsample(arr: np.ndarray, f: int) -> np.ndarray:  # store.py:429-441
    h, w = arr.shape[:2]
    ri, ci = np.arange(0, h, f), np.arange(0, w, f)
    sums = np.add.reduceat(np.add.reduceat(arr.astype(np.float64), ri, axis=0), ci, axis=1)
    cnt = np.outer(np.diff(np.append(ri, h)), np.diff(np.append(ci, w)))[:, :, None]
    return np.floor(sums / cnt + 0.5).astype(np.uint8)


def pyramid(level0: np.ndarray, tile: int, factor: int) -> list:  # store.py:496-498
    levels = [level0]
    while max(levels[-1].shape[0], levels[-1].shape[1]) > tile:
        levels.append(box_downsample(levels[-1], factor))
    return levels


def read_window(level: np.ndarray, sx: int, sy: int, w: int, h: int) -> np.ndarray:  # store.py:690-724
    H, W = level.shape[:2]
    if sx < -1 or sy < -1 or sx + w > W + 1 or sy + h > H + 1:
        raise IndexError("window out of bounds")
    cx0, cy0 = max(sx, 0), max(sy, 0)
    cx1, cy1 = max(min(sx + w, W), cx0 + 1), max(min(sy + h, H), cy0 + 1)
    cx0, cy0 = min(cx0, W - 1), min(cy0, H - 1)
    core = level[cy0:cy1, cx0:cx1]
    xs = np.clip(np.arange(sx, sx + w), cx0, cx1 - 1) - cx0
    ys = np.clip(np.arange(sy, sy + h), cy0, cy1 - 1) - cy0
    return core[np.ix_(ys, xs)]


def read_region(levels, mpps, downsamples, rect, target_mpp: float, out_size: int) -> np.ndarray:
    """Slide.read_region (store.py:651-688) over in-memory levels (PIL resize as the reference)."""
    from PIL import Image

    x, y, w, h = rect
    if out_size < 1:
        raise ValueError("out_size must be >= 1")
    lw, lh = levels[0].shape[1], levels[0].shape[0]
    if w < 1 or h < 1 or x < 0 or y < 0 or x + w > lw or y + h > lh:  # store.py:668-675
        raise IndexError(f"rect {tuple(rect)} outside level-0 bounds {lw}x{lh}")
    li = select_level(mpps, target_mpp)
    side = max(1, round_half_away(out_size * target_mpp / mpps[li]))
    sx, sy = round_half_away(x / downsamples[li]), round_half_away(y / downsamples[li])
    win = read_window(levels[li], sx, sy, side, side)
    if side == out_size:
        return np.ascontiguousarray(win)
    return np.asarray(Image.fromarray(np.ascontiguousarray(win)).resize((out_size, out_size), Image.Resampling.BILINEAR))


def normalize_patch(px, mean=0.5, std=0.5) -> np.ndarray:  # pipeline.py:152-155
    """(v/255 - mean)/std in float32; per-channel mean/std broadcast over a trailing RGB axis."""
    a = np.asarray(px, dtype=np.float32)
    return (a / np.float32(255.0) - np.asarray(mean, np.float32)) / np.asarray(std, np.float32)


# ---------------------------------------------------------------------------
# foreground — pkg/foreground.py
_LUMA = np.array([0.2126, 0.7152, 0.0722])


def mask_luminance(img: np.ndarray, thr: float = 0.9) -> np.ndarray:  # foreground.py:141-158
    return (np.asarray(img).astype(np.float64) @ _LUMA / 255.0) < thr


def mask_saturation(img: np.ndarray, thr: float = 0.07, radius: int = 1) -> np.ndarray:
    """BASELINE rule (not in the reference): HSV S > thr, then opening + closing (scipy)."""
    from scipy import ndimage

    a = np.asarray(img).astype(np.int64)
    mx, mn = a.max(axis=2), a.min(axis=2)
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.where(mx == 0, 0.0, (mx - mn).astype(np.float64) / mx.astype(np.float64))
    m = s > thr
    if radius > 0:
        st = np.ones((2 * radius + 1, 2 * radius + 1), dtype=bool)
        m = ndimage.binary_opening(m, structure=st)
        m = ndimage.binary_closing(m, structure=st)
    return m


def find_contours_binary(padded: np.ndarray):
    """Marching squares at iso 0.5, low-connected saddles, contour assembly in creation order.

    Restates the published algorithm behind skimage.measure.find_contours (the
    reference's call at foreground.py:184; scikit-image is not installed here):
    segments per 2x2 square in row-major order, then joined head/tail keeping
    the older contour's index.  Input values are 0/1 so every crossing is a
    midpoint.  Returns a list of (n, 2) (row, col) float arrays.
    """
    a = np.asarray(padded) > 0.5
    H, W = a.shape
    segs = []
    for r in range(H - 1):
        for c in range(W - 1):
            case = int(a[r, c]) | int(a[r, c + 1]) << 1 | int(a[r + 1, c]) << 2 | int(a[r + 1, c + 1]) << 3
            if case in (0, 15):
                continue
            top, bot = (r, c + 0.5), (r + 1, c + 0.5)
            lft, rgt = (r + 0.5, c), (r + 0.5, c + 1)
            table = {
                1: [(top, lft)], 2: [(rgt, top)], 3: [(rgt, lft)], 4: [(lft, bot)], 5: [(top, bot)],
                6: [(rgt, top), (lft, bot)], 7: [(rgt, bot)], 8: [(bot, rgt)], 9: [(top, lft), (bot, rgt)],
                10: [(bot, top)], 11: [(bot, lft)], 12: [(lft, rgt)], 13: [(top, rgt)], 14: [(lft, top)],
            }
            segs.extend(table[case])
    starts, ends, contours = {}, {}, {}
    nxt = 0
    for p, q in segs:
        if p == q:
            continue
        tail, tn = starts.pop(q, (None, None))
        head, hn = ends.pop(p, (None, None))
        if tail is not None and head is not None:
            if tail is head:
                head.append(q)
            elif tn > hn:
                head.extend(tail)
                contours.pop(tn, None)
                starts[head[0]] = (head, hn)
                ends[head[-1]] = (head, hn)
            else:
                tail.extendleft(reversed(head))
                starts.pop(head[0], None)
                contours.pop(hn, None)
                starts[tail[0]] = (tail, tn)
                ends[tail[-1]] = (tail, tn)
        elif tail is None and head is None:
            dq = deque((p, q))
            contours[nxt] = dq
            starts[p] = (dq, nxt)
            ends[q] = (dq, nxt)
            nxt += 1
        elif head is None:
            tail.appendleft(p)
            starts[p] = (tail, tn)
        else:
            head.append(q)
            ends[q] = (head, hn)
    return [np.array(list(c), dtype=np.float64) for _, c in sorted(contours.items())]


def shoelace(ring: np.ndarray) -> float:  # foreground.py:136-138
    x, y = ring[:, 0], ring[:, 1]
    return 0.5 * float(np.sum(x * np.roll(y, -1) - np.roll(x, -1) * y))


def points_in_polygon(points: np.ndarray, rings) -> np.ndarray:  # foreground.py:223-243
    pts = np.asarray(points, dtype=np.float64)
    px, py = pts[:, 0][:, None], pts[:, 1][:, None]
    inside = np.zeros(pts.shape[0], dtype=bool)
    for ring in rings:
        ring = np.asarray(ring, dtype=np.float64)
        x1, y1 = ring[:, 0][None, :], ring[:, 1][None, :]
        x2, y2 = np.roll(ring[:, 0], -1)[None, :], np.roll(ring[:, 1], -1)[None, :]
        crosses = (y1 > py) != (y2 > py)
        with np.errstate(divide="ignore", invalid="ignore"):
            x_at = x1 + (py - y1) * (x2 - x1) / (y2 - y1)
        inside ^= (crosses & (px < x_at)).sum(axis=1) % 2 == 1
    return inside


def polygon_from_mask(bits: np.ndarray, scale: float, min_region_px: float = 64.0):  # foreground.py:169-220
    if not np.asarray(bits).any():  # foreground.py:178-179 (EmptyForegroundError is a ValueError)
        raise ValueError("mask contains no foreground pixels")
    padded = np.pad(np.asarray(bits).astype(np.float64), 1)
    rings = []
    for ct in find_contours_binary(padded):
        ring = np.stack([ct[:, 1] - 1.0, ct[:, 0] - 1.0], axis=1)
        if np.array_equal(ring[0], ring[-1]):
            ring = ring[:-1]
        if ring.shape[0] < 3 or abs(shoelace(ring)) < min_region_px:
            continue
        rings.append(ring)
    out = []
    for i, ring in enumerate(rings):
        probe = ring.mean(axis=0)
        depth = sum(1 for j, o in enumerate(rings) if j != i and bool(points_in_polygon(probe.reshape(1, 2), [o])[0]))
        if (shoelace(ring) > 0) != (depth % 2 == 0):
            ring = ring[::-1]
        out.append(ring / scale)
    if not out:  # foreground.py:196-199
        raise ValueError(f"no region of at least {min_region_px} px^2 in the mask")
    return out


def bounding_box(rings) -> tuple:  # foreground.py:96-104
    p = np.concatenate(rings, axis=0)
    return float(p[:, 0].min()), float(p[:, 1].min()), float(p[:, 0].max()), float(p[:, 1].max())


def overlap_fraction(rings, rect, grid: int = 128, bbox=None) -> float:  # foreground.py:246-286
    x, y, w, h = rect
    bx0, by0, bx1, by1 = bbox or bounding_box(rings)
    if x >= bx1 or y >= by1 or x + w <= bx0 or y + h <= by0:
        return 0.0
    ex = x + np.arange(grid + 1) * (w / grid)
    ey = y + np.arange(grid + 1) * (h / grid)
    gx, gy = np.meshgrid(ex, ey, indexing="xy")
    corners = points_in_polygon(np.stack([gx.ravel(), gy.ravel()], axis=1), rings).reshape(grid + 1, grid + 1)
    cx, cy = (ex[:-1] + ex[1:]) / 2.0, (ey[:-1] + ey[1:]) / 2.0
    mx, my = np.meshgrid(cx, cy, indexing="xy")
    centres = points_in_polygon(np.stack([mx.ravel(), my.ravel()], axis=1), rings).reshape(grid, grid)
    cov = corners[:-1, :-1] & corners[1:, :-1] & corners[:-1, 1:] & corners[1:, 1:] & centres
    return float(cov.sum()) / float(grid * grid)


# ---------------------------------------------------------------------------
# sampler — pkg/sampler.py


def footprint_px(out_size: int, mpp: float, base_mpp: float) -> int:  # sampler.py:125-127
    return max(1, round_half_away(out_size * mpp / base_mpp))


def epoch_stream(slides, *, patch_size=256, min_fg=0.40, mpps=((0.25, 1.0),), seed=0, epoch_size=10,
                 max_attempts=100, strategy="uniform", weights=None, grid=128):
    """epoch_stream + sample_slide + sample_patch (sampler.py:130-227).

    slides: list of dicts {id, width, height, base_mpp, rings}.  Returns a list of
    (slide_index, x, y, fp, mpp, seq) plus the final stream counters.
    """
    s_slide, s_coords, s_mpp = Stream(seed, "slide"), Stream(seed, "coords"), Stream(seed, "mpp")
    ms = [m for m, _ in mpps]
    mw = [w for _, w in mpps]
    bboxes = [bounding_box(s["rings"]) for s in slides]
    limit = max(100, 10 * len(slides))
    fails, seq, out = 0, 0, []
    while seq < epoch_size:
        if strategy == "uniform":
            si = s_slide.randrange(len(slides))
        else:
            si = s_slide.weighted_index([(weights or {}).get(s["id"], 0.0) for s in slides])
        sl = slides[si]
        bx0, by0, bx1, by1 = bboxes[si]
        got = None
        for _ in range(max_attempts):
            mpp = ms[s_mpp.weighted_index(mw)]
            fp = footprint_px(patch_size, mpp, sl["base_mpp"])
            x_lo, y_lo = max(0, int(bx0)), max(0, int(by0))
            x_hi, y_hi = min(sl["width"] - fp, int(bx1)), min(sl["height"] - fp, int(by1))
            if x_hi < x_lo or y_hi < y_lo:
                continue
            x = s_coords.randint(x_lo, x_hi)
            y = s_coords.randint(y_lo, y_hi)
            if overlap_fraction(sl["rings"], (x, y, fp, fp), grid, bboxes[si]) >= min_fg:
                got = (si, x, y, fp, mpp, seq)
                break
        if got is None:
            fails += 1
            if fails >= limit:
                raise RuntimeError("NoSamplableSlideError")
            continue
        fails = 0
        out.append(got)
        seq += 1
    return out, (s_slide.n, s_coords.n, s_mpp.n)


def capped_stream(items, cap, seed: int, total=None) -> list:
    """capped_stream over a finite list (sampler.py:230-281): the first `cap` items pass through
    and are retained; then each output is retained[randrange(len)] from Stream(seed, "cache")."""
    out = []
    if cap is None:
        return list(items if total is None else items[:total])
    kept = []
    for it in items:
        if total is not None and len(out) >= total:
            return out
        if len(kept) >= cap:
            break
        kept.append(it)
        out.append(it)
    s = Stream(seed, "cache")
    while total is None or len(out) < total:
        out.append(kept[s.randrange(len(kept))])
        if total is None and len(out) > 10 ** 6:
            break
    return out


# ---------------------------------------------------------------------------
# antialiased bilinear resamplers (PIL Resample.c / torch uint8 AA), restated


def aa_axis_table(in_size: int, out_size: int, flavour: str):
    scale = in_size / out_size
    support = scale if scale >= 1.0 else 1.0
    inv = 1.0 / support
    ksize = int(math.ceil(support)) * 2 + 1
    mins, ws, wmax = [], [], 0.0
    for i in range(out_size):
        c = scale * (i + 0.5)
        xmin = max(int(c - support + 0.5), 0)
        xs = min(max(min(int(c + support + 0.5), in_size) - xmin, 0), ksize)
        w = []
        tot = 0.0
        for j in range(xs):
            t = abs(((j + xmin) - c + 0.5) * inv)
            v = 1.0 - t if t < 1.0 else 0.0
            w.append(v)
            tot += v
        if tot != 0.0:
            w = [v / tot for v in w]
        wmax = max([wmax] + w)
        mins.append(xmin)
        ws.append(w)
    if flavour == "torch":
        p = 0
        while p < 22 and int(0.5 + wmax * (1 << (p + 1))) < (1 << 15):
            p += 1
    else:
        p = 22
    q = [[int(-0.5 + v * (1 << p)) if v < 0 else int(0.5 + v * (1 << p)) for v in w] for w in ws]
    return mins, q, p


def aa_resize_axis(a: np.ndarray, axis: int, out: int, flavour: str) -> np.ndarray:
    n = a.shape[axis]
    if n == out:
        return a
    mins, q, p = aa_axis_table(n, out, flavour)
    b = np.moveaxis(a, axis, -1).astype(np.int64)
    res = np.empty(b.shape[:-1] + (out,), np.int64)
    for i in range(out):
        acc = np.full(b.shape[:-1], 1 << (p - 1), np.int64)
        for k, w in enumerate(q[i]):
            acc += b[..., mins[i] + k] * w
        res[..., i] = np.clip(acc >> p, 0, 255)
    return np.moveaxis(res.astype(np.uint8), -1, axis)


def aa_resize_hwc(img: np.ndarray, oh: int, ow: int, flavour: str) -> np.ndarray:
    """Horizontal pass then vertical, uint8 intermediate (both flavours)."""
    return aa_resize_axis(aa_resize_axis(img, 1, ow, flavour), 0, oh, flavour)
