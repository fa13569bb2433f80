"""Deterministic patch sampling on the GPU.

Mirrors pkg/sampler.py: ``SamplerConfig`` (34-58), ``PatchSpec`` (61-103),
``footprint_px`` (125-127), ``epoch_stream`` (196-227), manifests (284-297)
and ``validate_spec`` (300-323).  ``GpuSampler`` produces the exact spec
stream of ``epoch_stream`` — same slides, coordinates, magnifications and
seq numbers for the same (seed, config, slide set) — in device batches,
without host round trips between batches (csrc/pf_sampler.cu).
"""

from __future__ import annotations

import math

import ctypes as C
import json
from dataclasses import dataclass, field
from pathlib import Path


from . import _native as N
from . import rng
from .errors import NoSamplableSlideError
from .foreground import OVERLAP_GRID, ForegroundPolygon, overlap_fraction
from .store import SlideRecord, round_half_away, select_level

DEFAULT_PATCH_SIZE = 256
DEFAULT_MIN_FOREGROUND = 0.40
DEFAULT_EPOCH_SIZE = 1_280_000
DEFAULT_MAX_ATTEMPTS = 100


@dataclass
class SamplerConfig:
    patch_size: int = DEFAULT_PATCH_SIZE
    min_foreground: float = DEFAULT_MIN_FOREGROUND
    target_mpps: list = field(default_factory=lambda: [(0.25, 1.0)])
    slide_strategy: str = "uniform"
    slide_weights: dict | None = None
    epoch_size: int = DEFAULT_EPOCH_SIZE
    seed: int = 0
    max_attempts_per_slide: int = DEFAULT_MAX_ATTEMPTS

    def __post_init__(self):
        if not 0.0 <= self.min_foreground <= 1.0:
            raise ValueError("min_foreground must be in [0, 1]")
        if self.epoch_size < 1:
            raise ValueError("epoch_size must be >= 1")
        if self.patch_size < 1:
            raise ValueError("patch_size must be >= 1")
        if self.slide_strategy not in ("uniform", "weighted"):
            raise ValueError("slide_strategy must be 'uniform' or 'weighted'")
        if not self.target_mpps:
            raise ValueError("target_mpps must not be empty")
        ws = [w for _, w in self.target_mpps]
        if any(w < 0 for w in ws) or sum(ws) <= 0:
            raise ValueError("mpp weights must be >= 0 and not all zero")


@dataclass(frozen=True)
class PatchSpec:
    slide_id: str
    x: int
    y: int
    width: int
    height: int
    target_mpp: float
    out_size: int
    seq: int

    def rect(self) -> tuple:
        return (self.x, self.y, self.width, self.height)

    def to_json_line(self) -> str:
        return json.dumps({"slide_id": self.slide_id, "x": self.x, "y": self.y, "width": self.width,
                           "height": self.height, "target_mpp": self.target_mpp, "out_size": self.out_size,
                           "seq": self.seq})

    @classmethod
    def from_json_line(cls, line: str) -> "PatchSpec":
        d = json.loads(line)
        return cls(str(d["slide_id"]), int(d["x"]), int(d["y"]), int(d["width"]), int(d["height"]),
                   float(d["target_mpp"]), int(d["out_size"]), int(d["seq"]))


def footprint_px(out_size: int, target_mpp: float, base_mpp: float) -> int:
    return max(1, round_half_away(out_size * target_mpp / base_mpp))


def grid_positions(extent: int, size: int, stride: int) -> list:
    """Offsets 0, stride, ... while offset + size <= extent (pkg/sampler.py:187-193)."""
    if size > extent:
        raise ValueError(f"size {size} exceeds extent {extent}")
    if stride < 1:
        raise ValueError("stride must be >= 1")
    return list(range(0, extent - size + 1, stride))


class CappedCache:
    """Retains the first ``cap`` distinct specs; later draws replay them (pkg/sampler.py:230-252)."""

    def __init__(self, cap: int | None):
        if cap is not None and cap < 1:
            raise ValueError("cap must be >= 1 (or None for unlimited)")
        self.cap = cap
        self.stored: list = []

    @property
    def full(self) -> bool:
        return self.cap is not None and len(self.stored) >= self.cap

    def admit(self, spec) -> None:
        if self.cap is not None and not self.full:
            self.stored.append(spec)

    def draw(self, stream) -> "PatchSpec":
        if not self.stored:
            raise ValueError("cannot draw from an empty cache")
        return self.stored[stream.below(len(self.stored))]


def capped_stream(inner, cap: int | None, seed_or_stream, total: int | None = None):
    """Drop-in capped_stream (pkg/sampler.py:255-281): the first ``cap`` items pass through and
    are retained, afterwards every item is drawn uniformly from the retained set with the
    (seed, "cache") stream and the inner stream is not advanced.  ``seed_or_stream``: the seed of
    the reference's ``RandomStream(seed, "cache")`` or an ``rng.Stream``."""
    from . import rng

    stream = seed_or_stream if isinstance(seed_or_stream, rng.Stream) else rng.Stream(int(seed_or_stream), "cache")
    cache = CappedCache(cap)
    count = 0
    if cap is None:
        for item in inner:
            if total is not None and count >= total:
                return
            yield item
            count += 1
        return
    for item in inner:
        if total is not None and count >= total:
            return
        if cache.full:
            break
        cache.admit(item)
        yield item
        count += 1
    while total is None or count < total:
        yield cache.draw(stream)
        count += 1


def write_manifest(specs, path) -> int:
    n = 0
    with open(Path(path), "w", encoding="utf-8") as fh:
        for s in specs:
            fh.write(s.to_json_line() + "\n")
            n += 1
    return n


def read_manifest(path) -> list:
    with open(Path(path), encoding="utf-8") as fh:
        return [PatchSpec.from_json_line(line) for line in fh if line.strip()]


def validate_spec(spec: PatchSpec, record: SlideRecord, poly: ForegroundPolygon | None = None,
                  config: SamplerConfig | None = None) -> None:
    """Structural re-check of a spec (pkg/sampler.py:300-323); overlap on the GPU."""
    if spec.slide_id != record.slide_id:
        raise ValueError("spec references a different slide")
    if spec.x < 0 or spec.y < 0:
        raise ValueError("negative patch origin")
    if spec.x + spec.width > record.width or spec.y + spec.height > record.height:
        raise ValueError("patch footprint exceeds slide bounds")
    exp = footprint_px(spec.out_size, spec.target_mpp, record.base_mpp)
    if spec.width != exp or spec.height != exp:
        raise ValueError(f"footprint {spec.width} != round(out_size * mpp / base) = {exp}")
    if poly is not None and config is not None:
        frac = overlap_fraction(poly, spec.rect())
        if frac < config.min_foreground:
            raise ValueError(f"overlap {frac:.4f} below minimum {config.min_foreground}")


def _record_of(s) -> SlideRecord:
    return s.record if hasattr(s, "record") else s


class GpuSampler:
    """Device-resident epoch_stream: ``next_batch(n)`` -> [n, 64] uint8 spec tensor (pf_patch_spec).

    ``slides`` is a list of (GpuSlide or SlideRecord, ForegroundPolygon) pairs in
    the reference's order (it fixes the slide index a draw maps to).
    """

    def __init__(self, config: SamplerConfig, slides, *, slide_set=None, window: int | None = None,
                 rounds: int = 4, grid: int = OVERLAP_GRID, raster: bool = True):
        torch = N.require_cuda()
        if not slides:
            raise NoSamplableSlideError("no slides provided")
        if len(config.target_mpps) > N.PF_MAX_MPPS:
            raise ValueError(f"at most {N.PF_MAX_MPPS} target mpps")
        self.config = config
        self.records = [_record_of(s) for s, _ in slides]
        self.polys = [p for _, p in slides]
        self.ids = [r.slide_id for r in self.records]
        self.rounds = rounds
        self.grid = grid
        cfg = N.SamplerConfig()
        cfg.seed = config.seed & rng.M64
        cfg.key_slide = rng.stream_key(config.seed, "slide")
        cfg.key_coords = rng.stream_key(config.seed, "coords")
        cfg.key_mpp = rng.stream_key(config.seed, "mpp")
        cfg.min_foreground = float(config.min_foreground)
        for i, (m, w) in enumerate(config.target_mpps):
            cfg.mpp[i] = float(m)
            cfg.mpp_weight[i] = float(w)
        cfg.n_mpps = len(config.target_mpps)
        cfg.patch_size = int(config.patch_size)
        cfg.max_attempts = int(config.max_attempts_per_slide)
        cfg.n_slides = len(slides)
        cfg.grid = int(grid)
        if config.slide_strategy == "weighted":
            cfg.strategy = 1
            ws = [float((config.slide_weights or {}).get(sid, 0.0)) for sid in self.ids]
            if any(w < 0 for w in ws):
                raise ValueError("weights must be non-negative")
            if sum(ws) <= 0:
                raise ValueError("weights must not all be zero")
        else:
            cfg.strategy = 0
            ws = [0.0] * len(self.ids)
        self.cfg = cfg
        # per-slide tables
        table = (N.SamplerSlide * len(slides))()
        self.all_fit = True
        blobs = []
        fg_area = 0.0
        bbox_area = 0.0
        for i, (rec, poly) in enumerate(zip(self.records, self.polys)):
            t = table[i]
            blob = poly.device_blob()
            blobs.append(blob)
            t.poly_blob = int(blob.data_ptr())
            if raster:  # classification raster: windows far from every edge skip the lattice test
                ras = poly.device_raster()
                blobs.append(ras)
                t.raster = int(ras.data_ptr())
            bx0, by0, bx1, by1 = poly.bounding_box()
            t.bbox[:] = [bx0, by0, bx1, by1]
            t.weight = ws[i]
            t.width, t.height = rec.width, rec.height
            for k, (m, _) in enumerate(config.target_mpps):
                fp = footprint_px(config.patch_size, m, rec.base_mpp)
                t.fp[k] = fp
                t.x_lo[k] = max(0, int(bx0))
                t.y_lo[k] = max(0, int(by0))
                t.x_hi[k] = min(rec.width - fp, int(bx1))
                t.y_hi[k] = min(rec.height - fp, int(by1))
                if t.x_hi[k] < t.x_lo[k] or t.y_hi[k] < t.y_lo[k]:
                    self.all_fit = False
                li = select_level(rec, m)
                t.level[k] = li
                t.side[k] = max(1, round_half_away(config.patch_size * m / rec.levels[li].mpp))
            fg_area += max(poly.area(), 0.0)
            bbox_area += max((bx1 - bx0) * (by1 - by0), 1.0)
        self._blobs = blobs
        self.slides_dev = torch.frombuffer(bytearray(bytes(table)), dtype=torch.uint8).cuda()
        if slide_set is not None:
            if slide_set.ids != self.ids:
                raise ValueError("slide_set order must match the sampler's slide order")
            self.descs_dev = slide_set.descs
        else:
            from .store import GpuSlide  # noqa: F401  (records only: pointer-less descriptors)

            raw = b"".join(bytes(_desc_from_record(r)) for r in self.records)
            self.descs_dev = torch.frombuffer(bytearray(raw), dtype=torch.uint8).cuda()
        # acceptance-rate estimate sizes the speculation window
        self.p_est = max(0.05, min(1.0, 0.9 * fg_area / bbox_area))
        self.window = window
        self.state = torch.zeros(C.sizeof(N.SamplerState), dtype=torch.uint8, device="cuda")
        st = N.SamplerState()
        st.cur_slide = -1
        self.state.copy_(torch.frombuffer(bytearray(bytes(st)), dtype=torch.uint8))
        self._ws = None
        self._ws_stream = None
        self._ws_window = 0
        self._stats_host = torch.empty(C.sizeof(N.SamplerState), dtype=torch.uint8, pin_memory=True)
        self._stats_event = None

    def _window_for(self, n: int) -> int:
        if self.window:
            return max(32, (self.window + 31) // 32 * 32)
        # attempts for n accepts ~ negative binomial: mean n/p, sd sqrt(n(1-p))/p; 4 sd of slack
        # (overflow ~3e-5 per call), further rounds or the walk's exact path cover the rest.  p is
        # the stream's observed acceptance rate once a previous call's counters are back on the
        # host (copied asynchronously, never waited for), the polygon-area estimate before.
        self._poll_stats()
        p = self.p_est
        w = int(n / p + 4.0 * math.sqrt(n * (1.0 - p)) / p) + 32
        return min(max(32, (w + 31) // 32 * 32), 1 << 16)

    def _fits_table(self, window: int) -> bool:
        """pf_sample's walk keeps a next-accept table in shared memory when it fits (pf_sampler.cu,
        next_table): bitmaps + uint16 table + slide draws + emits <= 200 KB."""
        words = window // 32
        nt = (self.cfg.n_slides * words * 4 + 15) // 16 * 16 + self.cfg.n_slides * window * 2 + 8192 * 4 + window * 4
        return window < 0x4000 and window + self.cfg.max_attempts < 0x7FFF and nt <= 200 * 1024

    def next_batch(self, n: int, out=None, stream=None):
        """Next n specs of the stream as a device [n, 64] uint8 tensor; raises on stream failure lazily
        (call ``check()`` or read ``specs_host``).  A batch whose speculation window would not let
        the walk keep its table in shared memory is sampled in consecutive sub-batches (the stream
        is the same for any split)."""
        torch = N.require_cuda()
        st = stream if stream is not None else torch.cuda.current_stream()
        if self.rounds > 0 and not self.window and n > 64 and not self._fits_table(self._window_for(n)):
            with torch.cuda.stream(st):
                if out is None:
                    out = torch.empty((n, 64), dtype=torch.uint8, device="cuda")
            k = n
            while k > 64 and not self._fits_table(self._window_for(k)):
                k = (k + 1) // 2
            for i in range(0, n, k):
                self.next_batch(min(k, n - i), out=out[i:i + k], stream=st)
            return out
        window = self._window_for(n)
        nbytes = C.c_int64(0)
        N.check(N.lib().pf_sample_workspace_bytes(C.byref(self.cfg), window, C.byref(nbytes)), "pf_sample_workspace_bytes")
        # allocations belong to the stream the kernels run on: the caching allocator then never
        # hands a block still in use by a side-stream sampler launch to another stream
        with torch.cuda.stream(st):
            if out is None:
                out = torch.empty((n, 64), dtype=torch.uint8, device="cuda")
            if self._ws is None or self._ws.numel() < nbytes.value:
                self._ws = torch.empty((nbytes.value,), dtype=torch.uint8, device="cuda")
                self._ws_stream = st
        if st != self._ws_stream:  # used off its allocation stream: keep it alive past this launch
            self._ws.record_stream(st)
        N.check(
            N.lib().pf_sample(C.byref(self.cfg), self.slides_dev.data_ptr(), self.descs_dev.data_ptr(),
                              self.state.data_ptr(), n, out.data_ptr(), self._ws.data_ptr(), nbytes.value, window,
                              self.rounds, 1 if self.all_fit else 0, N.stream_ptr(stream)),
            "pf_sample",
        )
        if self._stats_event is None:  # the counters ride back to the host for the next window
            with torch.cuda.stream(st):
                self._stats_host.copy_(self.state[:C.sizeof(N.SamplerState)], non_blocking=True)
            self._stats_event = torch.cuda.Event()
            self._stats_event.record(st)
        return out

    def _poll_stats(self) -> None:
        if self._stats_event is None or not self._stats_event.query():
            return
        st = N.SamplerState.from_buffer_copy(self._stats_host.numpy().tobytes())
        self._stats_event = None
        if st.attempts >= 256 and st.seq > 0:
            self.p_est = max(0.02, min(1.0, st.seq / st.attempts))

    def state_host(self) -> N.SamplerState:
        return N.SamplerState.from_buffer_copy(self.state.cpu().numpy().tobytes())

    def check(self) -> N.SamplerState:
        st = self.state_host()
        if st.status != N.PF_OK:
            raise N.status_error(st.status, "no slide produced an admissible patch in "
                                 f"{st.consecutive_failures} consecutive slide draws")
        return st

    def update_estimate(self) -> None:
        st = self.state_host()
        if st.attempts > 0 and st.seq > 0:
            self.p_est = max(0.02, min(1.0, st.seq / st.attempts))

    def to_patch_specs(self, specs_dev) -> list:
        arr = specs_dev.cpu().numpy().view(N.SPEC_DTYPE).reshape(-1)
        return [PatchSpec(self.ids[r["slide"]], int(r["x"]), int(r["y"]), int(r["width"]), int(r["height"]),
                          float(r["target_mpp"]), int(r["out_size"]), int(r["seq"])) for r in arr]


def _desc_from_record(rec: SlideRecord) -> N.SlideDesc:
    d = N.SlideDesc()
    for i, lv in enumerate(rec.levels):
        d.mpp[i] = lv.mpp
        d.width[i] = lv.width
        d.height[i] = lv.height
        nx, ny = rec.tile_grid(i)
        d.tiles_x[i] = nx
        d.tiles_y[i] = ny
        d.downsample[i] = lv.downsample
    d.n_levels = len(rec.levels)
    d.tile_size = rec.tile_size
    d.base_mpp = rec.base_mpp
    return d


def epoch_stream(config: SamplerConfig, slides, batch: int = 4096):
    """Drop-in epoch_stream (pkg/sampler.py:196-227): exactly config.epoch_size PatchSpecs, GPU-sampled."""
    if not slides:
        raise NoSamplableSlideError("no slides provided")
    smp = GpuSampler(config, slides)
    left = config.epoch_size
    while left > 0:
        n = min(batch, left)
        dev = smp.next_batch(n)
        st = smp.state_host()
        yield from smp.to_patch_specs(dev[: st.emitted])
        if st.status != N.PF_OK:
            smp.check()
        smp.update_estimate()
        left -= n


class CappedSampler:
    """Device capped replay over a ``GpuSampler`` (capped_stream, pkg/sampler.py:255-281):
    the first ``cap`` specs come from the sampler and are kept in HBM; every later spec is a
    stored spec drawn with the (seed, "cache") stream on device (pf_capped_draw), so the
    sampler is no longer advanced.  ``next_batch`` returns [n, 64] device spec records, the
    same stream as the host ``capped_stream``."""

    def __init__(self, sampler: GpuSampler, cap: int, seed: int):
        torch = N.require_cuda()
        from . import rng

        if cap < 1:
            raise ValueError("cap must be >= 1")
        self.sampler, self.cap = sampler, int(cap)
        self.key = rng.stream_key(int(seed), "cache")
        self.stored = torch.empty((self.cap, 64), dtype=torch.uint8, device="cuda")
        self.n_stored = 0
        self.counter = torch.zeros(1, dtype=torch.int64, device="cuda")

    @property
    def full(self) -> bool:
        return self.n_stored >= self.cap

    def next_batch(self, n: int, out=None, stream=None):
        torch = N.require_cuda()
        st = stream if stream is not None else torch.cuda.current_stream()
        if out is None:
            with torch.cuda.stream(st):
                out = torch.empty((n, 64), dtype=torch.uint8, device="cuda")
        k = min(n, self.cap - self.n_stored)
        if k > 0:  # pass-through and retain: sampled straight into the retained range (no temporary)
            kept = self.stored[self.n_stored:self.n_stored + k]
            self.sampler.next_batch(k, out=kept, stream=st)
            with torch.cuda.stream(st):
                out[:k].copy_(kept)
            self.n_stored += k
        if n - k > 0:
            N.check(N.lib().pf_capped_draw(self.key, self.counter.data_ptr(), self.stored.data_ptr(), self.n_stored,
                                           n - k, out[k:].data_ptr(), N.stream_ptr(stream)), "pf_capped_draw")
        return out
