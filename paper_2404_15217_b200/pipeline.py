"""Loader, normalisation and the multi-crop training feed on the GPU.

Mirrors pkg/pipeline.py: ``LoaderConfig`` (43-56), ``run_loader`` (79-149),
``normalize_patch`` (152-155) and the KPB1 patch pack (158-205).  The thread
pool of the reference is replaced by batched device reads: ``run_loader``
keeps its contract (every spec exactly once, ordered by default, skip/raise
error policy, host (S, S, 3) uint8 arrays out) but assembles up to
``prefetch_depth`` patches per device call.  ``MultiCropLoader`` is the
training feed BASELINE config 2 measures: GPU sampler -> fused gather +
DINOv2 multi-crop -> bf16 NCHW batches that never leave HBM.
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as N
from .errors import LoaderError, PackFormatError
from .store import GpuSlide, SlideSet, plan_specs

IMAGENET_MEAN = (0.485, 0.456, 0.406)
IMAGENET_STD = (0.229, 0.224, 0.225)


@dataclass
class LoaderConfig:
    concurrency: int = 4
    prefetch_depth: int = 8
    ordered: bool = True
    on_error: str = "skip"

    def __post_init__(self):
        if self.concurrency < 1:
            raise ValueError("concurrency must be >= 1")
        if self.prefetch_depth < self.concurrency:
            raise ValueError("prefetch_depth must be >= concurrency")
        if self.on_error not in ("skip", "raise"):
            raise ValueError("on_error must be 'skip' or 'raise'")


@dataclass
class LoaderFailure:
    spec: object
    error: Exception


class LoaderRun:
    """Iterator over (spec, pixels); failures collect on ``.errors``."""

    def __init__(self, gen, errors: list):
        self._gen = gen
        self.errors = errors

    def __iter__(self):
        return self

    def __next__(self):
        return next(self._gen)


def run_loader(specs, slides, config: LoaderConfig | None = None, batch: int | None = None) -> LoaderRun:
    """Load every spec exactly once (pkg/pipeline.py:79-149) with batched GPU reads.

    ``slides``: a GpuSlide or mapping slide_id -> GpuSlide.  Specs are pulled from the
    iterable in chunks of ``batch`` (default max(prefetch_depth, 64)); a chunk is planned on the
    host, read in one device call per out_size, and emitted in input order.  Failures are
    handled at the failing spec's position, as the reference's ordered consumer does
    (pipeline.py:97-124): under "raise" every earlier spec is yielded before LoaderError, under
    "skip" the failure joins ``LoaderRun.errors`` when iteration reaches it.  ``ordered=False``
    may emit in any order (reference: completion order); this loader's completion order is the
    input order.  ``concurrency`` has no device meaning and is only validated.
    """
    config = config or LoaderConfig()
    if isinstance(slides, GpuSlide):
        slides = {slides.record.slide_id: slides}
    sset = SlideSet(list(slides.values()))
    errors: list = []
    bsz = batch or max(config.prefetch_depth, 64)

    def fail(spec, exc):
        if config.on_error == "raise":
            raise LoaderError(f"patch seq {spec.seq} failed: {exc}") from exc
        errors.append(LoaderFailure(spec, exc))

    def load_chunk(chunk):
        """[(pixels or None, exception or None)] in chunk order: one host plan of the chunk (the
        reference's read_region checks per spec), one device read per out_size."""
        res: list = [(None, None)] * len(chunk)
        pos, reqs = [], []
        for i, sp in enumerate(chunk):
            si = sset.index.get(sp.slide_id)
            if si is None:
                res[i] = (None, LoaderError(f"no open slide for id {sp.slide_id!r}"))
                continue
            pos.append(i)
            reqs.append((si, sp.rect(), sp.target_mpp, sp.out_size))
        errs: list = []
        plan = plan_specs(reqs, sset.records, errors=errs)
        bad = {}
        for j, exc in errs:
            bad[j] = exc
        for j, row in enumerate(plan):
            if j in bad:
                continue
            try:
                sset.slides[int(row["slide"])].require_resident(row)
            except Exception as exc:  # noqa: BLE001 - the error policy decides
                bad[j] = exc
        for j, exc in bad.items():
            res[pos[j]] = (None, exc)
        by_size: dict = {}
        for j in range(len(reqs)):
            if j not in bad:
                by_size.setdefault(reqs[j][3], []).append(j)
        for size, js in by_size.items():
            pix = sset.read_regions(plan[js], size).cpu().numpy()
            for k, j in enumerate(js):
                res[pos[j]] = (pix[k], None)
        return res

    def gen():
        it = iter(specs)
        while True:
            chunk = []
            for sp in it:
                chunk.append(sp)
                if len(chunk) >= bsz:
                    break
            if not chunk:
                return
            for sp, (pix, exc) in zip(chunk, load_chunk(chunk)):
                if exc is not None:
                    fail(sp, exc)
                    continue
                yield sp, pix

    return LoaderRun(gen(), errors)


def normalize_patch(pixels, mean=(0.5, 0.5, 0.5), std=(0.5, 0.5, 0.5), dtype: str = "f32"):
    """(v/255 - 0.5)/0.5 in FP32 on the GPU (pkg/pipeline.py:152-155); host arrays in -> host out."""
    torch = N.require_cuda()
    host = not isinstance(pixels, torch.Tensor)
    t = torch.from_numpy(np.ascontiguousarray(np.asarray(pixels, dtype=np.uint8))) if host else pixels
    t = t.to(device="cuda", dtype=torch.uint8).contiguous()
    if t.shape[-1] != 3:
        raise ValueError("pixels must be (..., 3) RGB")
    out = torch.empty(t.shape, dtype=torch.float32 if dtype == "f32" else torch.bfloat16, device="cuda")
    m = (C.c_float * 3)(*mean)
    s = (C.c_float * 3)(*std)
    N.check(N.lib().pf_normalize(t.data_ptr(), t.numel() // 3, N.PF_F32 if dtype == "f32" else N.PF_BF16,
                                 C.cast(m, C.c_void_p), C.cast(s, C.c_void_p), out.data_ptr(), N.stream_ptr()),
            "pf_normalize")
    return out.cpu().numpy() if host else out


# ---------------------------------------------------------------------------
# KPB1 patch pack (pkg/pipeline.py:158-205): format-compatible host I/O.
PACK_MAGIC = b"KPB1"
_PACK_HEADER = struct.Struct("<4sIIIB3x")
_DTYPE_TAGS = {np.dtype(np.uint8): 0, np.dtype(np.float32): 1}
_TAG_DTYPES = {0: np.dtype(np.uint8), 1: np.dtype(np.float32)}


def write_patch_pack(patches, path, specs=None) -> Path:
    arr = patches.cpu().numpy() if hasattr(patches, "cpu") else np.asarray(patches)
    if arr.ndim != 4 or arr.shape[3] != 3 or arr.shape[1] != arr.shape[2]:
        raise PackFormatError(f"patches must be (count, size, size, 3), got {arr.shape}")
    tag = _DTYPE_TAGS.get(arr.dtype)
    if tag is None:
        raise PackFormatError(f"unsupported dtype {arr.dtype}; use uint8 or float32")
    path = Path(path)
    with open(path, "wb") as fh:
        fh.write(_PACK_HEADER.pack(PACK_MAGIC, arr.shape[0], arr.shape[1], 3, tag))
        fh.write(np.ascontiguousarray(arr).astype(arr.dtype.newbyteorder("<")).tobytes())
    if specs is not None:
        with open(path.with_name(path.name + ".manifest.jsonl"), "w", encoding="utf-8") as fh:
            for sp in specs:
                fh.write(sp.to_json_line() + "\n")
    return path


def read_patch_pack(path) -> np.ndarray:
    data = Path(path).read_bytes()
    if len(data) < _PACK_HEADER.size:
        raise PackFormatError("file too short for a pack header")
    magic, count, size, ch, tag = _PACK_HEADER.unpack_from(data)
    if magic != PACK_MAGIC:
        raise PackFormatError(f"bad magic {magic!r}")
    if ch != 3:
        raise PackFormatError(f"channels must be 3, header says {ch}")
    dt = _TAG_DTYPES.get(tag)
    if dt is None:
        raise PackFormatError(f"unknown dtype tag {tag}")
    payload = data[_PACK_HEADER.size:]
    if len(payload) != count * size * size * 3 * dt.itemsize:
        raise PackFormatError(f"payload is {len(payload)} bytes, header implies {count * size * size * 3 * dt.itemsize}")
    return np.frombuffer(payload, dtype=dt.newbyteorder("<")).reshape(count, size, size, 3).astype(dt)


class RegionLoader:
    """Sampler -> read_region -> normalise, on device (BASELINE config 1, no augmentation).

    ``slides``: list of (GpuSlide, ForegroundPolygon).  Each ``next_batch`` returns a
    [batch, 3, S, S] tensor of (v/255 - mean)/std (``dtype`` f32/bf16) or raw uint8, for the
    next ``batch`` specs of the reference epoch_stream.  With ``prefetch`` the sampler runs on a
    side stream, ``chunk`` batches per call (the stream does not depend on how it is split), one
    chunk ahead of the reads: small batches amortise the sampler's fixed launch latency.
    """

    def __init__(self, slides, sampler_config, *, batch_size: int = 256, dtype: str = "f32", layout: str = "nchw",
                 mean=IMAGENET_MEAN, std=IMAGENET_STD, prefetch: bool = True, window=None, rounds: int = 1,
                 chunk: int | None = None):
        torch = N.require_cuda()
        from .sampler import GpuSampler

        self.slide_set = SlideSet([s for s, _ in slides])
        self.sampler = GpuSampler(sampler_config, slides, slide_set=self.slide_set, window=window, rounds=rounds)
        self.batch_size = batch_size
        self.out_size = sampler_config.patch_size
        self.dtype, self.layout, self.mean, self.std = dtype, layout, mean, std
        self.prefetch = prefetch
        self.chunk = max(1, chunk if chunk is not None else 8192 // max(1, batch_size)) if prefetch else 1
        rows = batch_size * self.chunk
        self.specs_slots = [torch.empty((rows, 64), dtype=torch.uint8, device="cuda") for _ in range(2)]
        self._side = torch.cuda.Stream(priority=-1)  # sampler prefetch ahead of the reads (see MultiCropLoader)
        self._ready = [None, None]
        self._free = [torch.cuda.Event(), torch.cuda.Event()]
        self._next = 0
        self._pos = 0  # batches of the current slot already served
        S = self.out_size
        tdt = {"u8": torch.uint8, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
        shape = (batch_size, 3, S, S) if layout == "nchw" else (batch_size, S, S, 3)
        self.out = torch.empty(shape, dtype=tdt, device="cuda")
        # every (slide, target mpp) reads its window unresampled: the lean passthrough kernel
        raw = self.sampler.slides_dev.cpu().numpy().tobytes()
        size = N.C.sizeof(N.SamplerSlide)
        table = [N.SamplerSlide.from_buffer_copy(raw[i * size:(i + 1) * size]) for i in range(len(raw) // size)]
        self.passthrough_only = all(int(t.side[k]) == S for t in table for k in range(len(sampler_config.target_mpps)))

    def next_batch(self, stream=None, marks: list | None = None):
        torch = N.require_cuda()
        st = stream or torch.cuda.current_stream()

        def mark(name):
            if marks is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(st)
                marks.append((name, ev))

        n = self.batch_size
        mark("begin")
        if not self.prefetch:
            cur, pos = 0, 0
            self.sampler.next_batch(n, out=self.specs_slots[0], stream=st)
            mark("sample")
        else:
            cur, pos = self._next, self._pos
            rows = n * self.chunk
            if self._ready[cur] is None:
                self._side.wait_stream(st)
                self.sampler.next_batch(rows, out=self.specs_slots[cur], stream=self._side)
                self._ready[cur] = torch.cuda.Event()
                self._ready[cur].record(self._side)
            st.wait_event(self._ready[cur])
            mark("sample_wait")
            if pos == 0:  # starting this slot: sample the next chunk into the other one
                nxt = 1 - cur
                self._side.wait_event(self._free[nxt])
                self.sampler.next_batch(rows, out=self.specs_slots[nxt], stream=self._side)
                self._ready[nxt] = torch.cuda.Event()
                self._ready[nxt].record(self._side)
        specs = self.specs_slots[cur][pos * n:(pos + 1) * n]
        self.slide_set.read_regions(specs, self.out_size, dtype=self.dtype, layout=self.layout,
                                    mean=self.mean, std=self.std, out=self.out, stream=st, planned=True,
                                    passthrough_only=self.passthrough_only)
        mark("read")
        if self.prefetch:
            self._pos = pos + 1
            if self._pos == self.chunk:  # slot consumed: free it for the chunk after next
                self._free[cur].record(st)
                self._next, self._pos = 1 - cur, 0
        return {"patches": self.out, "specs": specs}
