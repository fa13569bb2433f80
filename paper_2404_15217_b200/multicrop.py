"""DINOv2 multi-crop training feed on the GPU (BASELINE.json configs 2-5).

The reference stops at ``read_region`` + ``normalize_patch`` (SURVEY.md §0.1
D5); BASELINE config 2 asks for the DINOv2 multi-crop on every sampled patch:
2 global 224^2 crops (RandomResizedCrop scale (0.32, 1)) and 8 local 96^2
crops (scale (0.05, 0.32)), hflip p=0.5, ColorJitter(0.4, 0.4, 0.2, 0.1)
p=0.8, grayscale p=0.2, gaussian blur sigma U(0.1, 2) with p = 1.0 / 0.1 /
0.5, solarize p=0.2 on the second global crop, ImageNet normalisation, bf16.

Per-crop parameters come from Philox4x32-10 keyed by (seed, rank) with
counter (step, patch, crop) (pf_crop_params) and are explicit records, so the
torchvision oracle can replay them.  ``MultiCropLoader`` chains the device
sampler, the PIL resample for patches read off-level (mixed mpp, config 3),
the parameter generator and the fused kernel on one CUDA stream.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .pipeline import IMAGENET_MEAN, IMAGENET_STD


@dataclass
class MultiCropConfig:
    n_global: int = 2
    n_local: int = 8
    global_size: int = 224
    local_size: int = 96
    src_size: int = 224
    global_scale: tuple = (0.32, 1.0)
    local_scale: tuple = (0.05, 0.32)
    ratio: tuple = (3.0 / 4.0, 4.0 / 3.0)
    p_flip: float = 0.5
    p_jitter: float = 0.8
    p_gray: float = 0.2
    brightness: float = 0.4
    contrast: float = 0.4
    saturation: float = 0.2
    hue: float = 0.1
    sigma: tuple = (0.1, 2.0)
    p_blur: list = field(default_factory=lambda: [1.0, 0.1] + [0.5] * 8)
    p_solarize: list = field(default_factory=lambda: [0.0, 0.2] + [0.0] * 8)
    solarize_threshold: float = 128.0
    blur_kernel: int = 9

    def __post_init__(self):
        n = self.n_global + self.n_local
        if n < 1 or n > N.PF_MAX_CROPS:
            raise ValueError(f"1..{N.PF_MAX_CROPS} crops per patch")
        if len(self.p_blur) != n or len(self.p_solarize) != n:
            self.p_blur = (list(self.p_blur) + [0.5] * n)[:n]
            self.p_solarize = (list(self.p_solarize) + [0.0] * n)[:n]
        if self.blur_kernel != 9:
            raise ValueError("blur kernel is fixed at 9 (DINOv2)")
        if self.global_size % 8 or self.local_size % 8:
            raise ValueError("crop sizes must be multiples of 8")

    @property
    def n_crops(self) -> int:
        return self.n_global + self.n_local

    def to_c(self, with_tables: bool = True) -> N.MultiCropConfig:
        c = N.MultiCropConfig()
        if with_tables:
            c.rrc_table_global = rrc_table(self.src_size, self.global_size)
            c.rrc_table_local = rrc_table(self.src_size, self.local_size)
        c.n_global, c.n_local = self.n_global, self.n_local
        c.global_size, c.local_size, c.src_size = self.global_size, self.local_size, self.src_size
        c.blur_kernel = self.blur_kernel
        c.global_scale[:] = list(self.global_scale)
        c.local_scale[:] = list(self.local_scale)
        c.ratio[:] = list(self.ratio)
        c.p_flip, c.p_jitter, c.p_gray = self.p_flip, self.p_jitter, self.p_gray
        c.brightness, c.contrast, c.saturation, c.hue = self.brightness, self.contrast, self.saturation, self.hue
        c.sigma_min, c.sigma_max = self.sigma
        c.solarize_threshold = self.solarize_threshold
        for i in range(self.n_crops):
            c.p_blur[i] = self.p_blur[i]
            c.p_solarize[i] = self.p_solarize[i]
        return c

    def bytes_per_patch(self, dtype: str = "bf16") -> int:
        """Algorithmic HBM bytes per patch: u8 source read once + every crop written once."""
        el = {"bf16": 2, "f32": 4, "u8": 1}[dtype]
        out = 3 * el * (self.n_global * self.global_size**2 + self.n_local * self.local_size**2)
        return 3 * self.src_size**2 + out


_RRC_TABLES: dict = {}


def rrc_table(src_size: int, out_size: int) -> int:
    """Device address of the RandomResizedCrop tap table for (src_size -> out_size), built once
    per process (pf_rrc_table_build) and kept alive here."""
    torch = N.require_cuda()
    key = (torch.cuda.current_device(), src_size, out_size)  # the table lives on the current device
    t = _RRC_TABLES.get(key)
    if t is None:
        nbytes = C.c_int64(0)
        N.check(N.lib().pf_rrc_table_bytes(src_size, out_size, C.byref(nbytes)), "pf_rrc_table_bytes")
        t = torch.empty((nbytes.value,), dtype=torch.uint8, device="cuda")
        N.check(N.lib().pf_rrc_table_build(src_size, out_size, t.data_ptr(), N.stream_ptr()), "pf_rrc_table_build")
        _RRC_TABLES[key] = t
    return int(t.data_ptr())


def crop_params(cfg: MultiCropConfig, n_patches: int, seed: int, rank: int = 0, step: int = 0, out=None, stream=None):
    """[n_patches, n_crops, 64] uint8 device tensor of pf_crop_param records."""
    torch = N.require_cuda()
    if out is None:
        out = torch.empty((n_patches, cfg.n_crops, 64), dtype=torch.uint8, device="cuda")
    ccfg = cfg.to_c(with_tables=False)
    N.check(N.lib().pf_crop_params(seed & ((1 << 64) - 1), rank, step, n_patches, C.byref(ccfg), out.data_ptr(),
                                   N.stream_ptr(stream)), "pf_crop_params")
    return out


def params_host(params_dev) -> np.ndarray:
    return params_dev.cpu().numpy().reshape(-1, 64).view(N.CROP_DTYPE).reshape(params_dev.shape[:-1])


_DT = {"u8": N.PF_U8, "f32": N.PF_F32, "bf16": N.PF_BF16}


def multicrop(slide_set, specs_dev, params_dev, cfg: MultiCropConfig, *, dtype: str = "bf16", mean=IMAGENET_MEAN,
              std=IMAGENET_STD, src_hwc=None, out_global=None, out_local=None, stream=None):
    """Fused gather + multi-crop -> ([n_global, n, 3, G, G], [n_local, n, 3, L, L]) device tensors."""
    torch = N.require_cuda()
    n = int(specs_dev.shape[0])
    tdt = {"u8": torch.uint8, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
    if out_global is None:
        out_global = torch.empty((cfg.n_global, n, 3, cfg.global_size, cfg.global_size), dtype=tdt, device="cuda")
    if out_local is None:
        out_local = torch.empty((cfg.n_local, n, 3, cfg.local_size, cfg.local_size), dtype=tdt, device="cuda")
    ccfg = cfg.to_c()
    m = (C.c_float * 3)(*mean)
    s = (C.c_float * 3)(*std)
    N.check(
        N.lib().pf_multicrop(slide_set.descs.data_ptr(), specs_dev.data_ptr(),
                             src_hwc.data_ptr() if src_hwc is not None else None, n, params_dev.data_ptr(),
                             C.byref(ccfg), _DT[dtype], C.cast(m, C.c_void_p), C.cast(s, C.c_void_p),
                             out_global.data_ptr() if cfg.n_global else None,
                             out_local.data_ptr() if cfg.n_local else None, N.stream_ptr(stream)),
        "pf_multicrop",
    )
    return out_global, out_local


class MultiCropLoader:
    """Online patching training feed: sampler -> (resample) -> params -> fused multi-crop.

    The sampler (and the resample of mixed-mpp sources) of step k+1 runs on a side stream
    while step k's multi-crop runs.

    ``slides``: list of (GpuSlide, ForegroundPolygon).  Each ``next_batch``
    enqueues the whole step on the current stream and returns device tensors;
    per-rank streams follow the reference's seed + rank sharding for the
    coordinates and Philox(seed, rank, step) for the augmentation.
    """

    def __init__(self, slides, sampler_config, mc_config: MultiCropConfig | None = None, *, batch_size: int = 1024,
                 rank: int = 0, dtype: str = "bf16", mean=IMAGENET_MEAN, std=IMAGENET_STD, window=None, rounds: int = 1,
                 prefetch: bool = True, cap: int | None = None, aug_seed: int | None = None):
        torch = N.require_cuda()
        from .sampler import CappedSampler, GpuSampler
        from .store import SlideSet

        self.mc = mc_config or MultiCropConfig()
        if sampler_config.patch_size != self.mc.src_size:
            raise ValueError("sampler patch_size must equal the multi-crop source size")
        self.slide_set = SlideSet([s for s, _ in slides])
        self.sampler = GpuSampler(sampler_config, slides, slide_set=self.slide_set, window=window, rounds=rounds)
        # cap: capped replay of the first `cap` specs (capped_stream, pkg/sampler.py:255-281)
        self.specs_from = self.sampler if cap is None else CappedSampler(self.sampler, cap, sampler_config.seed)
        self.batch_size = batch_size
        self.rank = rank
        # Philox(seed, rank, step) for the crop parameters: the run's base seed (default: the
        # sampler's, which under sharding is already seed + rank)
        self.seed = sampler_config.seed if aug_seed is None else int(aug_seed)
        self.dtype = dtype
        self.mean, self.std = mean, std
        self.step = 0
        sides = {int(t.side[k]) for t in _table(self.sampler) for k in range(len(sampler_config.target_mpps))}
        self.needs_resample = any(sd != self.mc.src_size for sd in sides)
        S = self.mc.src_size
        self.specs_slots = [torch.empty((batch_size, 64), dtype=torch.uint8, device="cuda") for _ in range(2)]
        self.prefetch = prefetch
        # high priority: the next step's sampler blocks are scheduled ahead of this step's
        # multi-crop blocks as SMs free up, so the prefetch finishes inside the step
        self._side = torch.cuda.Stream(priority=-1)
        self._ready = [None, None]
        self._free = [torch.cuda.Event(), torch.cuda.Event()]
        self._next_slot = 0
        # crop parameters depend on (seed, rank, step) only, so each slot's are computed with its
        # specs (on the side stream under prefetch) instead of between two steps on the main stream
        self.params_slots = [torch.empty((batch_size, self.mc.n_crops, 64), dtype=torch.uint8, device="cuda")
                             for _ in range(2)]
        self.params = self.params_slots[0]
        # resampled sources, one per slot: the next step's PIL resample runs on the side stream
        # right after its sampler, under this step's multi-crop (memory-bound beside issue-bound)
        self.src_slots = ([torch.empty((batch_size, S, S, 3), dtype=torch.uint8, device="cuda") for _ in range(2)]
                          if self.needs_resample else [None, None])
        self.src = self.src_slots[0]
        self._res_ev = [None, None]  # (start, end) events of each slot's resample
        tdt = {"u8": torch.uint8, "f32": torch.float32, "bf16": torch.bfloat16}[dtype]
        self.out_global = torch.empty((self.mc.n_global, batch_size, 3, self.mc.global_size, self.mc.global_size),
                                      dtype=tdt, device="cuda")
        self.out_local = torch.empty((self.mc.n_local, batch_size, 3, self.mc.local_size, self.mc.local_size),
                                     dtype=tdt, device="cuda")
        # host-backed tile tiers (tier.py): each sampled batch's tiles are made resident on the
        # sampler's stream right after sampling, a batch ahead of its crops
        from .tier import TierSet

        ts = TierSet(self.slide_set)
        self.tiers = ts if ts.active else None

    def _sample(self, slot: int, st, step: int) -> None:
        """Specs of a slot, their tiles made resident (tiered slides), when some mpp needs it
        their resampled S x S sources, and the crop parameters of ``step`` -- all on stream ``st``."""
        torch = N.require_cuda()
        self.specs_from.next_batch(self.batch_size, out=self.specs_slots[slot], stream=st)
        crop_params(self.mc, self.batch_size, self.seed, self.rank, step, out=self.params_slots[slot], stream=st)
        if self.tiers is not None:
            self.tiers.prefetch(self.specs_slots[slot], self.batch_size, stream=st)
        if self.needs_resample:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            m = (C.c_float * 3)(0.5, 0.5, 0.5)
            N.check(N.lib().pf_read_regions(self.slide_set.descs.data_ptr(), self.specs_slots[slot].data_ptr(),
                                            self.batch_size, self.mc.src_size, N.PF_U8,
                                            N.PF_HWC | N.PF_SKIP_PASSTHROUGH, C.cast(m, C.c_void_p),
                                            C.cast(m, C.c_void_p), self.src_slots[slot].data_ptr(),
                                            N.stream_ptr(st)), "pf_read_regions")
            e1.record(st)
            self._res_ev[slot] = (e0, e1)

    def next_batch(self, stream=None, marks: list | None = None) -> dict:
        """Enqueue one step and return its device tensors.

        With ``prefetch`` (default) the specs of step k+1 are sampled on a side stream while
        step k's crops are computed: the sampler's serial walk overlaps the previous batch's
        multi-crop instead of idling the GPU in front of it.  ``marks`` (optional list) receives
        (stage, cuda.Event) pairs recorded on the main stream after each stage."""
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
            self._sample(0, st, self.step)
            cur = 0
            mark("sample")
        else:
            cur = self._next_slot
            if self._ready[cur] is None:  # first step: nothing prefetched yet
                self._side.wait_stream(st)
                self._sample(cur, self._side, self.step)
                self._ready[cur] = torch.cuda.Event()
                self._ready[cur].record(self._side)
            st.wait_event(self._ready[cur])
            if self.tiers is not None and self.tiers.stale():
                # a tier pool was resized after this batch was prefetched: make its tiles resident
                # in the new pool
                self.tiers.prefetch(self.specs_slots[cur], n, stream=st)
            mark("sample_wait")
        specs = self.specs_slots[cur]
        src = self.src_slots[cur]
        res_ev = self._res_ev[cur]
        self.params = self.params_slots[cur]  # computed with this slot's specs
        mark("params")
        if self.prefetch:
            nxt = 1 - cur
            self._side.wait_event(self._free[nxt])  # step k-1 finished reading that slot
            self._sample(nxt, self._side, self.step + 1)
            self._ready[nxt] = torch.cuda.Event()
            self._ready[nxt].record(self._side)
            self._next_slot = nxt
        multicrop(self.slide_set, specs, self.params, self.mc, dtype=self.dtype, mean=self.mean, std=self.std,
                  src_hwc=src, out_global=self.out_global, out_local=self.out_local, stream=st)
        mark("multicrop")
        if self.prefetch:
            self._free[cur].record(st)
        self.step += 1
        return {"global_crops": self.out_global, "local_crops": self.out_local, "specs": specs,
                "params": self.params, "resample_events": res_ev}

    def check(self) -> None:
        """Synchronise and raise on a failed stream: NoSamplableSlideError from the sampler state,
        OutOfBoundsError if a crop read a tile outside a compacted slide's resident set."""
        torch = N.require_cuda()
        self.drain()
        torch.cuda.current_stream().synchronize()
        self.sampler.check()
        self.slide_set.check_status()

    def drain(self) -> None:
        """Wait for the prefetched sampler work (so the sampler state is final)."""
        torch = N.require_cuda()
        torch.cuda.current_stream().wait_stream(self._side)



def _table(sampler):
    raw = sampler.slides_dev.cpu().numpy().tobytes()
    size = C.sizeof(N.SamplerSlide)
    return [N.SamplerSlide.from_buffer_copy(raw[i * size:(i + 1) * size]) for i in range(len(raw) // size)]
