"""Host-backed tile tier: slide sets whose reachable tiles exceed HBM.

The reference keeps a 64 MiB LRU of decoded tiles and fetches a chunk on a miss
(``TileCache`` + ``Slide.fetch_chunk``, pkg/store.py:270-319, 611-649).  Here a level is
compacted (``GpuSlide.compact``) to an HBM slot pool smaller than its reachable tile set
(residency.reachable_tiles), and every reachable tile lives in a pinned host store mapped into
the device address space.  Because the sampler runs a batch ahead, ``TierSet.prefetch`` makes
the next batch's tiles resident before its crops are cut -- mark hits, take victim slots by a
clock hand, copy the misses from host memory by zero-copy device reads, update ``tile_map`` --
all on the sampler's stream with no host round trip (csrc/pf_tier.cu).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


class TileTier(C.Structure):
    _fields_ = [
        ("host_tiles", C.c_uint64),
        ("host_index", C.c_uint64),
        ("slot_owner", C.c_uint64),
        ("slot_last_use", C.c_uint64),
        ("requested", C.c_uint64),
        ("miss_list", C.c_uint64),
        ("victims", C.c_uint64),
        ("counters", C.c_uint64),
        ("level", C.c_int32),
        ("n_slots", C.c_int32),
        ("max_miss", C.c_int32),
        ("_pad", C.c_int32),
    ]


assert C.sizeof(TileTier) == 8 * 8 + 16


class HostStore:
    """Pinned, device-mapped host memory (pf_host_alloc_mapped), freed with the object."""

    def __init__(self, nbytes: int):
        self.nbytes = int(nbytes)
        self.host, self.dev = C.c_void_p(), C.c_void_p()
        N.check(N.lib().pf_host_alloc_mapped(self.nbytes, C.byref(self.host), C.byref(self.dev)), "pf_host_alloc_mapped")

    def array(self) -> np.ndarray:
        return np.ctypeslib.as_array(C.cast(self.host, C.POINTER(C.c_uint8)), shape=(self.nbytes,))

    def __del__(self):
        if getattr(self, "host", None) is not None and self.host.value:
            N.lib().pf_host_free(self.host)
            self.host = C.c_void_p()


def tier_level(slide, level: int, keep: np.ndarray, hbm_slots: int, max_miss: int = 8192, chunk: int = 2048):
    """Move level ``level`` of a dense GpuSlide to a host-backed tier.

    keep: bool [tiles_y, tiles_x] of the tiles reads can reach (residency.reachable_tiles); they
    are copied to a pinned host store.  hbm_slots: HBM slots (tiles) kept resident -- the first
    ones of the plan are resident initially.  The dense level is freed.  Returns the slide's
    ``TileTierState`` (kept on the slide)."""
    import torch

    N.require_cuda()
    rec = slide.record
    T = rec.tile_size
    tb = T * T * 3
    nx, ny = rec.tile_grid(level)
    keep = np.asarray(keep, dtype=bool)
    if keep.shape != (ny, nx):
        raise ValueError(f"plan for level {level} must be ({ny}, {nx})")
    if slide.tile_maps[level] is not None:
        raise ValueError(f"level {level} is already compacted")
    idx = np.flatnonzero(keep.ravel())
    n_keep = len(idx)
    if n_keep == 0:
        raise ValueError("no reachable tiles")
    hbm_slots = int(max(1, min(hbm_slots, n_keep)))
    torch.cuda.synchronize()
    store = HostStore(n_keep * tb)
    host = store.array().reshape(n_keep, tb)
    src = slide.levels[level].view(ny * nx, tb)
    pinned = torch.empty((min(chunk, n_keep), tb), dtype=torch.uint8, pin_memory=True)
    for i in range(0, n_keep, chunk):  # D2H of the reachable tiles through a pinned bounce buffer
        sel = torch.from_numpy(idx[i:i + chunk]).cuda()
        k = len(sel)
        pinned[:k].copy_(src[sel])
        host[i:i + k] = pinned[:k].numpy()
    del src
    host_index = np.full(ny * nx, -1, dtype=np.int64)
    host_index[idx] = np.arange(n_keep, dtype=np.int64)
    slots = torch.empty((hbm_slots + 1, T, T, 3), dtype=torch.uint8, device="cuda")
    slots[0].zero_()
    first = torch.from_numpy(idx[:hbm_slots]).cuda()
    dense = slide.levels[level].view(ny * nx, T, T, 3)
    for i in range(0, hbm_slots, chunk):
        slots[1 + i:1 + i + len(first[i:i + chunk])] = dense[first[i:i + chunk]]
    del dense
    tile_map = np.zeros(ny * nx, dtype=np.int32)
    tile_map[idx[:hbm_slots]] = np.arange(1, hbm_slots + 1, dtype=np.int32)
    owner = np.full(hbm_slots + 1, -1, dtype=np.int32)
    owner[1:] = idx[:hbm_slots].astype(np.int32)
    st = TileTierState(store, host_index, owner, ny * nx, hbm_slots, level, max_miss)
    st.tile_ids = idx
    slide.levels[level] = slots
    slide.tile_maps[level] = torch.from_numpy(tile_map).cuda()
    slide.resident[level] = keep  # reads must stay on reachable tiles (host check in read_region)
    slide.tier = st
    slide.desc = slide._make_desc()
    slide._own_set = None
    for ss in list(slide._sets):
        ss._refresh(slide)
    torch.cuda.empty_cache()
    return st


def resize_pool(slide, n_slots: int, chunk: int = 2048) -> None:
    """Give a tiered level a pool of n_slots HBM slots, the first n_slots reachable tiles resident
    (copied from the host store); the old pool is freed first."""
    import torch

    st = slide.tier
    level, rec = st.level, slide.record
    T = rec.tile_size
    tb = T * T * 3
    idx = st.tile_ids
    n_slots = int(max(1, min(n_slots, len(idx))))
    torch.cuda.synchronize()
    slide.levels[level] = None
    torch.cuda.empty_cache()
    slots = torch.empty((n_slots + 1, tb), dtype=torch.uint8, device="cuda")
    slots[0].zero_()
    host = st.store.array().reshape(len(idx), tb)
    for i in range(0, n_slots, chunk):
        k = min(chunk, n_slots - i)
        slots[1 + i:1 + i + k].copy_(torch.from_numpy(host[i:i + k]))
    nx, ny = rec.tile_grid(level)
    tile_map = np.zeros(ny * nx, dtype=np.int32)
    tile_map[idx[:n_slots]] = np.arange(1, n_slots + 1, dtype=np.int32)
    owner = np.full(n_slots + 1, -1, dtype=np.int32)
    owner[1:] = idx[:n_slots].astype(np.int32)
    # in place: TierSets built earlier hold this state object and rebuild their device records
    # when its version changes
    st.reset_pool(owner, ny * nx, n_slots)
    slide.levels[level] = slots.view(n_slots + 1, T, T, 3)
    slide.tile_maps[level] = torch.from_numpy(tile_map).cuda()
    slide.desc = slide._make_desc()
    slide._own_set = None
    for ss in list(slide._sets):
        ss._refresh(slide)


class TileTierState:
    """Device arrays of one tiered level (pf_tile_tier)."""

    def __init__(self, store: HostStore, host_index, owner, n_tiles: int, n_slots: int, level: int, max_miss: int):
        import torch

        self.store = store
        self.host_index = torch.from_numpy(host_index).cuda()
        self.level, self.max_miss = level, max_miss
        self.miss_list = torch.zeros(max_miss, dtype=torch.int32, device="cuda")
        self.victims = torch.zeros(max_miss, dtype=torch.int32, device="cuda")
        self.counters = torch.zeros(8, dtype=torch.int32, device="cuda")
        self.batch = 1  # last batch id issued against this level (ids only grow, whoever prefetches)
        self.version = 0
        self.reset_pool(owner, n_tiles, n_slots)

    def reset_pool(self, owner, n_tiles: int, n_slots: int) -> None:
        """New slot pool bookkeeping (slot contents and the tile map are the caller's)."""
        import torch

        self.owner = torch.from_numpy(np.ascontiguousarray(owner, dtype=np.int32)).cuda()
        self.last_use = torch.zeros(n_slots + 1, dtype=torch.int32, device="cuda")
        self.requested = torch.zeros(n_tiles, dtype=torch.int32, device="cuda")
        self.counters[2] = 0  # clock hand
        self.n_slots = n_slots
        self.version += 1

    def record(self) -> TileTier:
        t = TileTier()
        t.host_tiles = int(self.store.dev.value)
        t.host_index = int(self.host_index.data_ptr())
        t.slot_owner = int(self.owner.data_ptr())
        t.slot_last_use = int(self.last_use.data_ptr())
        t.requested = int(self.requested.data_ptr())
        t.miss_list = int(self.miss_list.data_ptr())
        t.victims = int(self.victims.data_ptr())
        t.counters = int(self.counters.data_ptr())
        t.level, t.n_slots, t.max_miss = self.level, self.n_slots, self.max_miss
        return t

    def tiles_filled(self) -> int:
        return int(self.counters[4:6].cpu().numpy().view(np.uint64)[0])


class TierSet:
    """pf_tile_tier records for every slide of a SlideSet (zero records for untiered slides)."""

    def __init__(self, slide_set):
        import torch

        self.slide_set = slide_set
        self.states = [getattr(s, "tier", None) for s in slide_set.slides]
        self._versions = None
        self.dev = None
        self._upload()
        self.max_fill = max([s.max_miss for s in self.states if s is not None] or [1])

    def _upload(self) -> None:
        import torch

        recs = (TileTier * len(self.states))()
        for i, stt in enumerate(self.states):
            if stt is not None:
                recs[i] = stt.record()
        self.dev = torch.frombuffer(bytearray(bytes(recs)), dtype=torch.uint8).cuda()
        self._versions = [s.version if s is not None else -1 for s in self.states]

    @property
    def active(self) -> bool:
        return any(s is not None for s in self.states)

    def stale(self) -> bool:
        """A pool was resized since the last prefetch (its device records moved)."""
        return [s.version if s is not None else -1 for s in self.states] != self._versions

    def prefetch(self, specs_dev, n: int, stream=None, max_window: int = 512) -> int:
        """Make the tiles of these (planned) specs resident for the next batch; returns the batch id."""
        if self.stale():
            self._upload()  # a pool was resized since: device records point at the new arrays
        live = [s for s in self.states if s is not None]
        batch = 1 + max(s.batch for s in live)
        for s in live:
            s.batch = batch
        T = min(s.record.tile_size for s in self.slide_set.slides)
        per = (-(-max_window // T) + 1) ** 2
        N.check(N.lib().pf_tier_prefetch(self.slide_set.descs.data_ptr(), self.dev.data_ptr(), len(self.states),
                                         specs_dev.data_ptr(), n, batch, self.max_fill, per,
                                         N.stream_ptr(stream)), "pf_tier_prefetch")
        return batch

    def tiles_filled(self) -> int:
        return sum(s.tiles_filled() for s in self.states if s is not None)
