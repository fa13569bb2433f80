"""Host helpers for the counter-based SplitMix64 streams of pkg/rng.py.

The device sampler owns the draws (csrc/pf_common.cuh ``stream_u64``); the host
only derives per-purpose stream keys (pkg/rng.py:49), applies the seed + rank
shard rule (pkg/sampler.py:5-7) and offers a few vectorised draws for
host-side bookkeeping.  Constants are fixed by the reference (rng.py:13-21).
"""

from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
MUL1 = 0xBF58476D1CE4E5B9
MUL2 = 0x94D049BB133111EB
FNV_OFFSET = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3

PURPOSES = ("slide", "coords", "mpp", "cache")  # StreamSet, pkg/sampler.py:106-122


def mix64(x: int) -> int:
    x &= M64
    x = ((x ^ (x >> 30)) * MUL1) & M64
    x = ((x ^ (x >> 27)) * MUL2) & M64
    return x ^ (x >> 31)


def fnv1a(data: bytes) -> int:
    h = FNV_OFFSET
    for byte in data:
        h = ((h ^ byte) * FNV_PRIME) & M64
    return h


def stream_key(seed: int, purpose: str) -> int:
    return mix64((seed & M64) ^ fnv1a(purpose.encode("utf-8")))


def shard_seed(seed: int, rank: int) -> int:
    """Worker / rank r streams use seed + r (pkg/sampler.py:5-7)."""
    return seed + rank


def draws(key: int, first: int, count: int) -> np.ndarray:
    """u64 draws with counters first .. first+count-1 (1-based), vectorised."""
    c = np.arange(first, first + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = np.uint64(key) + c * np.uint64(GAMMA)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(MUL1)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(MUL2)
        return x ^ (x >> np.uint64(31))


class Stream:
    """Minimal stateful view used by host bookkeeping (capped replay draws)."""

    __slots__ = ("key", "counter")

    def __init__(self, seed: int, purpose: str):
        self.key = stream_key(seed, purpose)
        self.counter = 0

    def u64(self) -> int:
        self.counter += 1
        return mix64((self.key + self.counter * GAMMA) & M64)

    def below(self, n: int) -> int:
        """Unbiased integer in [0, n) by rejection (same rule as pkg/rng.py:69-77)."""
        if n < 1:
            raise ValueError("randrange() requires n >= 1")
        bound = (1 << 64) - ((1 << 64) % n)
        v = self.u64()
        while v >= bound:
            v = self.u64()
        return v % n
