"""Per-rank sharding of the online-patching feed.

Slides are independent units: rank r owns its own slide subset and runs the
reference sampler on seed + r (pkg/sampler.py:5-7); the
augmentation parameters use Philox keyed by (seed, r) with counter (step, …).
Nothing on the data path crosses ranks, so there is no collective; the only
distributed calls are a start barrier and the max-over-ranks timing.
"""

from __future__ import annotations

from dataclasses import dataclass

from .rng import shard_seed


@dataclass(frozen=True)
class RankPlan:
    rank: int
    world: int
    slide_indices: tuple  # global slide indices owned by this rank
    sampler_seed: int
    philox_seed: int
    philox_rank: int


def rank_plan(rank: int, world: int, n_slides_total: int, seed: int = 0) -> RankPlan:
    """Contiguous slide blocks per rank (BASELINE config 4: 128 slides, 16 per GPU)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    per = n_slides_total // world
    extra = n_slides_total % world
    start = rank * per + min(rank, extra)
    count = per + (1 if rank < extra else 0)
    return RankPlan(rank, world, tuple(range(start, start + count)), shard_seed(seed, rank), seed, rank)
