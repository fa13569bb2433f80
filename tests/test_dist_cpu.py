"""Multi-rank sharding on CPU (gloo, world_size 2): each rank's stream equals a single-process run
with seed + rank, ranks own disjoint slide blocks, and the only collectives are control-plane."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _slides(goldens):
    out = []
    for i in range(3):
        w, h = goldens[f"sampler_dims_b{i}"]
        out.append({"id": f"b{i}", "width": w, "height": h, "base_mpp": 0.25,
                    "rings": [np.asarray(r) for r in goldens[f"sampler_poly_b{i}"]["rings"]]})
    return out


def _worker(rank, world, port, goldens, q):
    import torch.distributed as dist

    from oracle import port as P
    from paper_2404_15217_b200.shard import rank_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = rank_plan(rank, world, 3, seed=7)
    slides = [_slides(goldens)[i] for i in plan.slide_indices]
    specs, _ = P.epoch_stream(slides, patch_size=32, seed=plan.sampler_seed, epoch_size=8)
    t = torch.tensor([len(specs)], dtype=torch.int64)
    dist.all_reduce(t)  # control plane only: total count
    gathered = [None] * world
    dist.all_gather_object(gathered, (plan.slide_indices, plan.sampler_seed, specs))
    dist.barrier()
    if rank == 0:
        q.put((int(t.item()), gathered))
    dist.destroy_process_group()


def test_two_rank_sharding(goldens):
    import torch.multiprocessing as mp

    from oracle import port as P
    from paper_2404_15217_b200.shard import rank_plan

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, goldens, q)) for r in range(2)]
    for p in procs:
        p.start()
    total, gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert total == 16
    (s0, seed0, specs0), (s1, seed1, specs1) = gathered
    assert set(s0).isdisjoint(s1) and sorted(s0 + s1) == [0, 1, 2]
    assert (seed0, seed1) == (7, 8)
    # each rank's stream is exactly the single-process stream with seed + rank
    all_slides = _slides(goldens)
    for idx, seed, specs in gathered:
        want, _ = P.epoch_stream([all_slides[i] for i in idx], patch_size=32, seed=seed, epoch_size=8)
        assert specs == want
    assert rank_plan(1, 8, 128).slide_indices == tuple(range(16, 32))
