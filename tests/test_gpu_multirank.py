"""bench.py's multi-rank product path, run as 2 ranks on one GPU over gloo:
each rank's device spec stream equals a single-process GpuSampler on its own slide block with
seed + rank (pkg/sampler.py:5-7), and its crop parameters are Philox(seed, rank, step) with its
own rank in the key (so the two ranks' augmentations differ)."""

import argparse
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_on_one_gpu_match_single_process_streams(cuda, tmp_path):
    import paper_2404_15217_b200 as pf
    from paper_2404_15217_b200.multicrop import MultiCropConfig, crop_params

    args = ["--gpus", "2", "--config", "2", "--slides", "2", "--width", "6144", "--height", "4608", "--batch", "96",
            "--steps", "2", "--warmup", "1", "--no-e2e", "--no-cpu-baseline", "--dist-backend", "gloo",
            "--device", "0", "--dump-dir", str(tmp_path)]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "bench.py"), *args]
    res = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1200,
                         env={**os.environ, "PYTHONPATH": str(ROOT)})
    assert res.returncode == 0, res.stderr[-3000:]
    line = [l for l in res.stdout.splitlines() if l.startswith("{")][-1]
    assert '"n_gpus": 2' in line
    import bench  # noqa: E402  (the same slide builder the ranks ran)

    dumps = [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]
    assert set(dumps[0]["slide_indices"]).isdisjoint(set(dumps[1]["slide_indices"]))
    params = []
    for r, d in enumerate(dumps):
        assert int(d["sampler_seed"]) == r and int(d["rank"]) == r  # seed + rank, base seed 0
        ns = argparse.Namespace(config="2", slides=2, width=6144, height=4608)
        _, plan, slides = bench.build_slides(ns, r, 2)
        assert tuple(plan.slide_indices) == tuple(d["slide_indices"])
        cfg = pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=[(0.25, 1.0)], seed=plan.sampler_seed)
        smp = pf.GpuSampler(cfg, slides)
        want = smp.next_batch(96).cpu().numpy()
        assert np.array_equal(d["specs"], want), f"rank {r}: spec stream != single-process seed + rank"
        mc = MultiCropConfig()
        wp = crop_params(mc, 96, seed=plan.philox_seed, rank=r, step=0).cpu().numpy()
        assert np.array_equal(d["params"], wp), f"rank {r}: crop params != Philox(seed, {r}, 0)"
        params.append(d["params"])
        del slides, smp
    assert not np.array_equal(params[0], params[1])  # the rank is in the Philox key
