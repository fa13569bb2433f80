"""Benchmark: augmented patches/s of the Online Patching training feed on B200.

Workload (BASELINE.json configs[1], "C2"): 16 synthetic 40000x30000 uint8 RGB
slides per GPU resident in HBM (tile 256, factor-4 pyramid), saturation(0.07)
+ morphology tissue masks on the 1/32 thumbnail, traced polygons, the
reference's epoch_stream sampler (224 px, min foreground 0.40) and the DINOv2
multi-crop (2 x 224^2 + 8 x 96^2, bf16 NCHW, ImageNet normalisation), batch
1024 patches per GPU per step.  A step = sample 1024 specs + crop params +
fused gather/multi-crop, all on device.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun each rank owns its own 16 slides (seed + rank) and streams
(reference rule seed + rank; Philox(seed, rank, step)); no collective on the
data path (weak scaling).  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "augmented patches/sec (224² global+96² local multi-crop) and % HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="2", choices=["1", "2", "3", "4", "5"],
                    help="BASELINE config: 1 normalise-only, 2 multi-crop (default), 3 mixed mpp, "
                         "4 whole-box slide set (tile residency), 5 sweep")
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--slides", type=int, default=None)
    ap.add_argument("--width", type=int, default=None)
    ap.add_argument("--height", type=int, default=None)
    ap.add_argument("--mixed-mpp", action="store_true", help="same as --config 3")
    ap.add_argument("--dtype", default=None, choices=["bf16", "f32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2)
    # test hooks (tests/test_gpu_multirank.py): N ranks on one GPU over gloo, per-rank stream dump
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--device", type=int, default=None, help="CUDA device of every rank (default LOCAL_RANK)")
    ap.add_argument("--dump-dir", default=None, help="each rank writes its first batch's specs + crop params")
    ap.add_argument("--tier-hbm-gb", type=float, default=None,
                    help="config 4: level-0 tiles in a host-backed tier with this many GB of HBM slots per GPU "
                         "(slide sets whose reachable tiles exceed HBM, e.g. --slides 32)")
    args = ap.parse_args()
    if args.mixed_mpp:
        args.config = "3"
    base = CONFIGS[args.config]
    for k in ("batch", "slides", "width", "height", "dtype"):
        if getattr(args, k) is None:
            setattr(args, k, base[k])
    args.mixed_mpp = args.config == "3"
    return args


# BASELINE.json configs (per GPU)
CONFIGS = {
    "1": dict(batch=256, slides=1, width=8192, height=8192, dtype="f32"),
    "2": dict(batch=1024, slides=16, width=40000, height=30000, dtype="bf16"),
    "3": dict(batch=2048, slides=16, width=40000, height=30000, dtype="bf16"),
    # 128 slides, W ~ U[40000, 100000], H ~ U[30000, 80000] from a seed, 16 per GPU (sizes below unused)
    "4": dict(batch=1024, slides=16, width=0, height=0, dtype="bf16"),
    "5": dict(batch=1024, slides=1, width=100000, height=80000, dtype="bf16"),
}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:  # noqa: BLE001
            pass
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "5"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:  # wait for the first sample
                time.sleep(0.05)
            self.rows.clear()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# B200 arm


def build_slides(args, rank, world):
    """Render this rank's slides in HBM, threshold the BASELINE saturation mask on the 1/32
    thumbnail and trace each slide's foreground polygon."""
    import paper_2404_15217_b200 as pf
    from paper_2404_15217_b200.shard import rank_plan
    from paper_2404_15217_b200.synthetic import synthetic_slide

    plan = rank_plan(rank, world, args.slides * world, seed=0)  # rank r owns slides [16r, 16r+16)
    slides = []
    resident, dense = 0, 0
    tier_gb = getattr(args, "tier_hbm_gb", None)
    tiered = []  # (slide, level-0 reachable plan) to move to the host-backed tier once all are built
    if args.config == "4":  # 128 slide sizes from one seed; rank r renders slides [16r, 16r + 16)
        rs = np.random.default_rng(4)
        dims = list(zip(rs.integers(40000, 100001, 128), rs.integers(30000, 80001, 128)))
    for gi in plan.slide_indices:
        sid = f"s{gi}"
        w, h = (int(dims[gi % 128][0]), int(dims[gi % 128][1])) if args.config == "4" else (args.width, args.height)
        for k in range(8):
            s = synthetic_slide(sid, w, h, seed=1000 + gi + 100_000 * k, downsample_factor=4)
            thumb, scale = s.thumbnail_device(32)
            mask = pf.foreground.mask_device(thumb, 1, 0.07, 1)  # BASELINE: saturation > 0.07 + morphology
            bm = pf.BinaryMask(mask.cpu().numpy().astype(bool), scale)
            try:
                poly = pf.polygon_from_mask(bm, slide_id=sid)
                break
            except ValueError as e:
                # the reference's ring orientation (vertex-mean probe, pkg/foreground.py:206-216) can
                # leave a non-convex layout with negative total area; redraw that slide's tissue
                print(f"[rank {rank}] {sid}: {e}; redrawing tissue (seed +{100_000 * (k + 1)})", file=sys.stderr)
                del s
        slides.append((s, poly))
        if args.config == "4":  # keep only the tiles an admissible window can reach
            from paper_2404_15217_b200 import residency as R

            tiles = R.reachable_tiles(s.record, bm.bits, scale, R.max_footprint(s.record, 224, [(0.25, 1.0)]))
            dense += R.dense_bytes(s.record)
            resident += R.resident_bytes(s.record, tiles)
            print(f"[rank {rank}] {sid} {w}x{h}: mask {bm.bits.mean():.3f}, pyramid {R.dense_bytes(s.record) / 1e9:.1f} GB"
                  f" -> {R.resident_bytes(s.record, tiles) / 1e9:.1f} GB resident", file=sys.stderr)
            import torch

            if tier_gb:  # level 0 -> pinned host store now (HBM for the next render), slots sized later
                from paper_2404_15217_b200 import tier as TR

                n0 = int(tiles[0].sum())
                st = TR.tier_level(s, 0, tiles[0], hbm_slots=1)
                tiered.append((s, n0))
                s.compact(tiles, levels=range(1, len(tiles)))
            else:
                s.compact(tiles)
            torch.cuda.empty_cache()
    if tiered:  # HBM slot pools, split over the slides by reachable level-0 tiles
        from paper_2404_15217_b200 import tier as TR

        tb = 256 * 256 * 3
        total = sum(n for _, n in tiered)
        budget = int(tier_gb * 1e9 / tb)
        for s, n in tiered:
            TR.resize_pool(s, max(1, budget * n // total))
        args.tier = {"reachable_l0_gb": round(total * tb / 1e9, 1), "hbm_slots_gb": round(budget * tb / 1e9, 1),
                     "slides": len(tiered)}
    args.residency = {"dense_gb": round(dense / 1e9, 1), "resident_gb": round(resident / 1e9, 1)} if dense else None
    return pf, plan, slides


class Feed:
    """One benchmark workload: a loader plus what the roofline needs to know about it."""

    def __init__(self, loader, stage, bytes_per_patch: int, kernel: str, workload: str, e2e_fn):
        # stage: the timed stage(s) whose summed time is the roofline's per-step kernel time
        self.loader, self.stages, self.bytes_per_patch = loader, (stage,) if isinstance(stage, str) else tuple(stage), \
            bytes_per_patch
        self.kernel, self.workload, self.e2e_fn = kernel, workload, e2e_fn

    @property
    def sampler(self):
        return self.loader.sampler


def make_feed(args, pf, plan, slides, rank, src_size=224, n_local=8, patch=224):
    # speculation rounds per sampler call (the loaders' default, 1; PF_SAMPLER_ROUNDS for experiments)
    rounds = int(os.environ.get("PF_SAMPLER_ROUNDS", "1"))
    from paper_2404_15217_b200.multicrop import MultiCropConfig, MultiCropLoader
    from paper_2404_15217_b200.pipeline import RegionLoader

    if args.config == "1":
        scfg = pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=[(0.25, 1.0)], seed=plan.sampler_seed)
        chunk = int(os.environ["PF_REGION_CHUNK"]) if os.environ.get("PF_REGION_CHUNK") else None  # experiment knob
        loader = RegionLoader(slides, scfg, batch_size=args.batch, dtype=args.dtype, chunk=chunk)
        el = 4 if args.dtype == "f32" else 2
        bpp = 224 * 224 * 3 + 224 * 224 * 3 * el
        wl = (f"C1: {args.slides} slide {args.width}x{args.height} in HBM, sat>0.07+morph mask on 1/32 thumbnail, "
              f"epoch_stream sampler 224px min_fg 0.40, read_region + ImageNet normalise to {args.dtype} NCHW")
        return Feed(loader, "read", bpp, "passthrough_kernel (pf_read_regions with PF_SKIP_RESAMPLED)", wl, run_e2e_regions)
    mpps = [(0.25, 1.0), (0.5, 1.0), (1.0, 1.0), (2.0, 1.0)] if args.config == "3" else [(0.25, 1.0)]
    if args.config == "5":
        mpps = [(0.25 * patch / 224.0, 1.0)]
    scfg = pf.SamplerConfig(patch_size=224, min_foreground=0.40, target_mpps=mpps, seed=plan.sampler_seed)
    mc = MultiCropConfig(n_local=n_local)
    loader = MultiCropLoader(slides, scfg, mc, batch_size=args.batch, rank=rank, dtype=args.dtype, rounds=rounds,
                             aug_seed=plan.philox_seed)
    tag = {"2": "C2", "3": "C3 (mpp U{0.25,0.5,1,2})", "4": "C4", "5": f"C5 point (patch {patch}->224, L={n_local})"}[args.config]
    if args.config == "4":
        r = getattr(args, "residency", None) or {}
        wl = (f"C4: 16 slides per GPU of W~U[40000,100000] x H~U[30000,80000] (128-slide set, seed 4), pyramids "
              f"{r.get('dense_gb')} GB dense -> {r.get('resident_gb')} GB HBM-resident (tiles reachable from the "
              f"foreground mask), sat>0.07+morph mask on 1/32 thumbnail, epoch_stream sampler 224px min_fg 0.40, "
              f"Philox(seed, rank, step) crops, DINOv2 multi-crop 2x224 + {n_local}x96 {args.dtype} NCHW")
    else:
        wl = (f"{tag}: {args.slides} slides {args.width}x{args.height} per GPU in HBM, sat>0.07+morph mask on 1/32 "
              f"thumbnail, epoch_stream sampler 224px min_fg 0.40, DINOv2 multi-crop 2x224 + {n_local}x96 {args.dtype} NCHW")
    if args.config == "3":  # E[source] over mpp U{0.25, 0.5, 1, 2}: 224^2, 448^2 (L0), 224^2, 448^2 (L1) u8
        src = (224 * 224 + 448 * 448 + 224 * 224 + 448 * 448) * 3 // 4
        bpp = mc.bytes_per_patch(args.dtype) - 3 * mc.src_size ** 2 + src
        return Feed(loader, ("resample", "multicrop"), bpp,
                    "read_regions_kernel (PIL 448->224, half the patches) + multicrop_kernel (both launches)", wl,
                    run_e2e_multicrop)
    return Feed(loader, "multicrop", mc.bytes_per_patch(args.dtype), "multicrop_kernel (global + local crop launches)",
                wl, run_e2e_multicrop)


def run_e2e_multicrop(pf, loader, steps, torch):
    """Reference-facing path with HOST buffers: pinned host specs -> H2D -> crop params -> fused
    multi-crop -> D2H of the whole batch into pinned host memory, double-buffered on two streams."""
    from paper_2404_15217_b200.multicrop import crop_params, multicrop

    mc = loader.mc
    n = loader.batch_size
    loader.drain()
    # a manifest of specs, as a host caller would hold it (run_loader / `patchforge load` input)
    host_specs = [loader.sampler.next_batch(n).cpu().pin_memory() for _ in range(2)]
    tdt = loader.out_global.dtype
    G, Lc = mc.n_global, mc.n_local
    bufs = []
    for _ in range(2):
        bufs.append({
            "specs": torch.empty((n, 64), dtype=torch.uint8, device="cuda"),
            "params": torch.empty((n, mc.n_crops, 64), dtype=torch.uint8, device="cuda"),
            "g": torch.empty((G, n, 3, mc.global_size, mc.global_size), dtype=tdt, device="cuda"),
            "l": torch.empty((Lc, n, 3, mc.local_size, mc.local_size), dtype=tdt, device="cuda"),
            "hg": torch.empty((G, n, 3, mc.global_size, mc.global_size), dtype=tdt).pin_memory(),
            "hl": torch.empty((Lc, n, 3, mc.local_size, mc.local_size), dtype=tdt).pin_memory(),
            "done": torch.cuda.Event(),
        })
    comp, copy = torch.cuda.Stream(), torch.cuda.Stream()
    src = loader.src

    def step(i):
        b = bufs[i % 2]
        with torch.cuda.stream(comp):
            comp.wait_event(b["done"])  # buffer free once its previous D2H finished
            b["specs"].copy_(host_specs[i % 2], non_blocking=True)
            if loader.needs_resample:
                loader.slide_set.read_regions(b["specs"], mc.src_size, out=src, planned=True)
            crop_params(mc, n, loader.seed, loader.rank, 10_000 + i, out=b["params"], stream=comp)
            multicrop(loader.slide_set, b["specs"], b["params"], mc, dtype=loader.dtype, src_hwc=src,
                      out_global=b["g"], out_local=b["l"], stream=comp)
            ev = torch.cuda.Event()
            ev.record(comp)
        with torch.cuda.stream(copy):
            copy.wait_event(ev)
            b["hg"].copy_(b["g"], non_blocking=True)
            if Lc:
                b["hl"].copy_(b["l"], non_blocking=True)
            b["done"].record(copy)

    return _time_e2e(step, steps, n, torch, n * 64,
                     bufs[0]["hg"].numel() * bufs[0]["hg"].element_size() + bufs[0]["hl"].numel() * bufs[0]["hl"].element_size(),
                     "pinned host specs -> pf_crop_params/pf_multicrop -> pinned host crops, 2 streams double-buffered")


def run_e2e_regions(pf, loader, steps, torch):
    """Pinned host specs -> H2D -> pf_read_regions (normalising epilogue) -> D2H of the batch."""
    n = loader.batch_size
    torch.cuda.synchronize()
    host_specs = [loader.sampler.next_batch(n).cpu().pin_memory() for _ in range(2)]
    bufs = [{"specs": torch.empty((n, 64), dtype=torch.uint8, device="cuda"), "out": torch.empty_like(loader.out),
             "host": torch.empty(loader.out.shape, dtype=loader.out.dtype).pin_memory(), "done": torch.cuda.Event()}
            for _ in range(2)]
    comp, copy = torch.cuda.Stream(), torch.cuda.Stream()

    def step(i):
        b = bufs[i % 2]
        with torch.cuda.stream(comp):
            comp.wait_event(b["done"])
            b["specs"].copy_(host_specs[i % 2], non_blocking=True)
            loader.slide_set.read_regions(b["specs"], loader.out_size, dtype=loader.dtype, layout=loader.layout,
                                          mean=loader.mean, std=loader.std, out=b["out"], stream=comp, planned=True)
            ev = torch.cuda.Event()
            ev.record(comp)
        with torch.cuda.stream(copy):
            copy.wait_event(ev)
            b["host"].copy_(b["out"], non_blocking=True)
            b["done"].record(copy)

    return _time_e2e(step, steps, n, torch, n * 64, bufs[0]["host"].numel() * bufs[0]["host"].element_size(),
                     "pinned host specs -> pf_read_regions -> pinned host patches, 2 streams double-buffered")


def _time_e2e(step, steps, n, torch, h2d, d2h, path):
    for i in range(2):
        step(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        step(i)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    return {"value": round(steps * n / dt, 1), "unit": "patches/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "path": path + "; wall clock over the steps"}


def timed_run(feed, args, torch, dist, world, local, N):
    """W warm-up steps, then K timed steps between barriers; per-stage CUDA events."""
    loader = feed.loader
    clk = ClockSampler(torch.cuda.current_device()).__enter__()  # sampling spans warm-up + timed steps (all under load)
    for _ in range(max(args.warmup, 0)):
        loader.next_batch()
    torch.cuda.synchronize()
    tiers = getattr(loader, "tiers", None)
    filled0 = tiers.tiles_filled() if tiers is not None else 0
    loader.sampler.update_estimate()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    marks_all = []
    l0 = N.launches()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed")
    start.record(stream)
    res_ev = []
    for _ in range(args.steps):
        marks = []
        out = loader.next_batch(marks=marks)
        marks_all.append(marks)
        if isinstance(out, dict) and out.get("resample_events") is not None:
            res_ev.append(out["resample_events"])
    end.record(stream)
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    launches = N.launches() - l0
    if tiers is not None:  # host-backed tier traffic of the timed steps (zero-copy H2D by the fill kernel)
        filled = tiers.tiles_filled() - filled0
        args.tier_stats = {"tiles_filled_per_step": round(filled / args.steps, 1),
                           "h2d_gb_per_step": round(filled * 256 * 256 * 3 / args.steps / 1e9, 3)}
    elapsed_ms = start.elapsed_time(end)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda" if args.dist_backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    stages: dict = {}
    for marks in marks_all:
        for (_, ea), (b, eb) in zip(marks[:-1], marks[1:]):
            stages.setdefault(b, []).append(ea.elapsed_time(eb))
    stage_ms = {k: sum(v) / len(v) for k, v in stages.items()}
    if res_ev:  # the resample runs on the loader's side stream (overlapping the previous multi-crop)
        stage_ms["resample"] = sum(a.elapsed_time(b) for a, b in res_ev) / len(res_ev)
    return float(t.item()), stage_ms, launches, clk.summary()


def issue_roofline(args, k_ms):
    """The bound that binds the multi-crop kernel: instruction issue.  Warp-instructions per patch
    come from the committed ncu capture (profiles/instr_config<N>.json); the ceiling is one
    warp-instruction per scheduler per clock: 148 SMs x 4 x sm_max_mhz."""
    ip = ROOT / "profiles" / f"instr_config{args.config}.json"
    if not ip.exists():
        return None
    try:
        wipp = float(json.loads(ip.read_text())["warp_instructions_per_patch"])
    except (ValueError, KeyError):
        return None
    peak = 148 * 4 * 1965e6
    achieved = wipp * args.batch / (k_ms / 1000.0)
    return {"unit": "warp-instr/s", "achieved": round(achieved, -6), "peak": peak, "frac": round(achieved / peak, 4),
            "warp_instructions_per_patch": wipp, "source": json.loads(ip.read_text()).get("source")}


def result_line(feed, args, world, elapsed_ms, stage_ms, launches, clocks, st, e2e, cpu):
    peak, peak_kind = measured_peak_hbm()
    n_total = args.steps * args.batch * world
    value = n_total / (elapsed_ms / 1000.0)
    k_ms = sum(stage_ms[k] for k in feed.stages)
    achieved = feed.bytes_per_patch * args.batch / (k_ms / 1000.0) / 1e9
    traffic = None
    tp = ROOT / "profiles" / f"traffic_config{args.config}.json"
    if tp.exists():
        try:
            tpp = json.loads(tp.read_text()).get("dram_bytes_per_patch")
            traffic = int(tpp * args.batch) if tpp else None
        except Exception:  # noqa: BLE001
            traffic = None
    return {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "patches/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(elapsed_ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (BASELINE generator: near-white background + N(0,4), H&E-like blobs ~40%)",
        "config": {
            "workload": feed.workload,
            "global_batch": args.batch * world,
            "batch_per_gpu": args.batch,
            "parallelism": f"slide-sharded x{world}, no data-path collective",
            "l2": "inputs larger than L2 (slides resident in HBM, random patches; outputs stream out)",
        },
        "roofline": {
            "bound": "hbm",
            "kernel": feed.kernel,
            "achieved": round(achieved, 1),
            "peak": peak,
            "peak_kind": peak_kind,
            "unit": "GB/s",
            "frac": round(achieved / peak, 4),
            "traffic": traffic,
            "algorithmic_bytes_per_patch": feed.bytes_per_patch,
            "per_launch_ms": round(k_ms, 4),
            "frac_of_nominal_8tbs": round(achieved / 8000.0, 4),  # north_star's ~8 TB/s nominal HBM3e
        },
        "issue_roofline": issue_roofline(args, k_ms),
        "stages_ms": {k: round(v, 4) for k, v in stage_ms.items()},
        "sampler": {"attempts": int(st.attempts), "specs": int(st.seq), "slow_evals": int(st.slow_evals)},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": e2e,
        "cpu_baseline": cpu,
        **({"tier": {**args.tier, **getattr(args, "tier_stats", {}),
                     "stall_ms_per_step": round(stage_ms.get("sample_wait", 0.0), 4)}}
           if getattr(args, "tier", None) else {}),
    }


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2404_15217_b200 import _native as N

    rank, world, local = dist_env()
    dev = local if args.device is None else args.device
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    pf, plan, slides = build_slides(args, rank, world)
    if args.config == "5":
        run_sweep(args, pf, plan, slides, rank, world, local, torch, dist, N)
        return
    feed = make_feed(args, pf, plan, slides, rank)
    if args.dump_dir:  # the rank's first batch (step 0): specs + crop parameters
        out = feed.loader.next_batch()
        torch.cuda.synchronize()
        Path(args.dump_dir).mkdir(parents=True, exist_ok=True)
        extra = {"params": out["params"].cpu().numpy()} if "params" in out else {}
        np.savez(Path(args.dump_dir) / f"rank{rank}.npz", specs=out["specs"].cpu().numpy(), rank=rank, world=world,
                 sampler_seed=plan.sampler_seed, philox_seed=plan.philox_seed,
                 slide_indices=np.array(plan.slide_indices), **extra)
    elapsed_ms, stage_ms, launches, clocks = timed_run(feed, args, torch, dist, world, local, N)
    st = feed.sampler.check()
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(3, min(args.steps, 10))
        if world > 1:
            dist.barrier()
        e2e = feed.e2e_fn(pf, feed.loader, e2e_steps, torch)
        if world > 1:  # whole job: every rank's patches over the slowest rank's wall time
            n_rank = e2e_steps * feed.loader.batch_size
            te = torch.tensor([n_rank / e2e["value"]], dtype=torch.float64,
                              device="cuda" if args.dist_backend == "nccl" else "cpu")
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
            e2e["value"] = round(world * n_rank / float(te.item()), 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, steps=args.cpu_steps, slides=slides)
    if rank == 0:
        print(json.dumps(result_line(feed, args, world, elapsed_ms, stage_ms, launches, clocks, st, e2e, cpu)), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sweep(args, pf, plan, slides, rank, world, local, torch, dist, N):
    """BASELINE config 5: one 100000x80000 slide; patch 224/256/512 -> 224, batch 256..8192,
    L in {0, 4, 8} local crops, fp32 vs bf16.  Every point -> profiles/sweep (JSON lines);
    the headline line is the default point (224, 1024, L=8, bf16)."""
    out_dir = Path(os.environ.get("PF_SWEEP_DIR", ROOT / "gpurun_out"))
    out_dir.mkdir(parents=True, exist_ok=True)
    points = []
    head = None
    for patch in (224, 256, 512):
        for batch in (256, 1024, 4096, 8192):
            for n_local in (0, 4, 8):
                for dtype in ("bf16", "f32"):
                    a = argparse.Namespace(**vars(args))
                    a.batch, a.dtype, a.steps, a.warmup = batch, dtype, max(3, min(args.steps, 5)), 3
                    print(f"[sweep] patch {patch} batch {batch} L={n_local} {dtype}", file=sys.stderr, flush=True)
                    feed = make_feed(a, pf, plan, slides, rank, n_local=n_local, patch=patch)
                    elapsed_ms, stage_ms, launches, clocks = timed_run(feed, a, torch, dist, world, local, N)
                    st = feed.sampler.check()
                    line = result_line(feed, a, world, elapsed_ms, stage_ms, launches, clocks, st, None, None)
                    line["point"] = {"patch": patch, "batch": batch, "n_local": n_local, "dtype": dtype}
                    points.append(line)
                    if (patch, batch, n_local, dtype) == (224, 1024, 8, "bf16"):
                        head = line
                    del feed
                    torch.cuda.empty_cache()
    if rank == 0:
        (out_dir / "sweep_config5.jsonl").write_text("".join(json.dumps(p) + "\n" for p in points))
        head = dict(head or points[-1])
        head["sweep"] = [{**p["point"], "patches_per_s": p["value"], "achieved_gbs": p["roofline"]["achieved"],
                          "frac": p["roofline"]["frac"]} for p in points]
        print(json.dumps(head), flush=True)


# ---------------------------------------------------------------------------
# CPU arms (oracle port on the host cores)


def _cpu_polygons(args, slides=None):
    """Rings for the CPU arm: the GPU arm's traced saturation+morphology polygons when this process
    built them (same_config), else the committed masks of the 16 C2 slides (tests/golden/
    c2_masks16.npz, made by the GPU arm's renderer and mask kernel) traced by the oracle, else
    the synthetic field's mask."""
    if slides is not None:
        return [[np.asarray(r) for r in poly.rings] for _, poly in slides], "gpu_arm"
    p = ROOT / "tests" / "golden" / "c2_masks16.npz"
    if args.config in ("2", "3") and (args.width, args.height) == (40000, 30000) and args.slides <= 16 and p.exists():
        from oracle import port

        z = np.load(p)
        polys = []
        for g in range(args.slides):
            shape = tuple(z[f"s{g}_shape"])
            bits = np.unpackbits(z[f"s{g}_mask"])[: shape[0] * shape[1]].reshape(shape).astype(bool)
            polys.append(port.polygon_from_mask(bits, float(z[f"s{g}_scale"][0]), 64.0))
        return polys, "c2_masks16"
    return None, "field"


def _cpu_run(args, steps, polygons):
    from oracle import cpu_pipeline as cp

    cores = cp.cpu_count()
    if args.config == "4":  # the C4 set's sizes come from a seed; the CPU sample uses its mean slide
        args.width, args.height = 70000, 55000
    per_step, cands = cp.run(cores, args.slides, args.width, args.height, candidates_per_step=1, steps=steps,
                             augment=args.config != "1", polygons=polygons)
    return cp, cores, per_step, cands


def cpu_baseline(args, steps=2, slides=None):
    polygons, poly_src = _cpu_polygons(args, slides)
    cp, cores, per_step, cands = _cpu_run(args, steps + 1, polygons)
    timed = per_step[1:]
    value, stages = cp.summarize(timed, cores, cands, augment=args.config != "1")
    return {"value": round(value, 4), "unit": "patches/s", "cores": cores, "kind": "port",
            "cpu_model": cp.cpu_model(), "stages": stages, "polygons": poly_src,
            "same_config": poly_src in ("gpu_arm", "c2_masks16"),
            "sample": f"{steps} steps x {cores} workers: 1 epoch_stream candidate, 48 read_region+normalize_patch, "
                      f"4 torchvision multi-crops each; value = 1/(1/sampler + 1/loader + 1/augment) "
                      f"over all workers; {cands} candidates total"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    polygons, poly_src = _cpu_polygons(args)
    cp, cores, per_step, cands = _cpu_run(args, args.warmup + args.steps, polygons)
    timed = per_step[args.warmup:]
    value, stages = cp.summarize(timed, cores, cands, augment=args.config != "1")
    t = sum(max(s["sampler"][0], 0) + s["loader"][0] + s["augment"][0] for s in timed)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 4),
        "unit": "patches/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(1000 * t / max(len(timed), 1), 1),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": args.dtype,
        "data": "synthetic (numpy restatement of the same generator, tiles rendered on first touch)",
        "config": {"workload": f"C{args.config} on CPU: {args.slides} slides {args.width}x{args.height}, reference "
                               "epoch_stream (numpy even-odd overlap), read_region + normalize_patch, " +
                               ("(no augmentation)" if args.config == "1" else
                                "torchvision multi-crop 2x224+8x96, bf16"),
                   "global_batch": args.batch, "parallelism": f"{cores} worker processes, seed + worker"},
        "cpu_baseline": {"value": round(value, 4), "unit": "patches/s", "cores": cores, "kind": "port",
                         "cpu_model": cp.cpu_model(), "stages": stages, "polygons": poly_src,
                         "same_config": poly_src in ("gpu_arm", "c2_masks16"),
                         "sample": f"{len(timed)} steps x {cores} workers: 1 sampler candidate, 48 loads, 4 "
                                   f"multi-crops each; {cands} candidates"},
        "e2e": {"value": round(value, 4), "unit": "patches/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
