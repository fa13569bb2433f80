"""GPU probes of the arithmetic the multi-crop kernel relies on (tools/*.cu, built with the
library's nvcc flags): the packed f32x2 ops round exactly like their scalar IEEE forms, and the
packed adjust_hue equals the scalar one on every RGB colour."""

import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _build_and_run(name, tmp_path):
    from paper_2404_15217_b200 import build as b

    exe = tmp_path / name
    cmd = [b.NVCC, *b.ARCH, "-O3", "-std=c++17", "-fmad=false", "-o", str(exe), str(ROOT / "tools" / f"{name}.cu")]
    subprocess.run(cmd, check=True, capture_output=True)
    return subprocess.run([str(exe)], check=True, capture_output=True, text=True, timeout=120).stdout


def test_f32x2_ops_match_scalar(cuda, tmp_path):
    out = _build_and_run("probe_f32x2", tmp_path)
    lines = [l for l in out.splitlines() if l.startswith("mode")]
    assert len(lines) == 3 and all("mismatches 0, add.rm2 0, mul2 0" in l for l in lines), out


def test_packed_hue_matches_scalar_on_every_colour(cuda, tmp_path):
    out = _build_and_run("probe_hue", tmp_path)
    lines = [l for l in out.splitlines() if l.startswith("hf")]
    assert len(lines) == 5 and all(l.endswith(": 0 mismatches") for l in lines), out
