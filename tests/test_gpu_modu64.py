"""GPU: the sampler's division-free v % n (pf_common.cuh mod_u64) and its randrange acceptance
shortcut equal the plain 64-bit operators on ~155 M draws spanning every divisor magnitude
and the numerator edge cases (top of the range, multiples, small values)."""

import shutil
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def test_mod_u64_matches_operator(cuda, tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "mod_check"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-fmad=false",
                    f"-I{ROOT / 'include'}", f"-I{ROOT / 'paper_2404_15217_b200' / 'csrc'}",
                    str(ROOT / "tests" / "cuda" / "mod_u64_check.cu"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches 0" in r.stdout
