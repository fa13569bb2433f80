"""The package's exceptions are caught by the reference's own `except` clauses when the
reference (patchforge) is importable (the shim raises the reference's classes).
Runs in a subprocess with the reference imported from /root/reference (skimage stubbed, as in
tests/golden/make_goldens.py); skipped where the reference is absent (GPU boxes)."""

import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r'''
import sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {root!r} + "/tests/golden")
from make_goldens import import_reference
rng, store, foreground, sampler, pipeline = import_reference()
from paper_2404_15217_b200 import errors as E
pairs = [(E.OutOfBoundsError, store.OutOfBoundsError), (E.StoreError, store.StoreError),
         (E.SlideNotFoundError, store.SlideNotFoundError), (E.IntegrityError, store.IntegrityError),
         (E.DecodeError, store.DecodeError), (E.TransportError, store.TransportError),
         (E.EmptyForegroundError, foreground.EmptyForegroundError),
         (E.ExhaustedAttemptsError, sampler.ExhaustedAttemptsError),
         (E.NoSamplableSlideError, sampler.NoSamplableSlideError),
         (E.PackFormatError, pipeline.PackFormatError), (E.LoaderError, pipeline.LoaderError)]
for ours, ref in pairs:
    assert issubclass(ours, ref), (ours, ref)
    try:
        raise ours("x")
    except ref:
        pass
assert issubclass(E.OutOfBoundsError, E.StoreError) and issubclass(E.EmptyForegroundError, ValueError)
# the product's own raise sites
from paper_2404_15217_b200.store import plan_specs, make_record
rec = make_record("r", 100, 100, 0.25, 64, 2)
try:
    plan_specs([(0, (90, 90, 20, 20), 0.25, 20)], [rec])
except store.OutOfBoundsError:
    print("caught")
'''


def test_reference_except_clauses_catch_package_errors():
    if not Path("/root/reference/pkg/src/patchforge").is_dir():
        pytest.skip("reference not present")
    res = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT))], capture_output=True, text=True,
                         timeout=300)
    assert res.returncode == 0, res.stderr
    assert "caught" in res.stdout


def test_standalone_hierarchy_without_reference():
    res = subprocess.run([sys.executable, "-c", "import sys; sys.path.insert(0, %r)\n"
                          "from paper_2404_15217_b200 import errors as E\n"
                          "assert E.OutOfBoundsError.__mro__[1] is E.StoreError\n"
                          "assert E.StoreError.__bases__ == (Exception,)\n"
                          "assert issubclass(E.LoaderError, RuntimeError)\n" % str(ROOT)],
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
