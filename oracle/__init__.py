"""TEST INFRASTRUCTURE ONLY — CPU oracle for the Online Patching hot path.

This package restates the reference algorithm (patchforge, mounted read-only
at /root/reference; cited as pkg/<module>.py:<line>) in numpy / plain Python
so the CUDA path can be checked against it.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import it, and only as
the checker or the timed CPU baseline — never as part of the product path.

Parity pinning: tests/golden/ holds vectors produced by importing the real
reference in the build container (tests/golden/make_goldens.py); the oracle
is checked against them by tests/test_oracle.py.  Rows the reference does not
contain (HSV-saturation mask, multi-crop augmentation) are oracled against
scipy.ndimage / torchvision and are "parity unpinned" by the reference.
"""
