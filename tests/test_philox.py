"""Philox4x32-10 of the augmentation parameter generator: native implementation vs the
Random123 known-answer vectors and the Python restatement (CPU, host entry point)."""

import ctypes as C

import numpy as np

from oracle import philox


def test_native_philox_kats():
    from paper_2404_15217_b200 import _native as N

    L = N.lib()
    for ctr, key, want in philox.KATS:
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        L.pf_philox4x32_10(c, k, o)
        assert tuple(o) == want
    rs = np.random.default_rng(0)
    for _ in range(200):
        ctr = [int(v) for v in rs.integers(0, 2**32, 4)]
        key = [int(v) for v in rs.integers(0, 2**32, 2)]
        c, k, o = (C.c_uint32 * 4)(*ctr), (C.c_uint32 * 2)(*key), (C.c_uint32 * 4)()
        L.pf_philox4x32_10(c, k, o)
        assert list(o) == philox.philox4x32_10(ctr, key)
