"""T1 mapping parity WITHOUT a GPU: the library's hash (implementation #2, the
`__host__ __device__` code the kernels run, incl. the reciprocal `mod R`) evaluated
on the host through roast_debug_hash_host, against the oracle (implementation #1,
Python integers, plain `%`).  Bit-exact."""
import random

import numpy as np
import pytest

from oracle import hashing as H


@pytest.fixture(scope="module")
def R():
    from paper_2207_10702_b200 import build, roast
    build.build()
    return roast


@pytest.mark.parametrize("mem,span,align", [
    (8192, 1024, 8), (47192, 4096, 8), (4720, 4096, 8), (471864, 4096, 8),
    (33_280_000, 32, 8), (4096, 4096, 8), (4103, 4096, 8), (1 << 20, 1, 1), (2 ** 33 + 5, 64, 8),
    (1000, 1, 1), (3, 1, 1),
])
def test_library_hash_equals_oracle(R, mem, span, align):
    rnd = random.Random(mem * 31 + span)
    keys = [0, 1, 2, (1 << 60) - 1] + [rnd.randrange(1 << 60) for _ in range(1500)] + \
           [H.tile_key(x, y) for x in range(6) for y in range(6)]
    for seed, module in [(0x5EED, 0), (0x5EED, 7), (123456789, 2)]:
        off, sgn = R.roast_debug_hash_host(seed, module, keys, mem, span, align)
        mh = H.ModuleHash(seed, module, mem, span, align)
        assert off.tolist() == [mh.offset(k) for k in keys]
        assert sgn.astype(int).tolist() == [mh.sign(k) for k in keys]


def test_reciprocal_mod_edges(R):
    """R values around powers of two and the largest residues of the 61-bit range."""
    rnd = random.Random(5)
    for Rv in [1, 2, 3, 7, 8, 9, 255, 256, 257, 5388, 58472, (1 << 31) - 1, 1 << 31, (1 << 32) + 1,
               (1 << 33) - 3]:
        mem = Rv - 1 + 1          # span 1, align 1: R = mem
        keys = [rnd.randrange(1 << 60) for _ in range(300)] + [(1 << 60) - 1 - i for i in range(20)]
        off, _ = R.roast_debug_hash_host(99, 3, keys, mem, 1, 1)
        mh = H.ModuleHash(99, 3, mem, 1, 1)
        assert mh.R == Rv
        assert off.tolist() == [mh.offset(k) for k in keys]


def test_rejects_bad_geometry(R):
    with pytest.raises(R.RoastError):
        R.roast_debug_hash_host(1, 0, [1, 2], 10, 11, 1)
    with pytest.raises(R.RoastError):
        R.roast_debug_hash_host(1, 0, [1 << 60], 100, 1, 1)


def test_lms_segments_product_matches_oracle():
    """The library's roast_lms_segments (C ABI, host) == the oracle's reading R23."""
    from oracle import hashing as OH
    from paper_2207_10702_b200 import roast
    for sizes, mem, A in [([768 * 3072, 3072 * 768], 47_192, 8), ([1, 2, 3, 4, 5], 100_000, 32), ([7], 64, 8),
                          ([10 ** 9, 1, 1], 1 << 20, 8)]:
        assert roast.lms_segments(sizes, mem, A) == OH.lms_segments(sizes, mem, A)


def test_lms_segments_rejects_bad_arguments(R):
    with pytest.raises(R.RoastError):
        R.lms_segments([], 100, 8)
    with pytest.raises(R.RoastError):
        R.lms_segments([1, 0], 100, 8)
    with pytest.raises(R.RoastError):
        R.lms_segments([1, 2], 100, 0)
