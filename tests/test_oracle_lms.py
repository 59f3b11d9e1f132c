"""Pins for the oracle's local-memory-sharing (LMS) segments (NEXT #4).

LMS is defined by the paper as "each layer will have independent compressed
memory" M_i with sum |M_i| = |M| and |M_i| = f_i |M|.  So a
module hashed into segment (b, s) of M must be exactly the GMS module of a store
of size s that *is* M[b : b + s] - checked here against the GMS oracle, whose own
pins live in test_oracle_mm.py / test_oracle_embedding.py.
"""
import numpy as np
import pytest

import synth
from oracle import embedding as OE
from oracle import hashing
from oracle import roast_mm as RM


@pytest.mark.parametrize("sizes,mem,A", [([1, 1], 16, 8), ([3, 1], 1000, 8), ([768 * 3072, 3072 * 768, 30522 * 768], 471_864, 8),
                                         ([5, 7, 11, 13], 4096, 32), ([1], 64, 8)])
def test_lms_segments_partition(sizes, mem, A):
    segs = hashing.lms_segments(sizes, mem, A)
    n = sum(sizes)
    assert segs[0][0] == 0 and sum(s for _, s in segs) == mem
    for i, (b, s) in enumerate(segs):
        assert b % A == 0
        if i + 1 < len(segs):
            assert segs[i + 1][0] == b + s                      # contiguous, disjoint
            assert 0 <= sizes[i] * mem / n - s < A              # floor(f_i m) aligned down (R14/R23)
    assert hashing.lms_segments([1, 1], 16, 8) == [(0, 8), (8, 8)]
    # worked by hand: f = (3/4, 1/4) of 1000 -> floor(750) aligned down to 8 = 744, rest 256;
    # f = (1/3, 1/3, 1/3) of 100 (A = 1) -> 33, 33, remainder 34
    assert hashing.lms_segments([3, 1], 1000, 8) == [(0, 744), (744, 256)]
    assert hashing.lms_segments([2, 2, 2], 100, 1) == [(0, 33), (33, 33), (66, 34)]


def test_lms_linear_is_gms_on_its_submemory():
    mem, A, z = 4096, 8, 8
    M = synth.uniform(11, (mem,))
    X = synth.normal(12, (5, 32))
    dY = synth.normal(13, (5, 24))
    for mid, (b, s) in enumerate([(0, 1024), (1024, 1536), (2560, 1536)]):
        lms = RM.LinearSpec(32, 24, z, z, mem, 7, mid, align=A, segment=(b, s))
        gms = RM.LinearSpec(32, 24, z, z, s, 7, mid, align=A)
        slots = lms.slot_index()
        assert slots.min() >= b and slots.max() < b + s
        assert np.array_equal(slots, gms.slot_index() + b)
        assert np.array_equal(lms.forward(X, M), gms.forward(X, M[b:b + s]))
        assert np.array_equal(lms.backward_dx(dY, M), gms.backward_dx(dY, M[b:b + s]))
        dM = lms.backward_dm(X, dY)
        assert not dM[:b].any() and not dM[b + s:].any()
        assert np.array_equal(dM[b:b + s], gms.backward_dm(X, dY))


def test_lms_whole_memory_is_gms():
    mem = 2048
    a = RM.LinearSpec(64, 64, 8, 8, mem, 3, 1, segment=(0, mem))
    g = RM.LinearSpec(64, 64, 8, 8, mem, 3, 1)
    assert np.array_equal(a.off, g.off) and np.array_equal(a.sgn, g.sgn)


def test_lms_embedding_is_gms_on_its_submemory():
    mem, b, s = 5000, 1600, 2400
    M = synth.uniform(21, (mem,))
    rows = synth.uniform_indices(22, 50, 1000)
    dOut = synth.normal(23, (50, 20))
    lms = OE.EmbeddingSpec(1000, 20, 8, mem, 9, 2, segment=(b, s))
    gms = OE.EmbeddingSpec(1000, 20, 8, s, 9, 2)
    off, _ = lms.chunk_map(rows)
    assert off.min() >= b and off.max() + 8 <= b + s
    assert np.array_equal(lms.forward(rows, M), gms.forward(rows, M[b:b + s]))
    dM = lms.backward(rows, dOut)
    assert not dM[:b].any() and not dM[b + s:].any()
    assert np.array_equal(dM[b:b + s], gms.backward(rows, dOut))
