"""Touched-set dM exchange (large-|M| regime): the host interval logic of
libroast (roast_touched_intervals, no GPU) against brute force.

The set of dM slots a linear can write is exactly {slot_index(i, j)} of its virtual weights
(the oracle's element-by-element mapping); the library's merged intervals of
[off_t, off_t + Z1 Z2) must equal that set — brute force over every weight pins it.
"""
import numpy as np
import pytest

import synth
from oracle import roast_mm as OM
from paper_2207_10702_b200 import roast as R


def _covered(starts, lens, mem):
    m = np.zeros(mem, dtype=bool)
    for s, l in zip(starts, lens):
        m[s:s + l] = True
    return m


def test_merge_matches_bruteforce_coverage():
    rng = np.random.default_rng(7)
    for trial in range(50):
        mem = int(rng.integers(100, 5000))
        span = int(rng.integers(1, 300))
        n = int(rng.integers(0, 60))
        starts = rng.integers(0, mem - span + 1, size=n)
        s, l = R.roast_touched_intervals(starts, span)
        cover = np.zeros(mem, dtype=bool)
        for a in starts:
            cover[a:a + span] = True
        assert np.array_equal(_covered(s, l, mem), cover)
        # sorted, disjoint and non-adjacent (maximal runs)
        assert np.all(l > 0)
        assert np.all(s[1:] > s[:-1] + l[:-1])


@pytest.mark.parametrize("H,O,mem", [(256, 256, 1 << 20), (512, 192, 4720 * 4), (4096, 4096, 2 << 20)])
def test_intervals_equal_every_slot_the_layer_maps_to(H, O, mem):
    spec = OM.LinearSpec(H, O, 64, 64, mem, synth.HASH_SEED, 0)
    s, l = R.roast_touched_intervals(spec.off.ravel(), 64 * 64)
    slots = np.zeros(mem, dtype=bool)
    slots[spec.slot_index().ravel()] = True
    assert np.array_equal(_covered(s, l, mem), slots)
    assert int(l.sum()) == int(slots.sum())


def test_gradient_lives_in_the_touched_set():
    """dM of random X, dY (oracle, fp64) is zero outside the intervals: packing loses nothing."""
    mem = 1 << 18
    layers = [OM.LinearSpec(128, 192, 64, 64, mem, synth.HASH_SEED, 0),
              OM.LinearSpec(192, 128, 64, 64, mem, synth.HASH_SEED, 1)]
    dM = np.zeros(mem)
    layers[0].backward_dm(synth.normal(2, (33, 128)), synth.normal(3, (33, 192)), dM)
    layers[1].backward_dm(synth.normal(4, (33, 192)), synth.normal(5, (33, 128)), dM)
    s, l = R.roast_touched_intervals(np.concatenate([sp.off.ravel() for sp in layers]), 4096)
    inside = _covered(s, l, mem)
    assert np.count_nonzero(dM[~inside]) == 0
    assert np.count_nonzero(dM[inside]) == int(l.sum())   # generic inputs: every touched slot nonzero


def test_capacity_and_argument_errors():
    import ctypes
    starts = np.array([0, 10000], dtype=np.int64)
    out_s = np.empty(1, dtype=np.int64)
    out_l = np.empty(1, dtype=np.int64)
    cnt = ctypes.c_int64()
    st = R._lib.roast_touched_intervals(starts.ctypes.data, 2, 64, out_s.ctypes.data, out_l.ctypes.data, 1,
                                        ctypes.byref(cnt))
    assert st == R.ERR_CAPACITY and cnt.value == 2
    assert R._lib.roast_touched_intervals(starts.ctypes.data, 2, 0, None, None, 0, ctypes.byref(cnt)) == R.ERR_CONFIG
