"""Pins for oracle/hashing.py (no GPU).  SURVEY.md §8(c) tests O1-O9."""
import os
import random
import subprocess
import sys

import numpy as np
import pytest

from oracle import hashing as H

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hash_c1.txt")


def test_golden_survey_prototype():
    """Appendix-A transcription check against an independent prototype."""
    rows = [l.split() for l in open(GOLDEN) if l.strip() and not l.startswith("#")]
    mh = H.ModuleHash(0x5EED, 0, 8192, 32 * 32, 8)
    for r in rows:
        if r[0] == "R":
            assert mh.R == int(r[1])
        elif r[0] == "RC2":
            assert H.num_positions(int(r[1]), 64 * 64, 8) == int(r[2])
        else:
            x, y, off, sg = map(int, r)
            k = H.tile_key(x, y)
            assert mh.offset(k) == off and mh.sign(k) == sg


def test_splitmix64_reference_vector():
    """splitmix64 seeded with 0: the first outputs of the published generator
    (Steele, Lea & Flood 2014; Vigna's reference C code) are
    0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4 for states 0x9E37..15 * {1, 2} - golden."""
    assert H.splitmix64(0) == 0xE220A8397B1DCDAF
    assert H.splitmix64(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_mersenne_poly_matches_bruteforce_small():
    """poly61 is Horner for c3 k^3 + c2 k^2 + c1 k + c0 mod p: compare the expanded sum."""
    rnd = random.Random(1)
    for _ in range(200):
        c = tuple(rnd.randrange(H.P61) for _ in range(4))
        k = rnd.randrange(1 << 60)
        expanded = (c[3] * k ** 3 + c[2] * k ** 2 + c[1] * k + c[0]) % H.P61
        assert H.poly61(c, k) == expanded


def test_O1_range_and_alignment_fuzz():
    rnd = random.Random(7)
    for _ in range(20000):
        T = rnd.choice([1, 64, 1024, 4096])
        A = rnd.choice([1, 8])
        m = rnd.randrange(T, 1 << 31)
        seed, mod = rnd.randrange(1 << 64), rnd.randrange(1 << 16)
        key = rnd.randrange(1 << 60)
        off = H.offset(seed, mod, key, m, T, A)
        assert 0 <= off <= m - T and off % A == 0


def test_O2_determinism_across_processes():
    keys = list(range(0, 10 ** 6, 997))
    mh = H.ModuleHash(123, 4, 1 << 20, 64, 8)
    here = [mh.offset(k) * 2 + (mh.sign(k) > 0) for k in keys]
    code = ("import sys; sys.path.insert(0, %r); from oracle import hashing as H;"
            "mh=H.ModuleHash(123,4,1<<20,64,8);"
            "print(sum((mh.offset(k)*2+(mh.sign(k)>0))*(i+1) for i,k in enumerate(range(0,10**6,997))))"
            % os.path.dirname(os.path.dirname(__file__)))
    out = subprocess.check_output([sys.executable, "-c", code], text=True)
    assert int(out) == sum(v * (i + 1) for i, v in enumerate(here))


def test_O3_single_legal_offset():
    for key in range(100):
        assert H.offset(7, 0, key, 1024, 1024, 8) == 0      # |M| = T
        assert H.offset(7, 0, key, 1031, 1024, 8) == 0      # |M| < T + A
        assert H.offset(7, 0, key, 8, 8, 1) == 0
    with pytest.raises(ValueError):
        H.num_positions(8, 9, 1)                            # geometry error S:42


def test_O4_uniformity_chi_square():
    mh = H.ModuleHash(11, 2, 1000, 1, 1)
    n = 200000
    counts = np.bincount([mh.offset(k) for k in range(n)], minlength=1000)
    e = n / 1000
    chi2 = float(np.sum((counts - e) ** 2 / e))
    assert chi2 < 1143.0        # df 999, p = 0.001


def test_O5_birthday_collisions():
    rnd = random.Random(5)
    pairs = set()
    while len(pairs) < 100000:
        pairs.add((rnd.randrange(1 << 16), rnd.randrange(1 << 16)))
    R = 1 << 20
    mh = H.ModuleHash(99, 1, R, 1, 1)
    cnt = np.bincount([mh.offset(H.tile_key(x, y)) for x, y in pairs], minlength=R)
    colliding_pairs = int(np.sum(cnt * (cnt - 1) // 2))
    n = len(pairs)
    expected = n * (n - 1) / 2 / R
    assert abs(colliding_pairs - expected) <= 3 * np.sqrt(expected)


def test_O6_seed_sensitivity():
    m = 1 << 20
    a = H.ModuleHash(1000, 0, m, 64, 8)
    b = H.ModuleHash(1001, 0, m, 64, 8)
    differ = sum(a.offset(k) != b.offset(k) for k in range(10000))
    assert differ >= 9900
    c = H.ModuleHash(1000, 1, m, 64, 8)                     # module id also keys the family
    assert sum(a.offset(k) != c.offset(k) for k in range(10000)) >= 9900


def test_O7_sign_balance_and_square():
    mh = H.ModuleHash(0x5EED, 3, 1 << 20, 64, 8)
    s = np.array([mh.sign(k) for k in range(200000)])
    assert set(np.unique(s)) <= {-1, 1}
    assert np.all(s * s == 1)
    assert abs(s.mean()) <= 3 / np.sqrt(len(s))


def test_O8_four_wise_sign_moments():
    rnd = random.Random(8)
    N = 20000
    q4 = np.empty(N)
    q2 = np.empty(N)
    for t in range(N):
        a, b, c, d = rnd.sample(range(1 << 40), 4)
        mh = H.ModuleHash(rnd.randrange(1 << 64), 0, 1 << 20, 64, 8)
        ga, gb, gc, gd = (mh.sign(k) for k in (a, b, c, d))
        q4[t] = ga * gb * gc * gd
        q2[t] = ga * gb
    assert abs(q4.mean()) <= 4 / np.sqrt(N)
    assert abs(q2.mean()) <= 4 / np.sqrt(N)


def test_O9_lambda():
    assert H.lam(1.0, 4) == 0.5
    assert H.lam(2.0, 16) == 0.5
    assert H.lam(1.0, 256) == 0.0625
    assert H.lam(1.0, 768) == float(np.float32(1 / np.sqrt(768)))
