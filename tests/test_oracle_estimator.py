"""Pins for oracle/estimator.py (no GPU).  SURVEY.md §8(c) tests O17-O20."""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import estimator as S


@pytest.mark.parametrize("x,y,m", [
    ((1, 0), (0, 1), 1), ((1, 1), (1, 1), 2), ((2, -1, 3), (1, 4, -2), 2),
    ((1, 2, 3, 4), (4, -3, 2, 1), 3), ((1, -1, 2, 0), (3, 1, 1, -2), 4), ((5,), (7,), 3),
])
def test_O19_exhaustive_equals_closed_form(x, y, m):
    mean, var = S.exhaustive_moments(x, y, m)
    xf, yf = [Fraction(v) for v in x], [Fraction(v) for v in y]
    ip = sum(a * b for a, b in zip(xf, yf))
    nx = sum(a * a for a in xf)
    ny = sum(b * b for b in yf)
    had = sum((a * b) ** 2 for a, b in zip(xf, yf))
    assert mean == ip
    assert var == (nx * ny + ip * ip - 2 * had) / m
    assert float(var) == pytest.approx(S.v_whole(x, y, m), rel=1e-15, abs=1e-15)


def test_worked_values():
    assert S.exhaustive_moments((1, 0), (0, 1), 1)[1] == 1
    assert S.exhaustive_moments((1, 1), (1, 1), 2)[1] == 2
    assert S.gms_estimate([3.0], [5.0], [0], [-1], 4) == 15.0          # n = 1


def test_O20_decomposition_identity_and_expressivity():
    rng = np.random.default_rng(20)
    xs = [rng.standard_normal(16) for _ in range(4)]
    ys = [rng.standard_normal(16) for _ in range(4)]
    m = 16
    whole = S.v_whole(np.concatenate(xs), np.concatenate(ys), m)
    assert S.v_gms_decomposed(xs, ys, m) == pytest.approx(whole, rel=1e-10)
    assert S.v_whole_pairs(np.concatenate(xs), np.concatenate(ys), m) == pytest.approx(whole, rel=1e-10)
    g, l = S.expressivity_log_count([2, 2], [2, 2], 4)
    assert g == pytest.approx(4 * math.log(4)) and l == pytest.approx(4 * math.log(2))
    assert round(g, 4) == 5.5452 and round(l, 4) == 2.7726 and g >= l


def test_O17_O18_monte_carlo_moments_random_family():
    rng = np.random.default_rng(17)
    k, n_l, m = 4, 16, 16
    for fixture in range(3):
        xs = [rng.standard_normal(n_l) for _ in range(k)]
        ys = [rng.standard_normal(n_l) for _ in range(k)]
        x, y = np.concatenate(xs), np.concatenate(ys)
        ip = float(x @ y)
        trials = 200000
        g = S.monte_carlo_random(x, y, m, trials, 100 + fixture)
        se = g.std() / np.sqrt(trials)
        assert abs(g.mean() - ip) <= 4 * se
        vG = S.v_whole(x, y, m)
        # SE of the sample variance from the 4th central moment
        c = g - g.mean()
        se_var = np.sqrt((np.mean(c ** 4) - np.mean(c ** 2) ** 2) / trials)
        assert abs(g.var() - vG) <= 3 * se_var
        # LMS: sum of per-piece GMS with m_l = f_l m = 4
        ms = S.lms_sizes([0.25] * 4, m)
        lsamp = sum(S.monte_carlo_random(xs[l], ys[l], ms[l], trials, 200 + 10 * fixture + l)
                    for l in range(k))
        se = lsamp.std() / np.sqrt(trials)
        assert abs(lsamp.mean() - ip) <= 4 * se
        vL = S.v_lms(xs, ys, ms)
        c = lsamp - lsamp.mean()
        se_var = np.sqrt((np.mean(c ** 4) - np.mean(c ** 2) ** 2) / trials)
        assert abs(lsamp.var() - vL) <= 3 * se_var


def test_monte_carlo_appendix_a_family():
    """The implemented polynomial family reproduces Theorem 1's moments too."""
    rng = np.random.default_rng(18)
    x, y = rng.standard_normal(12), rng.standard_normal(12)
    m, trials = 8, 6000
    g = S.monte_carlo_family(x, y, m, trials, 0x5EED)
    se = g.std() / np.sqrt(trials)
    assert abs(g.mean() - x @ y) <= 4 * se
    c = g - g.mean()
    se_var = np.sqrt((np.mean(c ** 4) - np.mean(c ** 2) ** 2) / trials)
    assert abs(g.var() - S.v_whole(x, y, m)) <= 3 * se_var
