"""Oracle feature-hashing estimator lab (GMS vs LMS, Theorem 1) — TEST INFRASTRUCTURE ONLY.

Chunk size 1, alignment 1 ("using a chunk size of one").

    GMS:  <x,y>^_G,m = sum_{j<m} (sum_i [h(i)=j] g(i) x_i) (sum_i [h(i)=j] g(i) y_i)
    LMS:  <x,y>^_L   = sum_l <x_l, y_l>^_G,(f_l m)
    E = <x, y> for both
    V(whole) = (1/m) (sum_{i!=j} x_i^2 y_j^2 + sum_{i!=j} x_i y_i x_j y_j)
             = (1/m) (|x|^2 |y|^2 + <x,y>^2 - 2 |x o y|^2)
    V_l      = 1/(f_l m) (sum_{i!=j} a_i^2 b_j^2 + sum_{i!=j} a_i b_i a_j b_j)
    V_L      = sum_l V_l
    V_G      = sum_l f_l V_l + (1/m) sum_{l1!=l2} (|x_l1|^2 |y_l2|^2 + <x_l1,y_l1><x_l2,y_l2>)
                                                   (P:370 / P:649, typo-corrected per R13)
    expressivity: GMS |M|^n vs LMS prod |M_i|^{n_i}

Pinned by tests/test_oracle_estimator.py: exhaustive enumeration of every
(h, g) assignment for n, m <= 4 equals the closed form exactly in rational
arithmetic; Monte Carlo unbiasedness within 4 SE and variance within 3 SE;
the worked values x=(1,0), y=(0,1), m=1 -> V=1 and a=b=(1,1), m=2 -> V=2
(S:324); n=1 -> estimate x0 y0 exactly; decomposition == whole
form; expressivity n=(2,2), m=4.
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np

from . import hashing


def gms_estimate(x, y, h, g, m):
    """Literal P:357: bucket sums of g*x and g*y, then their dot product."""
    bx = [0.0] * m
    by = [0.0] * m
    for i in range(len(x)):
        bx[h[i]] += g[i] * x[i]
        by[h[i]] += g[i] * y[i]
    return sum(bx[j] * by[j] for j in range(m))


def lms_sizes(fractions, m):
    """m_l = floor(f_l m), remainder to the last piece (R14)."""
    ms = [int(math.floor(f * m)) for f in fractions]
    ms[-1] += m - sum(ms)
    return ms


def lms_estimate(xs, ys, hs, gs, ms):
    """sum over pieces of the GMS estimator in each piece's own memory."""
    return sum(gms_estimate(xs[l], ys[l], hs[l], gs[l], ms[l]) for l in range(len(xs)))


def v_whole(x, y, m):
    """Closed form: (|x|^2|y|^2 + <x,y>^2 - 2|x o y|^2) / m."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    return (x @ x * (y @ y) + (x @ y) ** 2 - 2.0 * np.sum((x * y) ** 2)) / m


def v_whole_pairs(x, y, m):
    """The pair-sum form, term by term."""
    n = len(x)
    s = 0.0
    for i in range(n):
        for j in range(n):
            if i != j:
                s += x[i] ** 2 * y[j] ** 2 + x[i] * y[i] * x[j] * y[j]
    return s / m


def v_piece(a, b, m_l):
    """V_l with the piece's own memory size m_l = f_l m."""
    return v_whole_pairs(a, b, 1) / m_l


def v_lms(xs, ys, ms):
    return sum(v_piece(xs[l], ys[l], ms[l]) for l in range(len(xs)))


def v_gms_decomposed(xs, ys, m):
    """Theorem 1's piece form of V_G (R13): within-piece + cross-piece terms."""
    k = len(xs)
    within = sum(v_whole_pairs(xs[l], ys[l], 1) for l in range(k)) / m
    cross = 0.0
    for l1 in range(k):
        for l2 in range(k):
            if l1 != l2:
                cross += (np.dot(xs[l1], xs[l1]) * np.dot(ys[l2], ys[l2])
                          + np.dot(xs[l1], ys[l1]) * np.dot(xs[l2], ys[l2]))
    return within + cross / m


def exhaustive_moments(x, y, m):
    """Exact mean and variance over ALL m^n hash maps and 2^n sign maps (Fractions)."""
    n = len(x)
    xf = [Fraction(v) for v in x]
    yf = [Fraction(v) for v in y]
    total = Fraction(0)
    total_sq = Fraction(0)
    count = 0
    for h in itertools.product(range(m), repeat=n):
        for g in itertools.product((1, -1), repeat=n):
            e = gms_estimate(xf, yf, h, g, m)
            total += e
            total_sq += e * e
            count += 1
    mean = total / count
    return mean, total_sq / count - mean * mean


def monte_carlo_random(x, y, m, trials, seed):
    """Estimator samples with fully random h, g (numpy Generator), vectorised over trials."""
    rng = np.random.default_rng(seed)
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    n = len(x)
    out = np.empty(trials)
    chunk = 20000
    for s in range(0, trials, chunk):
        t = min(chunk, trials - s)
        h = rng.integers(0, m, size=(t, n))
        g = rng.integers(0, 2, size=(t, n)) * 2.0 - 1.0
        bx = np.zeros((t, m))
        by = np.zeros((t, m))
        rows = np.repeat(np.arange(t), n)
        np.add.at(bx, (rows, h.ravel()), (g * x).ravel())
        np.add.at(by, (rows, h.ravel()), (g * y).ravel())
        out[s:s + t] = np.sum(bx * by, axis=1)
    return out


def monte_carlo_family(x, y, m, trials, master_seed):
    """Estimator samples with the Appendix-A family (A = 1, T = 1, R = m); seed = mix(master, trial)."""
    n = len(x)
    out = np.empty(trials)
    for t in range(trials):
        seed = hashing.splitmix64(master_seed ^ (t * 0x100000001B3))
        mh = hashing.ModuleHash(seed, 0, m, 1, 1, True)
        h = [mh.offset(i) for i in range(n)]
        g = [mh.sign(i) for i in range(n)]
        out[t] = gms_estimate(x, y, h, g, m)
    return out


def expressivity_log_count(ns, ms_local, m):
    """(n ln m, sum_i n_i ln |M_i|): log-counts of expressible functions."""
    return sum(ns) * math.log(m), sum(n * math.log(mi) for n, mi in zip(ns, ms_local))
