"""Pins for oracle/embedding.py (no GPU).  SURVEY.md §8(c) test O16."""
import numpy as np
import pytest

import synth
from oracle import embedding as E


def test_single_row_store_equals_lambda_g_M():
    """m = row_len = Z: one chunk, offset forced to 0 -> out = lambda g M."""
    d = 32
    M = synth.uniform(1, (d,)).astype(np.float32)
    spec = E.EmbeddingSpec(1, d, d, d, 0x5EED, 0)
    off, sgn = spec.chunk_map([0])
    assert off.tolist() == [[0]]
    out = spec.forward([0], M)
    assert np.array_equal(out[0], sgn[0, 0] * (np.float32(spec.lam) * M).astype(np.float64))


def test_zero_store_and_bounds():
    spec = E.EmbeddingSpec(100, 16, 8, 256, 1, 0)
    assert np.all(spec.forward([3, 4, 99], np.zeros(256)) == 0)
    with pytest.raises(IndexError):
        spec.forward([100], np.zeros(256))


def test_linearity_and_adjoint():
    rng = np.random.default_rng(3)
    spec = E.EmbeddingSpec(1000, 64, 16, 256, 7, 2)
    rows = rng.integers(0, 1000, 50)
    v1, v2 = rng.standard_normal(256), rng.standard_normal(256)
    f = lambda v: spec.forward(rows, v, "exact")
    assert np.allclose(f(2 * v1 - 3 * v2), 2 * f(v1) - 3 * f(v2), rtol=0, atol=1e-12)
    G = rng.standard_normal((50, 64))
    lhs = np.sum(G * f(v1))
    rhs = v1 @ spec.backward(rows, G)
    assert abs(lhs - rhs) <= 1e-10 * max(1, abs(lhs))


def test_finite_differences_every_slot_with_duplicates():
    spec = E.EmbeddingSpec(10, 12, 4, 24, 0x5EED, 1)          # d not a multiple of Z? 12 = 3*4
    rows = [1, 3, 3, 9, 1]                                      # duplicates accumulate
    M = synth.uniform(1, (24,))
    G = synth.uniform(3, (5, 12))
    loss = lambda v: np.sum(G * spec.forward(rows, v, "exact"))
    dM = spec.backward(rows, G)
    eps = 1e-3
    fd = np.array([(loss(M + eps * np.eye(24)[s]) - loss(M - eps * np.eye(24)[s])) / (2 * eps)
                   for s in range(24)])
    assert np.max(np.abs(fd - dM)) <= 1e-8 * np.max(np.abs(dM))


def test_collision_example():
    """S:190 for L: two elements on one slot, grad 1 each, lambda 0.5, g = +1 -> 1.0."""
    spec = E.EmbeddingSpec(2, 1, 1, 1, 0, 0, align=1, C=1.0, fan_in=4, use_sign=False)
    dM = spec.backward([0, 1], np.ones((2, 1)))
    assert spec.lam == 0.5 and dM.tolist() == [1.0]


def test_padded_row_chunks():
    """d = 10, Z = 4: rows padded to 12 (R16): 3 chunks per row, last chunk uses 2 elements."""
    spec = E.EmbeddingSpec(5, 10, 4, 64, 3, 0)
    assert spec.chunks_per_row == 3
    M = synth.uniform(1, (64,)).astype(np.float32)
    out = spec.forward([2], M)
    off, sgn = spec.chunk_map([2])
    for k in range(10):
        j, o = divmod(k, 4)
        assert out[0, k] == sgn[0, j] * float(np.float32(spec.lam) * M[off[0, j] + o])
