"""Pins for oracle/optim.py (no GPU)."""
import numpy as np

from oracle import optim as O


def test_sgd_on_quadratic_closed_form():
    # f(M) = 0.5 |M - c|^2 -> grad M - c; one step: M - lr (M - c)
    rng = np.random.default_rng(1)
    M, c = rng.standard_normal(100), rng.standard_normal(100)
    Mn, _ = O.step("sgd", M, M - c, {}, lr=0.25)
    assert np.allclose(Mn, 0.75 * M + 0.25 * c, rtol=0, atol=1e-15)


def test_adam_first_step_is_lr_sign():
    rng = np.random.default_rng(2)
    M, g = rng.standard_normal(1000), rng.standard_normal(1000)
    Mn, st = O.step("adam", M, g, {}, lr=1e-3, t=1, eps=0.0)
    assert np.allclose(M - Mn, 1e-3 * np.sign(g), rtol=0, atol=1e-15)
    assert np.allclose(st["m"], 0.1 * g) and np.allclose(st["v"], 0.001 * g * g)


def test_adagrad_first_step():
    rng = np.random.default_rng(3)
    M, g = rng.standard_normal(1000), rng.standard_normal(1000)
    Mn, st = O.step("adagrad", M, g, {}, lr=0.1, eps=1e-10)
    assert np.allclose(M - Mn, 0.1 * g / (np.abs(g) + 1e-10), rtol=1e-12)
    assert np.array_equal(st["G"], g * g)


def test_weight_decay_enters_the_gradient():
    M, g = np.array([2.0, -4.0]), np.array([0.0, 0.0])
    Mn, _ = O.step("sgd", M, g, {}, lr=0.5, wd=0.1)
    assert np.allclose(Mn, M - 0.5 * 0.1 * M)
