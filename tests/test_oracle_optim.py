"""Pins for oracle/optim.py (no GPU)."""
import numpy as np
import pytest

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


# ---- multi-step recurrences with carried state (t >= 2) --------------------------------
# The values below are worked by hand from the update rules the paper's training uses
# (PyTorch SGD / Adagrad / Adam), in exact rationals, for a scalar
# gradient sequence g = (1, -2, 3), so a dropped decay term (b1 m_prev, b2 v_prev), an
# Adagrad accumulator that does not carry G across steps, or a bias correction that uses
# the wrong t would each change the third step.
import math  # noqa: E402


def _run(kind, gs, **kw):
    M, st = np.array([0.0]), {}
    out = []
    for t, g in enumerate(gs, start=1):
        M, st = O.step(kind, M, np.array([float(g)]), st, t=t, **kw)
        out.append(float(M[0]))
    return out, st


def test_adam_three_steps_hand_derived():
    # b1 = 1/2, b2 = 3/4, lr = 1, eps = 0:
    #  t=1: m = 1/2,  v = 1/4,   m^ = 1,   v^ = 1      -> M = -1
    #  t=2: m = -3/4, v = 19/16, m^ = -1,  v^ = 19/7   -> M = -1 + sqrt(7/19)
    #  t=3: m = 9/8,  v = 201/64, m^ = 9/7, v^ = 201/37 -> M -= (9/7) sqrt(37/201)
    got, st = _run("adam", [1, -2, 3], lr=1.0, b1=0.5, b2=0.75, eps=0.0)
    m1 = -1.0
    m2 = m1 + math.sqrt(7 / 19)
    m3 = m2 - (9 / 7) * math.sqrt(37 / 201)
    assert np.allclose(got, [m1, m2, m3], rtol=0, atol=1e-14)
    assert math.isclose(st["m"][0], 9 / 8, abs_tol=1e-15) and math.isclose(st["v"][0], 201 / 64, abs_tol=1e-15)


def test_adagrad_three_steps_hand_derived():
    # lr = 1, eps = 0: G = 1, 5, 14; steps g / sqrt(G) = 1, -2/sqrt(5), 3/sqrt(14)
    got, st = _run("adagrad", [1, -2, 3], lr=1.0, eps=0.0)
    e1 = -1.0
    e2 = e1 + 2 / math.sqrt(5)
    e3 = e2 - 3 / math.sqrt(14)
    assert np.allclose(got, [e1, e2, e3], rtol=0, atol=1e-14)
    assert st["G"][0] == 14.0


def test_adagrad_constant_gradient_closed_form():
    # constant g: G_t = t g^2, so M_t = M_0 - lr sign(g) sum_{s<=t} 1/sqrt(s)  (eps = 0)
    got, _ = _run("adagrad", [-0.5] * 6, lr=0.1, eps=0.0)
    ref = [0.1 * sum(1 / math.sqrt(s) for s in range(1, t + 1)) for t in range(1, 7)]
    assert np.allclose(got, ref, rtol=1e-14, atol=0)


def test_sgd_three_steps_on_quadratic_closed_form():
    # f = 1/2 (M - c)^2: M_t - c = (1 - lr)^t (M_0 - c); the gradient is taken at each new M
    c, lr, M = 3.0, 0.25, np.array([1.0])
    for t in range(1, 4):
        M, _ = O.step("sgd", M, M - c, {}, lr=lr, t=t)
        assert math.isclose(M[0] - c, (1 - lr) ** t * (1.0 - c), rel_tol=1e-15)


@pytest.mark.parametrize("kind", ["sgd", "adagrad", "adam"])
def test_matches_torch_optim_over_five_steps(kind):
    """A library routine as the second, independent implementation: torch.optim (CPU, fp64)
    on the same parameter vector and gradient sequence, weight decay included."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(17)
    M0 = rng.standard_normal(257)
    gs = [rng.standard_normal(257) for _ in range(5)]
    kw = dict(lr=3e-2, weight_decay=0.01)
    p = torch.nn.Parameter(torch.tensor(M0, dtype=torch.float64))
    if kind == "sgd":
        opt = torch.optim.SGD([p], **kw)
    elif kind == "adagrad":
        opt = torch.optim.Adagrad([p], eps=1e-10, **kw)
    else:
        opt = torch.optim.Adam([p], betas=(0.9, 0.999), eps=1e-8, **kw)
    M, st = M0.copy(), {}
    for t, g in enumerate(gs, start=1):
        p.grad = torch.tensor(g, dtype=torch.float64)
        opt.step()
        extra = dict(eps=1e-10) if kind == "adagrad" else dict(eps=1e-8) if kind == "adam" else {}
        M, st = O.step(kind, M, g, st, lr=3e-2, t=t, wd=0.01, **extra)
        assert np.allclose(M, p.detach().numpy(), rtol=1e-13, atol=1e-15), (kind, t)
