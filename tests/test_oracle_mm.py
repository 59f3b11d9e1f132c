"""Pins for oracle/roast_mm.py (no GPU).  SURVEY.md §8(c) tests O10-O15, O21."""
import numpy as np
import pytest

import synth
from oracle import roast_mm as RM


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb else 1.0)


def test_O10_identity_mapping_equals_dense_reshape():
    """North star: |M| >= n, identity mapping, Z2 = O  ->  W = reshape(M[:H*O], H, O)."""
    H, O, T = 96, 40, 16          # H != O catches a transposed operand
    M = synth.uniform(1, (H * O + 24,))
    spec = RM.LinearSpec(H, O, 8, O, len(M), 0, 0, mapping=RM.IDENTITY, use_sign=False)
    Wd = M[:H * O].reshape(H, O)
    X = synth.uniform(2, (T, H))
    dY = synth.uniform(3, (T, O))
    assert np.array_equal(spec.materialize(M), Wd)
    assert np.array_equal(spec.forward(X, M), X @ Wd)
    assert np.array_equal(spec.backward_dx(dY, M), dY @ Wd.T)
    dM = spec.backward_dm(X, dY)
    assert np.array_equal(dM[:H * O], (X.T @ dY).ravel())
    assert np.all(dM[H * O:] == 0)


def test_identity_blocked_tiles_equal_block_reshape():
    """Identity mapping with Z1 != Z2 and Z2 < O: tile (x, y) is the (x, y) block of a
    block-major rearrangement of M; rebuild W with np.block from independent reshapes."""
    H, O, z1, z2 = 24, 32, 8, 16
    M = synth.uniform(4, (H * O,))
    spec = RM.LinearSpec(H, O, z1, z2, len(M), 0, 0, mapping=RM.IDENTITY, use_sign=False)
    ny = O // z2
    blocks = [[M[(x * ny + y) * z1 * z2:(x * ny + y + 1) * z1 * z2].reshape(z1, z2)
               for y in range(ny)] for x in range(H // z1)]
    assert np.array_equal(spec.materialize(M), np.block(blocks))


def test_O11_X_identity_and_zero_store():
    H = O = 64
    M = synth.uniform(1, (1000,))
    spec = RM.LinearSpec(H, O, 16, 16, len(M), 0x5EED, 0)
    X = np.eye(H)
    assert np.array_equal(spec.forward(X, M), spec.materialize(M))
    Z = np.zeros_like(M)
    dY = synth.uniform(3, (H, O))
    assert np.all(spec.forward(X, Z) == 0)
    assert np.all(spec.backward_dx(dY, Z) == 0)
    assert np.all(spec.backward_dm(X, np.zeros((H, O))) == 0)


def test_single_tile_covering_W():
    """Z1 >= H, Z2 >= O: dM = lambda g vec(X^T dY) at the one hashed offset."""
    H, O = 16, 8
    M = synth.uniform(1, (200,))
    spec = RM.LinearSpec(H, O, H, O, len(M), 0x5EED, 2)
    X = synth.uniform(2, (5, H))
    dY = synth.uniform(3, (5, O))
    off, g = int(spec.off[0, 0]), int(spec.sgn[0, 0])
    dM = spec.backward_dm(X, dY)
    expect = np.zeros(len(M))
    expect[off:off + H * O] = spec.lam * g * (X.T @ dY).ravel()
    assert rel(dM, expect) < 1e-15
    W = spec.materialize(M)
    assert np.array_equal(W, g * spec.lam * M[off:off + H * O].reshape(H, O))


def test_O12_adjoint_identities():
    rng = np.random.default_rng(12)
    for trial in range(25):
        z1, z2 = int(rng.choice([4, 8, 16])), int(rng.choice([4, 8, 16]))
        H = z1 * int(rng.integers(1, 5))
        O = z2 * int(rng.integers(1, 5))
        m = int(rng.integers(z1 * z2, z1 * z2 * 3)) // 8 * 8 + 8
        spec = RM.LinearSpec(H, O, z1, z2, m, 1234 + trial, trial % 3)
        M = rng.uniform(-1, 1, m)
        X = rng.standard_normal((7, H))
        G = rng.standard_normal((7, O))
        lhs = np.sum(G * spec.forward(X, M))
        rhs = M @ spec.backward_dm(X, G)
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))
        lhs2 = np.sum(G * spec.forward(X, M))
        rhs2 = np.sum(X * spec.backward_dx(G, M))
        assert abs(lhs2 - rhs2) <= 1e-10 * max(1.0, abs(lhs2))


def _two_layer_model(M_len=40):
    a = RM.LinearSpec(16, 16, 4, 4, M_len, 0x5EED, 0)
    b = RM.LinearSpec(16, 16, 4, 4, M_len, 0x5EED, 1)
    return a, b


def test_O13_finite_differences_every_slot():
    """Two linears sharing one tiny M (R = 4, every tile overlaps); L is linear in M,
    so central differences are exact up to rounding."""
    a, b = _two_layer_model()
    assert a.off.max() < 40 and len(np.unique(a.off)) > 1
    M = synth.uniform(1, (40,))
    X1 = synth.uniform(2, (4, 16))
    X2 = synth.uniform(5, (4, 16))
    G1 = synth.uniform(3, (4, 16))
    G2 = synth.uniform(6, (4, 16))

    def loss(Mv):
        return np.sum(G1 * a.forward(X1, Mv)) + np.sum(G2 * b.forward(X2, Mv))

    dM = a.backward_dm(X1, G1)
    dM = b.backward_dm(X2, G2, dM)
    eps = 1e-3
    fd = np.empty(40)
    for s in range(40):
        e = np.zeros(40)
        e[s] = eps
        fd[s] = (loss(M + e) - loss(M - e)) / (2 * eps)
    assert np.max(np.abs(fd - dM)) <= 1e-8 * np.max(np.abs(dM))


def test_O14_shared_slot_sum_of_partials():
    a, b = _two_layer_model()
    rng = np.random.default_rng(14)
    X1, X2 = rng.integers(-3, 4, (4, 16)), rng.integers(-3, 4, (4, 16))
    G1, G2 = rng.integers(-3, 4, (4, 16)), rng.integers(-3, 4, (4, 16))
    only1 = a.backward_dm(X1, G1)
    only2 = b.backward_dm(X2, G2)
    both = b.backward_dm(X2, G2, a.backward_dm(X1, G1))
    # small integers * lambda (0.25, a power of two): every sum is exact in fp64
    assert np.array_equal(both, only1 + only2)


def test_O15_collision_example():
    """two weights on one slot, grad 1 each, lambda = 0.5, g = +1 -> slot grad 1.0."""
    spec = RM.LinearSpec(1, 2, 1, 1, 1, 0, 0, align=1, use_sign=False, lam=0.5)
    assert spec.off.tolist() == [[0, 0]]
    dM = spec.backward_dm(np.array([[1.0]]), np.array([[1.0, 1.0]]))
    assert dM.tolist() == [1.0]


def test_O21_padding_invariance():
    H, O, z = 33, 70, 16
    M = synth.uniform(1, (2000,))
    spec = RM.LinearSpec(H, O, z, z, len(M), 0x5EED, 0)
    pad = RM.LinearSpec(48, 80, z, z, len(M), 0x5EED, 0, lam=spec.lam)   # same module, same fan-in
    X = synth.uniform(2, (9, H))
    Xp = np.zeros((9, 48))
    Xp[:, :H] = X
    assert np.allclose(pad.forward(Xp, M)[:, :O], spec.forward(X, M), rtol=0, atol=1e-14)
    assert np.array_equal(pad.materialize(M)[:H, :O], spec.materialize(M))


def test_fp32_recovered_weight_definition():
    """g * fp32(lambda32 * M32): compare against numpy float32 multiplication (IEEE RNE)."""
    H = O = 64
    M = synth.uniform(1, (5000,)).astype(np.float32)
    spec = RM.LinearSpec(H, O, 32, 32, len(M), 0x5EED, 0)
    W32 = spec.materialize(M, "fp32")
    slot = spec.slot_index()
    ref = spec.sign_matrix() * (np.float32(spec.lam) * M[slot]).astype(np.float64)
    assert np.array_equal(W32, ref)


def test_bf16_operand_definition():
    H = O = 64
    M = synth.uniform(1, (5000,)).astype(np.float32)
    spec = RM.LinearSpec(H, O, 64, 64, len(M), 0x5EED, 0)
    Wop = spec.materialize(M, "operand")
    ref = spec.sign_matrix() * synth.round_to_bf16(M)[spec.slot_index()]
    assert np.array_equal(Wop, ref)


def test_sw128_layout_is_tilewise_bijection():
    T = 64 * 64
    pos = {RM.pi(o1, o2, 64, RM.SW128) for o1 in range(64) for o2 in range(64)}
    assert pos == set(range(T))
    # rows stay rows: element (o1, *) lives in [64 o1, 64 o1 + 64)
    assert all(64 * o1 <= RM.pi(o1, o2, 64, RM.SW128) < 64 * o1 + 64
               for o1 in range(64) for o2 in range(64))


def test_grad_slot_matches_full_scatter():
    spec = RM.LinearSpec(64, 128, 64, 64, 4720, 0x5EED, 0)
    X = synth.normal(2, (32, 64))
    dY = synth.normal(3, (32, 128))
    full = spec.backward_dm(X, dY)
    for s in [0, 7, 100, 1000, 4095, 4600, 4719]:
        assert abs(spec.grad_slot(X, dY, s) - full[s]) <= 1e-12 * max(1, abs(full[s]))
