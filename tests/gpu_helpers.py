"""Shared helpers for the -m gpu parity tests: build inputs with synth, move them to the GPU."""
import numpy as np

import synth


def rel_frob(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    if nb == 0:
        return float(np.linalg.norm(a))
    return float(np.linalg.norm(a - b) / nb)


def to_dev(a, dtype):
    import torch
    return torch.tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def bf16_input(seed, shape, dist="normal"):
    """bf16-valued fp32 numpy array (R18: rounded once, both sides consume it)."""
    x = synth.normal(seed, shape) if dist == "normal" else synth.uniform(seed, shape)
    return synth.round_to_bf16(x.astype(np.float32))


def store(mem_size, seed=synth.SEED_M):
    """M ~ U(-1, 1) (C = 1) as fp32."""
    return synth.uniform(seed, (mem_size,)).astype(np.float32)


def grad_condition(dM, M_prev, wd, dM_abs=None):
    """Condition number of the decayed gradient g = dM + wd M: (|dM| + |wd M|) / |g|.  Where dM
    nearly cancels wd M, an fp32 kernel's g carries a relative error ~ cond * 2^-24 that the
    update inherits (Adagrad / Adam divide by ~|g|), so such elements cannot be held to an
    element-wise 1e-5 — check_update exempts them from (b); (a) still covers them.  dM_abs:
    sum of |terms| when dM is itself an fp32 sum (the ranks' gradients)."""
    dM = np.asarray(dM, dtype=np.float64)
    wm = wd * np.asarray(M_prev, dtype=np.float64)
    g = dM + wm
    with np.errstate(divide="ignore", invalid="ignore"):
        a = np.abs(dM) if dM_abs is None else np.asarray(dM_abs, dtype=np.float64)
        return np.where(g != 0, (a + np.abs(wm)) / np.abs(g), np.inf)


def check_update(M_prev, got, ref_new, tol=1e-5, cond=None):
    """The optimizer's UPDATE, not just the new value: M ~ 1 and a step ~ lr, so comparing M
    alone would check the update only to ~ulp(M) / lr.  Asserts (a) the update dM_got = got -
    M_prev against the oracle's dM_ref = ref_new - M_prev at relative Frobenius <= tol, and (b)
    element by element |got - ref_new| <= ulp32(ref_new) / 2 + tol (|dM_ref| + rms(dM_ref) / 10):
    the update is right to tol, up to the one unavoidable fp32 rounding of the stored M (the
    rms term covers elements whose step nearly cancels, e.g. Adam's m ~ 0, where the kernel's
    fp32 state arithmetic has absolute, not relative, error)."""
    M_prev = np.asarray(M_prev, dtype=np.float64)
    got = np.asarray(got, dtype=np.float64)
    ref_new = np.asarray(ref_new, dtype=np.float64)
    d_got, d_ref = got - M_prev, ref_new - M_prev
    assert rel_frob(d_got, d_ref) <= tol, rel_frob(d_got, d_ref)
    half_ulp = 0.5 * np.spacing(np.abs(ref_new).astype(np.float32)).astype(np.float64)
    rms = float(np.sqrt(np.mean(d_ref * d_ref))) if d_ref.size else 0.0
    bad = np.abs(got - ref_new) > half_ulp + tol * (np.abs(d_ref) + 0.1 * rms) + 1e-30
    if cond is not None:                 # ill-conditioned g (grad_condition > 1e3): (a) only
        bad &= np.asarray(cond) <= 1e3
    assert not bad.any(), (int(bad.sum()), np.flatnonzero(bad)[:5])
