"""Full-size parity on sampled outputs (BASELINE.json configs at their real sizes, in the
launch configuration bench.py times: tcgen05 path, atomic dM).  The oracle computes the
sampled outputs one by one: Y / dX rows are independent; a dM slot is the sum over the
(i, j) that map to it (oracle LinearSpec.grad_slot)."""
import numpy as np
import pytest

import synth
from oracle import roast_mm as OM
from tests.gpu_helpers import rel_frob, to_dev

pytestmark = pytest.mark.gpu
HS = synth.HASH_SEED


def _layer_check(R, torch, H, O, T, mem, z=64, n_rows=48, n_slots=24, tol=1e-2, seed_off=0):
    M_np = synth.uniform(synth.SEED_M, (mem,)).astype(np.float32)
    M = to_dev(M_np, torch.float32)
    ctx = R.Roast(M, z, z, seed=HS)
    mid = ctx.linear(H, O)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7 + seed_off)
    X = torch.randn(T, H, device="cuda", generator=gen).to(torch.bfloat16)
    dY = torch.randn(T, O, device="cuda", generator=gen).to(torch.bfloat16)
    ctx.zero_grad()
    Y = ctx.fwd(mid, X)
    dX = ctx.bwd(mid, X, dY)
    torch.cuda.synchronize()
    spec = OM.LinearSpec(H, O, z, z, mem, HS, mid)
    rng = np.random.default_rng(11 + seed_off)
    rows = np.unique(np.concatenate([rng.integers(0, T, n_rows), [0, T - 1]]))
    Xr = X[rows].float().cpu().numpy()
    dYr = dY[rows].float().cpu().numpy()
    Wop = np.float64(spec.lam) * spec.materialize(M_np, "operand")
    assert rel_frob(Y[rows].float().cpu().numpy(), Xr @ Wop) <= tol
    assert rel_frob(dX[rows].float().cpu().numpy(), dYr @ Wop.T) <= tol
    # dM on slots that some tile covers (first element, last element, random interior)
    Xf = X.float().cpu().numpy().astype(np.float64)
    dYf = dY.float().cpu().numpy().astype(np.float64)
    dM = ctx.dM.cpu().numpy()
    offs = spec.off.ravel()
    pick = rng.choice(len(offs), size=min(n_slots, len(offs)), replace=False)
    slots = sorted({int(offs[t] + e) for t in pick for e in (0, z * z - 1, int(rng.integers(0, z * z)))})
    got = np.array([dM[s] for s in slots])
    ref = np.array([spec.grad_slot(Xf, dYf, s) for s in slots])
    assert rel_frob(got, ref) <= tol
    ctx.close()


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


@pytest.fixture(scope="module")
def R():
    from paper_2207_10702_b200 import roast
    return roast


@pytest.mark.parametrize("ratio", [10, 100, 1000])
def test_c2_full_size_sampled(R, torch, ratio):
    cfg = synth.mlp_block(ratio)
    for i, (H, O) in enumerate(cfg["layers"]):
        _layer_check(R, torch, H, O, cfg["tokens"], cfg["mem_size"], seed_off=i)


@pytest.mark.parametrize("mem_mb", [8, 2048])
def test_c5_sweep_endpoints_sampled(R, torch, mem_mb):
    """C5: 4096 x 4096 at batch 16384, |M| from L2-resident (8 MB) to HBM-resident (2 GB)."""
    mem = mem_mb * 1024 * 1024 // 4
    _layer_check(R, torch, 4096, 4096, 16384, mem, n_rows=24, n_slots=16)
