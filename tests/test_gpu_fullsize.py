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


@pytest.mark.parametrize("dist,align", [("uniform", 32), ("zipf", 32), ("zipf", 8)])
def test_c4_full_size(R, torch, dist, align):
    """C4 at its real size in the bench's launch configuration (26 tables x 10^7 rows, dim 128,
    chunk 32, 1000x, 65 536 lookups per table, all tables in one launch): sampled forward rows
    bit-exact against the oracle; the backward through the adjoint identity that holds at any
    size, <dOut, L(M)> = <M, dM(dOut)> (L is linear in M, P:268-276 / P:338-341), in fp64."""
    from oracle import embedding as OE
    tables, rows, dim, Z, batch = 26, 10 ** 7, 128, 32, 65536
    mem = synth.compressed_size(tables * rows * dim, 1000, align=align)
    M_np = synth.uniform(synth.SEED_M, (mem,)).astype(np.float32)
    M = to_dev(M_np, torch.float32)
    ctx = R.Roast(M, 64, 64, seed=HS, align=align)
    mids = [ctx.embedding(rows, dim, Z) for _ in range(tables)]
    gen = synth.uniform_indices if dist == "uniform" else synth.zipf_indices
    idx_np = np.stack([gen(synth.SEED_IDX + t, batch, rows) for t in range(tables)])
    idx = to_dev(idx_np, torch.int64)
    out = ctx.emb_fwd_multi(mids, idx)
    torch.cuda.synchronize()
    M64 = M_np.astype(np.float64)
    rng = np.random.default_rng(5)
    for t, b in zip(rng.integers(0, tables, 48), rng.integers(0, batch, 48)):
        spec = OE.EmbeddingSpec(rows, dim, Z, mem, HS, mids[t], align=align)
        ref = spec.forward(idx_np[t, b:b + 1], M64)
        assert np.array_equal(out[t * batch + b].cpu().numpy().astype(np.float64), ref[0]), (t, b)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    dout = torch.randn(tables * batch, dim, device="cuda", generator=g)
    ctx.zero_grad()
    ctx.emb_bwd_multi(mids, idx, dout)
    torch.cuda.synchronize()
    lhs = float((dout.double() * out.double()).sum())
    rhs = float((ctx.M.double() * ctx.dM.double()).sum())
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs), (lhs, rhs)
    ctx.check()
    ctx.close()


@pytest.mark.parametrize("dist,align,deterministic", [("uniform", 32, False), ("zipf", 32, False),
                                                      ("zipf", 32, True), ("uniform", 8, True)])
def test_c4_full_size_backward_element_by_element(R, torch, dist, align, deterministic):
    """C4's backward at full size, element by element: the launch is the bench's (26 tables x
    65 536 lookups, all tables in one call), but dOut is non-zero only for two tables, so every
    slot of dM has an oracle value the oracle can compute (the L rule, over those
    two tables' 131 072 lookups; duplicates add, R15).  Deterministic mode: bitwise identical
    over 3 runs as well."""
    from oracle import embedding as OE
    tables, rows, dim, Z, batch = 26, 10 ** 7, 128, 32, 65536
    mem = synth.compressed_size(tables * rows * dim, 1000, align=align)
    M_np = synth.uniform(synth.SEED_M, (mem,)).astype(np.float32)
    ctx = R.Roast(to_dev(M_np, torch.float32), 64, 64, seed=HS, align=align, deterministic=deterministic)
    mids = [ctx.embedding(rows, dim, Z) for _ in range(tables)]
    gen = synth.uniform_indices if dist == "uniform" else synth.zipf_indices
    idx_np = np.stack([gen(synth.SEED_IDX + t, batch, rows) for t in range(tables)])
    live = (3, 17)
    dout_np = np.zeros((tables, batch, dim), np.float32)
    for t in live:
        dout_np[t] = synth.normal(synth.SEED_DY + t, (batch, dim)).astype(np.float32)
    idx, dout = to_dev(idx_np, torch.int64), to_dev(dout_np.reshape(-1, dim), torch.float32)
    runs = []
    for _ in range(3 if deterministic else 1):
        ctx.zero_grad()
        ctx.emb_bwd_multi(mids, idx, dout)
        torch.cuda.synchronize()
        runs.append(ctx.dM.cpu().numpy())
    ctx.check()
    for r in runs[1:]:
        assert np.array_equal(r, runs[0])
    ref = np.zeros(mem)
    for t in live:
        OE.EmbeddingSpec(rows, dim, Z, mem, HS, mids[t], align=align).backward(idx_np[t], dout_np[t], ref)
    got = runs[0].astype(np.float64)
    assert rel_frob(got, ref) <= 1e-5
    # element by element: fp32 sums of at most a few hundred terms (Zipf-hot rows) of N(0, 1)
    scale = np.abs(ref).max()
    assert np.max(np.abs(got - ref)) <= 1e-5 * scale
    assert np.all(got[ref == 0] == 0)     # slots no live lookup reaches stay exactly zero
    ctx.close()
