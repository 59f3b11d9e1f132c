"""GELU fused into the tcgen05 GEMM epilogues (roast_linear_fwd_act / roast_linear_bwd_dx_act,
include/roast.h): against the fp64 oracle ROAST-MM composed with the tanh-form GELU (the
activation is an N-op of the BERT workload; the linear is the paper's, P:294-313 / P:338-346)."""
import numpy as np
import pytest

import synth
from oracle import roast_mm as OM
from tests.gpu_helpers import bf16_input, rel_frob, store, to_dev

pytestmark = pytest.mark.gpu
HS = synth.HASH_SEED


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


@pytest.fixture(scope="module")
def R():
    from paper_2207_10702_b200 import roast
    return roast


def gelu(x):
    return 0.5 * x * (1 + np.tanh(np.sqrt(2 / np.pi) * (x + 0.044715 * x ** 3)))


def gelu_grad(x):
    t = np.tanh(np.sqrt(2 / np.pi) * (x + 0.044715 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * np.sqrt(2 / np.pi) * (1 + 3 * 0.044715 * x * x)


@pytest.mark.parametrize("T", [1000, 300, 1, 8192])
def test_fused_gelu_forward_and_dx(R, torch, T):
    mem = 47192
    M_np = store(mem)
    ctx = R.Roast(to_dev(M_np, torch.float32), 64, 64, seed=HS)
    a, b = ctx.linear(768, 3072), ctx.linear(3072, 768)
    sa, sb = OM.LinearSpec(768, 3072, 64, 64, mem, HS, a), OM.LinearSpec(3072, 768, 64, 64, mem, HS, b)
    X_np = bf16_input(synth.SEED_X, (T, 768))
    dY_np = bf16_input(synth.SEED_DY, (T, 768))
    bias_np = synth.normal(synth.SEED_X + 3, (3072,)).astype(np.float32)
    X, dY = to_dev(X_np, torch.bfloat16), to_dev(dY_np, torch.bfloat16)
    bias = to_dev(bias_np, torch.float32)
    for _ in range(2):   # the first call tunes the unit width
        U, A = ctx.fwd_act(a, X, bias=bias)
        dU = ctx.bwd_dx_act(b, dY, U)
    torch.cuda.synchronize()
    ctx.check()
    U_np = U.float().cpu().numpy().astype(np.float64)
    A_np = A.float().cpu().numpy().astype(np.float64)
    rows = slice(None) if T <= 1000 else np.random.default_rng(1).choice(T, 256, replace=False)
    u_ref = sa.forward(X_np[rows], M_np, True) + bias_np.astype(np.float64)
    assert rel_frob(U_np[rows], u_ref) <= 1e-2
    # the activation is taken of the stored (bf16) U, as an unfused op would see it
    assert rel_frob(A_np, gelu(U_np)) <= 1e-2
    assert np.max(np.abs(A_np - gelu(U_np))) <= 2 ** -7 * max(1.0, np.abs(A_np).max())
    du_ref = sb.backward_dx(dY_np[rows], M_np, True) * gelu_grad(U_np[rows])
    assert rel_frob(dU.float().cpu().numpy()[rows], du_ref) <= 1e-2
    ctx.close()


def test_fused_gelu_unsupported_geometry_is_an_error(R, torch):
    """A handle whose tiles the tcgen05 path cannot take (32 x 32) reports UNSUPPORTED; the
    BERT MLP (nn.mlp) then runs the same math unfused."""
    ctx = R.Roast(torch.rand(1 << 16, device="cuda"), 32, 32, seed=HS, simt_bf16=True)
    a = ctx.linear(256, 512)
    X = torch.randn(64, 256, device="cuda").to(torch.bfloat16)
    with pytest.raises(R.RoastError) as e:
        ctx.fwd_act(a, X)
    assert e.value.status == R.ERR_UNSUPPORTED
    ctx.close()


def test_mlp_fused_equals_unfused_autograd(R, torch):
    """nn.mlp's fused autograd op against the unfused composition ff2(gelu(ff1(x))) through the
    same handle: output, input gradient and dM within the bf16 tolerance."""
    from paper_2207_10702_b200 import nn as RN
    M = torch.rand(47192, device="cuda") * 2 - 1
    outs = []
    for fused in (True, False):
        ctx = R.Roast(M.clone(), 64, 64, seed=HS)
        f1, f2 = RN.RoastLinear(ctx, 768, 3072, bias=True), RN.RoastLinear(ctx, 3072, 768, bias=True)
        g = torch.Generator(device="cuda").manual_seed(3)
        x = torch.randn(4, 250, 768, device="cuda", generator=g).to(torch.bfloat16).requires_grad_(True)
        dy = torch.randn(4, 250, 768, device="cuda", generator=g).to(torch.bfloat16)
        ctx.zero_grad()
        y = RN.mlp(f1, f2, x) if fused else f2(RN.gelu(f1(x)))
        y.backward(dy)
        ctx.flush_bias_grads()
        torch.cuda.synchronize()
        outs.append((y.float(), x.grad.float(), ctx.dM.clone()))
        ctx.close()
    for a, b in zip(outs[0], outs[1]):
        assert float((a - b).norm() / b.norm()) <= 1e-2


@pytest.mark.parametrize("T", [1000, 300, 8192])
def test_fused_chain_act_matches_oracle(R, torch, T):
    """The MLP pair with the GELU inside the chained forward and the fused backward
    (roast_linear_fwd_chain_act / _bwd_chain_act): every output against the fp64 oracle chain."""
    mem = 47192
    M_np = store(mem)
    ctx = R.Roast(to_dev(M_np, torch.float32), 64, 64, seed=HS)
    a, b = ctx.linear(768, 3072), ctx.linear(3072, 768)
    sa, sb = OM.LinearSpec(768, 3072, 64, 64, mem, HS, a), OM.LinearSpec(3072, 768, 64, 64, mem, HS, b)
    X_np = bf16_input(synth.SEED_X, (T, 768))
    dY_np = bf16_input(synth.SEED_DY, (T, 768))
    X, dY = to_dev(X_np, torch.bfloat16), to_dev(dY_np, torch.bfloat16)
    for _ in range(2):
        ctx.zero_grad()
        U, A, Y = ctx.fwd_chain_act(a, b, X)
        dU, dX = ctx.bwd_chain_act(a, b, X, A, U, dY)
    torch.cuda.synchronize()
    ctx.check()
    f = lambda t: t.float().cpu().numpy().astype(np.float64)   # noqa: E731
    U_np, A_np, dU_np = f(U), f(A), f(dU)
    rows = slice(None) if T <= 1000 else np.random.default_rng(2).choice(T, 192, replace=False)
    assert rel_frob(U_np[rows], sa.forward(X_np[rows], M_np, True)) <= 1e-2
    assert rel_frob(A_np, gelu(U_np)) <= 1e-2
    assert rel_frob(f(Y)[rows], sb.forward(A_np[rows], M_np, True)) <= 1e-2
    assert rel_frob(dU_np[rows], sb.backward_dx(dY_np[rows], M_np, True) * gelu_grad(U_np[rows])) <= 1e-2
    assert rel_frob(f(dX)[rows], sa.backward_dx(dU_np[rows], M_np, True)) <= 1e-2
    if T <= 1000:   # dM of both layers, the oracle's own dU chain
        dU_o = sb.backward_dx(dY_np, M_np, True) * gelu_grad(U_np)
        dM_ref = sb.backward_dm(A_np, dY_np) + sa.backward_dm(X_np, dU_o)
        assert rel_frob(ctx.dM.cpu().numpy(), dM_ref) <= 1e-2
    ctx.close()


def test_fused_gelu_shape_fuzz(R, torch):
    """Seeded random geometries through the fused-activation epilogues (both unit widths the tuner
    may pick, ragged tokens, small and odd tile counts, |M| small enough for shadow replicas):
    act(Y) and (dY W^T) * act'(U) against the oracle."""
    rng = np.random.default_rng(77)
    for case in range(8):
        mem = int(rng.choice([4720, 60_000]))
        M_np = store(mem)
        ctx = R.Roast(to_dev(M_np, torch.float32), 64, 64, seed=HS)
        H = 64 * int(rng.integers(1, 20))
        O = 192 * int(rng.integers(1, 8)) if rng.random() < 0.5 else 64 * int(rng.integers(1, 25))
        T = int(rng.integers(1, 3000))
        mid = ctx.linear(H, O)
        spec = OM.LinearSpec(H, O, 64, 64, mem, HS, mid)
        X_np = bf16_input(synth.SEED_X + case, (T, H))
        dY_np = bf16_input(synth.SEED_DY + case, (T, O))
        U_in = bf16_input(synth.SEED_X + 100 + case, (T, H))
        X, dY, Uin = to_dev(X_np, torch.bfloat16), to_dev(dY_np, torch.bfloat16), to_dev(U_in, torch.bfloat16)
        for _ in range(2):
            U, A = ctx.fwd_act(mid, X)
            dX = ctx.bwd_dx_act(mid, dY, Uin)
        torch.cuda.synchronize()
        ctx.check()
        where = (case, mem, H, O, T)
        U_np = U.float().cpu().numpy().astype(np.float64)
        assert rel_frob(U_np, spec.forward(X_np, M_np, True)) <= 1e-2, where
        assert rel_frob(A.float().cpu().numpy(), gelu(U_np)) <= 1e-2, where
        ref = spec.backward_dx(dY_np, M_np, True) * gelu_grad(U_in.astype(np.float64))
        assert rel_frob(dX.float().cpu().numpy(), ref) <= 1e-2, where
        ctx.close()


@pytest.mark.parametrize("T", [1, 300, 1000, 8192])
def test_residual_dx_equals_dx_plus_r(R, torch, T):
    """ROAST_ACT_RESIDUAL: dX = bf16(bf16(lambda dY W~^T) + R) in the dX epilogue has the bits of
    the plain dX GEMM followed by a separate bf16 add, for a single module (768-wide dX) and the
    fused QKV group (K = 2304), both unit widths (the tuner times both on the first call), R
    aliasing the output too; and it is the oracle's dX + R within the bf16 tolerance."""
    mem = 47192
    M_np = store(mem)
    ctx = R.Roast(to_dev(M_np, torch.float32), 64, 64, seed=HS)
    f1 = ctx.linear(768, 3072)
    q, k, v = ctx.linear(768, 768), ctx.linear(768, 768), ctx.linear(768, 768)
    gid = ctx.linear_concat([q, k, v])
    for mid, O, spec in ((f1, 3072, OM.LinearSpec(768, 3072, 64, 64, mem, HS, f1)), (gid, 2304, None)):
        dY_np = bf16_input(synth.SEED_DY + O, (T, O))
        R_np = bf16_input(synth.SEED_X + O, (T, 768))
        dY, Rr = to_dev(dY_np, torch.bfloat16), to_dev(R_np, torch.bfloat16)
        for _ in range(2):   # the first call tunes the unit width (times both)
            fused = ctx.bwd_dx_act(mid, dY, Rr, act=R.ACT_RESIDUAL)
        plain = torch.empty(T, 768, device="cuda", dtype=torch.bfloat16)
        ctx.bwd_dx(mid, dY, plain)
        inplace = Rr.clone()
        ctx.bwd_dx_act(mid, dY, inplace, dX=inplace, act=R.ACT_RESIDUAL)
        torch.cuda.synchronize()
        ctx.check()
        assert torch.equal(fused, plain + Rr), (mid, T)
        assert torch.equal(inplace, fused), (mid, T)
        if spec is not None:
            rows = slice(None) if T <= 1000 else np.random.default_rng(3).choice(T, 256, replace=False)
            ref = spec.backward_dx(dY_np[rows], M_np, True) + R_np[rows].astype(np.float64)
            assert rel_frob(fused.float().cpu().numpy()[rows], ref) <= 1e-2
    with pytest.raises(R.RoastError) as e:   # the residual form is a dX-only epilogue
        ctx.fwd_act(f1, torch.zeros(8, 768, device="cuda", dtype=torch.bfloat16), act=R.ACT_RESIDUAL)
    assert e.value.status == R.ERR_CONFIG
    ctx.close()


@pytest.mark.parametrize("fuse_min_tokens", [0, None])
def test_encoder_layer_residual_hand_off_is_bit_identical(R, torch, fuse_min_tokens, monkeypatch):
    """The BERT layer with the residual gradients handed to the QKV / MLP dX epilogues
    (nn.ResidualGrad) against the same layer with autograd adding them: output, input gradient,
    dM (deterministic mode: fast mode's reduce-adds land in any order) and the LayerNorm parameter
    gradients bit for bit (both add two bf16 tensors once)."""
    from paper_2207_10702_b200 import nn as RN
    if fuse_min_tokens is not None:   # 0: the fused epilogue at this size too (else plain dX + add)
        monkeypatch.setattr(RN, "RESIDUAL_FUSE_MIN_TOKENS", fuse_min_tokens)
    M = torch.rand(849352, device="cuda") * 2 - 1
    res = []
    for hand_off in (True, False):
        ctx = R.Roast(M.clone(), 64, 64, seed=HS, deterministic=True)
        layers = torch.nn.ModuleList([RN.EncoderLayer(ctx, 768, 3072, 12) for _ in range(2)]).cuda()
        for m in layers.modules():
            if isinstance(m, torch.nn.LayerNorm):
                m.to(torch.bfloat16)
        for lay in layers:
            lay.fuse_residual_grad = hand_off
        g = torch.Generator(device="cuda").manual_seed(9)
        x = torch.randn(4, 128, 768, device="cuda", generator=g).to(torch.bfloat16).requires_grad_(True)
        dy = torch.randn(4, 128, 768, device="cuda", generator=g).to(torch.bfloat16)
        ctx.zero_grad()
        y = x
        for lay in layers:
            y = lay(y)
        y.backward(dy)
        torch.cuda.synchronize()
        ctx.check()
        res.append([y, x.grad, ctx.dM.clone()] + [p.grad for lay in layers for p in (lay.ln1.weight, lay.ln2.bias)])
        ctx.close()
    for a, b in zip(res[0], res[1]):
        assert torch.equal(a, b)
