"""roast_layernorm_fwd / _bwd (the BERT workload's LayerNorm, include/roast.h) against torch's
LayerNorm evaluated in fp64 on the same values: forward, input gradient (with and without the
fused residual) and parameter gradients; the parameter gradients are bitwise reproducible."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available()
    return torch


def _rel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm())


@pytest.mark.parametrize("dtype,n,rows,resid", [("bf16", 768, 4099, True), ("bf16", 768, 3, False),
                                                ("fp32", 1024, 777, True), ("fp32", 2048, 64, False),
                                                ("bf16", 8, 1000, True), ("bf16", 768, 70001, True),
                                                ("fp32", 768, 5000, False), ("bf16", 2048, 3001, True)])
def test_layernorm_matches_torch(torch, dtype, n, rows, resid):
    from paper_2207_10702_b200 import nn as RN
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    tol = 1e-2 if dtype == "bf16" else 1e-5
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(rows, n, device="cuda", generator=g).to(dt).requires_grad_(True)
    r = torch.randn(rows, n, device="cuda", generator=g).to(dt).requires_grad_(True) if resid else None
    dy = torch.randn(rows, n, device="cuda", generator=g).to(dt)
    ln = RN.LayerNorm(n, device="cuda", dtype=dt)
    with torch.no_grad():
        ln.weight.copy_(torch.randn(n, device="cuda", generator=g))
        ln.bias.copy_(torch.randn(n, device="cuda", generator=g))
    y = ln(x, r)
    y.backward(dy)
    # reference: fp64 on the same (rounded) inputs; the LN input is x + r rounded to dt, as stored
    xd = x.detach().double().requires_grad_(True)
    rd = r.detach().double().requires_grad_(True) if resid else None
    s = (xd + rd).to(dt).double() if resid else xd
    ref = torch.nn.LayerNorm(n, device="cuda", dtype=torch.float64)
    with torch.no_grad():
        ref.weight.copy_(ln.weight.double())
        ref.bias.copy_(ln.bias.double())
    yr = ref(s.detach())
    assert _rel(y, yr) <= tol
    # the gradient w.r.t. the LN input (the rounding of s to dt is not differentiated): ds flows
    # to x and r alike
    sd = s.detach().requires_grad_(True)
    ref.zero_grad()
    ref(sd).backward(dy.double())
    assert _rel(x.grad, sd.grad) <= tol
    if resid:
        assert torch.equal(x.grad, r.grad)
    assert _rel(ln.weight.grad, ref.weight.grad) <= tol
    assert _rel(ln.bias.grad, ref.bias.grad) <= tol
    # reproducible parameter gradients (fixed-order reduction)
    w1 = ln.weight.grad.clone()
    ln.zero_grad()
    x.grad = None
    ln(x, r).backward(dy)
    assert torch.equal(ln.weight.grad, w1)


def test_layernorm_errors(torch):
    from paper_2207_10702_b200 import roast as R
    buf = torch.empty(64, device="cuda")
    with pytest.raises(R.RoastError):
        R.roast_layernorm_fwd(buf.data_ptr(), None, buf.data_ptr(), buf.data_ptr(), buf.data_ptr(), None,
                              buf.data_ptr(), buf.data_ptr(), 1, 12, 1e-5, R.FP32, R.FP32)   # n % 8 != 0
    with pytest.raises(R.RoastError):
        R.roast_layernorm_fwd(buf.data_ptr(), buf.data_ptr(), buf.data_ptr(), buf.data_ptr(), buf.data_ptr(), None,
                              buf.data_ptr(), buf.data_ptr(), 1, 16, 1e-5, R.FP32, R.FP32)   # residual without s_out


def test_layernorm_zero_rows(torch):
    """rows = 0: the forward writes nothing; the backward's parameter gradients are zero (overwritten,
    as for any row count) and nothing else is touched."""
    from paper_2207_10702_b200 import roast as R
    n = 768
    g = torch.ones(n, device="cuda")
    b = torch.zeros(n, device="cuda")
    dg = torch.full((n,), 7.0, device="cuda")
    db = torch.full((n,), 7.0, device="cuda")
    buf = torch.empty(16, device="cuda")
    R.roast_layernorm_fwd(buf.data_ptr(), None, g.data_ptr(), b.data_ptr(), buf.data_ptr(), None,
                          buf.data_ptr(), buf.data_ptr(), 0, n, 1e-5, R.FP32, R.FP32)
    R.roast_layernorm_bwd(buf.data_ptr(), buf.data_ptr(), g.data_ptr(), buf.data_ptr(), buf.data_ptr(), buf.data_ptr(),
                          dg.data_ptr(), db.data_ptr(), 0, n, R.FP32, R.FP32)
    torch.cuda.synchronize()
    assert torch.count_nonzero(dg) == 0 and torch.count_nonzero(db) == 0


@pytest.mark.parametrize("rows", [1, 7, 2000, 2100])
def test_layernorm_backward_row_ranges(torch, rows):
    """The backward's per-warp row ranges (a fixed function of the row count: rows per warp 1 or 2
    around 148 x 12 warps) against fp64 torch, parameter gradients reproducible."""
    from paper_2207_10702_b200 import nn as RN
    n = 256
    gen = torch.Generator(device="cuda").manual_seed(rows)
    x = torch.randn(rows, n, device="cuda", generator=gen).to(torch.bfloat16).requires_grad_(True)
    dy = torch.randn(rows, n, device="cuda", generator=gen).to(torch.bfloat16)
    ln = RN.LayerNorm(n, device="cuda", dtype=torch.bfloat16)
    ln(x).backward(dy)
    ref = torch.nn.LayerNorm(n, device="cuda", dtype=torch.float64)
    xd = x.detach().double().requires_grad_(True)
    ref(xd).backward(dy.double())
    assert _rel(x.grad, xd.grad) <= 1e-2
    assert _rel(ln.weight.grad, ref.weight.grad) <= 1e-2
    assert _rel(ln.bias.grad, ref.bias.grad) <= 1e-2
