"""Fused-GELU epilogue cost at C3's MLP shapes (T = 65 536): ROAST fwd / dX with and without the
activation, against torch's GELU kernels on the same tensors (graph replays, median)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import roast as R  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 65536


def t_us(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return sorted(ts)[len(ts) // 2]


ctx = R.Roast(torch.rand(849352, device="cuda") * 2 - 1, 64, 64)
a, b = ctx.linear(768, 3072), ctx.linear(3072, 768)
bf = torch.bfloat16
X = torch.randn(T, 768, device="cuda").to(bf)
dY = torch.randn(T, 768, device="cuda").to(bf)
U = torch.empty(T, 3072, device="cuda", dtype=bf)
A = torch.empty_like(U)
dU = torch.empty_like(U)
res = dict(T=T)
res["fwd_plain_us"] = t_us(lambda: ctx.fwd(a, X, U))
res["fwd_act_us"] = t_us(lambda: ctx.fwd_act(a, X, U, A))
res["dx_plain_us"] = t_us(lambda: ctx.bwd_dx(b, dY, dU))
res["dx_act_us"] = t_us(lambda: ctx.bwd_dx_act(b, dY, U, dU))
res["torch_gelu_fwd_us"] = t_us(lambda: torch.nn.functional.gelu(U, approximate="tanh"))
Ur = U.clone().requires_grad_(True)
res["torch_gelu_bwd_us"] = t_us(lambda: torch.ops.aten.gelu_backward(dU, Ur, approximate="tanh"))
# residual form (ROAST_ACT_RESIDUAL) on the 768-wide dX GEMMs of the layer: ff1 (K = 3072) and the
# fused QKV group (K = 2304), against the plain dX GEMM + torch's bf16 add
q, k, v = ctx.linear(768, 768), ctx.linear(768, 768), ctx.linear(768, 768)
gid = ctx.linear_concat([q, k, v])
Rr = torch.randn(T, 768, device="cuda").to(bf)
dX = torch.empty(T, 768, device="cuda", dtype=bf)
dQ = torch.randn(T, 2304, device="cuda").to(bf)
res["ff1_dx_plain_us"] = t_us(lambda: ctx.bwd_dx(a, dU, dX))
res["ff1_dx_residual_us"] = t_us(lambda: ctx.bwd_dx_act(a, dU, Rr, dX, act=R.ACT_RESIDUAL))
res["qkv_dx_plain_us"] = t_us(lambda: ctx.bwd_dx(gid, dQ, dX))
res["qkv_dx_residual_us"] = t_us(lambda: ctx.bwd_dx_act(gid, dQ, Rr, dX, act=R.ACT_RESIDUAL))
res["torch_add_us"] = t_us(lambda: torch.add(dX, Rr))
print(json.dumps({k: round(v, 1) if isinstance(v, float) else v for k, v in res.items()}))
