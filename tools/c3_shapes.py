"""The C3 encoder's GEMM shapes (per layer: fused QKV 768->2304, O 768->768, FF1 768->3072,
FF2 3072->768; 8192 tokens) through the tuned tcgen05 kernels next to cuBLAS: where the
linears' share of the step goes.  Graph-replayed, L2 warm (as inside the step).

    python tools/c3_shapes.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import roast as R  # noqa: E402


def t_us(fn, reps=30):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    T = 8192
    M = torch.rand(849352, device="cuda") * 2 - 1
    ctx = R.Roast(M, 64, 64)
    ctx.set_autotune(2)
    bf = torch.bfloat16
    tot_r = tot_c = 0.0
    for H, O in [(768, 2304), (768, 768), (768, 3072), (3072, 768)]:
        mid = ctx.linear(H, O)
        X = torch.randn(T, H, device="cuda").to(bf)
        dY = torch.randn(T, O, device="cuda").to(bf)
        Y = torch.empty(T, O, device="cuda", dtype=bf)
        dX = torch.empty(T, H, device="cuda", dtype=bf)
        W = ctx.materialize(mid, bf)
        row = dict(shape=f"{H}x{O}")
        for name, f, d in [("fwd", lambda: ctx.fwd(mid, X, Y), lambda: torch.matmul(X, W, out=Y)),
                           ("dx", lambda: ctx.bwd_dx(mid, dY, dX), lambda: torch.matmul(dY, W.t(), out=dX)),
                           ("dm", lambda: ctx.bwd_dm(mid, X, dY), lambda: torch.matmul(X.t(), dY))]:
            f()
            torch.cuda.synchronize()
            r, c = t_us(f), t_us(d)
            row[name] = dict(roast_us=round(r, 1), cublas_us=round(c, 1), tuned=ctx.tuned(mid, ["fwd", "dx", "dm"].index(name), T))
            tot_r += r
            tot_c += c
        print(json.dumps(row), flush=True)
    print(json.dumps(dict(per_layer_roast_us=round(tot_r, 1), per_layer_cublas_us=round(tot_c, 1),
                          ratio=round(tot_c / tot_r, 3))))


if __name__ == "__main__":
    main()
