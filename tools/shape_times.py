"""Per-launch times of the six C2 GEMMs (graph-replayed, L2 flushed before each) next to
cuBLAS on the same virtual shapes: where the ROAST kernels lose to the library.

    python tools/shape_times.py [--tune 0|2]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import roast as R  # noqa: E402


def timed(fn, flush, reps=30, warm=False):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(reps):
        if not warm:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tune", type=int, default=2)
    ap.add_argument("--T", type=int, default=8192)
    ap.add_argument("--warm", action="store_true", help="no L2 flush between replays")
    args = ap.parse_args()
    T = args.T
    M = torch.rand(47192, device="cuda") * 2 - 1
    ctx = R.Roast(M, 64, 64)
    ctx.set_autotune(args.tune)
    l1 = ctx.linear(768, 3072)
    l2 = ctx.linear(3072, 768)
    bf = torch.bfloat16
    X = torch.randn(T, 768, device="cuda").to(bf)
    dY2 = torch.randn(T, 768, device="cuda").to(bf)
    Y1 = torch.randn(T, 3072, device="cuda").to(bf)
    Y2 = torch.empty(T, 768, device="cuda", dtype=bf)
    dY1 = torch.randn(T, 3072, device="cuda").to(bf)
    dX = torch.empty(T, 768, device="cuda", dtype=bf)
    W1 = ctx.materialize(l1, bf)
    W2 = ctx.materialize(l2, bf)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = [
        ("fwd L1 768->3072", lambda: ctx.fwd(l1, X, Y1), lambda: torch.matmul(X, W1, out=Y1), (l1, 0)),
        ("fwd L2 3072->768", lambda: ctx.fwd(l2, Y1, Y2), lambda: torch.matmul(Y1, W2, out=Y2), (l2, 0)),
        ("dx L2 768->3072", lambda: ctx.bwd_dx(l2, dY2, dY1), lambda: torch.matmul(dY2, W2.t(), out=dY1), (l2, 1)),
        ("dx L1 3072->768", lambda: ctx.bwd_dx(l1, dY1, dX), lambda: torch.matmul(dY1, W1.t(), out=dX), (l1, 1)),
        ("dm L2 3072x768", lambda: ctx.bwd_dm(l2, Y1, dY2), lambda: torch.matmul(Y1.t(), dY2), (l2, 2)),
        ("dm L1 768x3072", lambda: ctx.bwd_dm(l1, X, dY1), lambda: torch.matmul(X.t(), dY1), (l1, 2)),
    ]
    ctx.fwd_chain(l1, l2, X, Y1, Y2)          # plan the chains eagerly
    ctx.bwd_dx_chain(l1, l2, dY2, dY1, dX)
    dYa = torch.empty_like(dY1)
    rows += [
        ("fwd chain L1+L2", lambda: ctx.fwd_chain(l1, l2, X, Y1, Y2),
         lambda: (torch.matmul(X, W1, out=Y1), torch.matmul(Y1, W2, out=Y2)), (l1, 0)),
        ("dx chain L2+L1", lambda: ctx.bwd_dx_chain(l1, l2, dY2, dYa, dX),
         lambda: (torch.matmul(dY2, W2.t(), out=dYa), torch.matmul(dYa, W1.t(), out=dX)), (l1, 1)),
    ]
    flop = 2.0 * T * 768 * 3072
    out = []
    for name, f, d, (mid, k) in rows:
        f()   # tune outside capture
        torch.cuda.synchronize()
        tr, td = timed(f, flush), timed(d, flush)
        if args.warm:
            tr, td = timed(f, flush, warm=True), timed(d, flush, warm=True)
        nf = 2 if "chain" in name else 1
        out.append(dict(kernel=name, roast_us=round(tr, 2), cublas_us=round(td, 2), ratio=round(td / tr, 3),
                        roast_tflops=round(nf * flop / tr / 1e6, 1), tuned=ctx.tuned(mid, k, T)))
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
