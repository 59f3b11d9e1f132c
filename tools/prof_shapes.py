"""Where the tcgen05 ROAST-MM kernels lose time, per C2 shape and kernel configuration.

For each of the six C2 GEMMs and each (WM, split-K) it times the launch (L2 warm, eager,
CUDA events) under the diagnostic knobs of `ROAST_EXP` (0 = the real kernel, 1 = no
epilogue drain, 2 = no TMA operand loads, 3 = MMAs only) next to cuBLAS on the same
virtual shape.  The gaps between the four say what bounds each kernel: MMA issue, operand
feed, or the accumulator drain.  Timing only: diagnostic launches compute garbage.

    ROAST_DIAG=1 python -m paper_2207_10702_b200.build -f    # knobs are compiled out otherwise
    python tools/prof_shapes.py [--T 8192] [--exps 0,1,2,3]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2207_10702_b200 import roast as R  # noqa: E402


def time_us(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=8192)
    ap.add_argument("--exps", default="0,1,2,3")
    ap.add_argument("--only", default="", help="substring filter on the kernel name")
    ap.add_argument("--dims", default="768,3072", help="d_model,d_ff of the two layers (C3 attention: 768,768)")
    ap.add_argument("--wm", default="", help="restrict to these WM values, e.g. 1,2")
    ap.add_argument("--prof", action="store_true", help="also print one ROAST_PROF counter line per config")
    ap.add_argument("--mem", type=int, default=47192, help="|M| (C2: 471864 / 47192 / 4720 at 10x / 100x / 1000x)")
    args = ap.parse_args()
    T = args.T
    D, F = [int(v) for v in args.dims.split(",")]
    M = torch.rand(args.mem, device="cuda") * 2 - 1
    ctx = R.Roast(M, 64, 64)
    ctx.set_autotune(0)
    l1 = ctx.linear(D, F)
    l2 = ctx.linear(F, D)
    bf = torch.bfloat16
    X = torch.randn(T, D, device="cuda").to(bf)
    dY2 = torch.randn(T, D, device="cuda").to(bf)
    Y1 = torch.randn(T, F, device="cuda").to(bf)
    Y2 = torch.empty(T, D, device="cuda", dtype=bf)
    dY1 = torch.randn(T, F, device="cuda").to(bf)
    dX = torch.empty(T, D, device="cuda", dtype=bf)
    W1 = ctx.materialize(l1, bf)
    W2 = ctx.materialize(l2, bf)
    rows = [
        (f"fwd L1 {D}->{F}", l1, 0, lambda: ctx.fwd(l1, X, Y1), lambda: torch.matmul(X, W1, out=Y1)),
        (f"fwd L2 {F}->{D}", l2, 0, lambda: ctx.fwd(l2, Y1, Y2), lambda: torch.matmul(Y1, W2, out=Y2)),
        (f"dx L2 {D}->{F}", l2, 1, lambda: ctx.bwd_dx(l2, dY2, dY1), lambda: torch.matmul(dY2, W2.t(), out=dY1)),
        (f"dx L1 {F}->{D}", l1, 1, lambda: ctx.bwd_dx(l1, dY1, dX), lambda: torch.matmul(dY1, W1.t(), out=dX)),
        (f"dm L2 {F}x{D}", l2, 2, lambda: ctx.bwd_dm(l2, Y1, dY2), lambda: torch.matmul(Y1.t(), dY2)),
        (f"dm L1 {D}x{F}", l1, 2, lambda: ctx.bwd_dm(l1, X, dY1), lambda: torch.matmul(X.t(), dY1)),
    ]
    flop = 2.0 * T * D * F
    exps = [int(e) for e in args.exps.split(",")]
    for name, mid, kind, f, d in rows:
        if args.only and args.only not in name:
            continue
        td = time_us(d)
        cfgs = [(1, 1), (2, 1), (2, 3)] if kind < 2 else [(1, 1), (1, 2), (1, 3), (1, 4), (1, 8), (2, 1), (2, 2), (2, 4)]
        if args.wm:
            cfgs = [c for c in cfgs if str(c[0]) in args.wm.split(",")]
        for wm, sp in cfgs:
            ctx.set_tuned(mid, kind, T, wm, sp)
            res = {}
            for e in exps:
                os.environ["ROAST_EXP"] = str(e)
                res[e] = round(time_us(f), 2)
            os.environ.pop("ROAST_EXP", None)
            line = dict(kernel=name, wm=wm, splits=sp, us=res, tflops=round(flop / res[exps[0]] / 1e6, 1),
                        cublas_us=round(td, 2), cublas_tflops=round(flop / td / 1e6, 1))
            print(json.dumps(line), flush=True)
            if args.prof:
                os.environ["ROAST_PROF"] = "1"
                f()
                torch.cuda.synchronize()
                os.environ.pop("ROAST_PROF")


if __name__ == "__main__":
    main()
